"""Throughput benchmark of the B200 relaxation loop (spring updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload at N=1 (BASELINE.json configs[3]): the synthetic 10M-spring cube
lattice ``block_scene(91)`` (9,896,068 springs, 778,688 masses, pitch 0.1 m,
k=1000/l0, m=0.1 kg, gravity off), excited like reference
tests/test_acceptance.py:75-83 (seed 11), position Verlet (the reference
default, engine.py:182), dt=1e-4.  The headline is the fp64 validation mode,
bitwise equal to the reference's serial engine (the reference computes in
fp64); the fp32 production mode is reported beside it (``fp32_production``).
One bench step = ``Engine.step(100)`` -- 100 substeps, the reference bench's
MIN_STEPS (bench.py:21) -- so value = springs x 100 x K / time.

N>1 (torchrun): the 400M-spring cube (configs[4], ``block_scene(313)``) split
into x-slabs, one per rank, with the halo exchange fused into every substep
(paper_2207_09334_b200/sharded.py).  The N=1 line carries the same 400M cube
on one GPU through the sharded path as ``scaling_1gpu`` (same workload
string), the denominator of a 1->N curve.

``--impl reference``: the reference's CPU algorithm (oracle/ port of
_kernels.py + engine.py, the reference bench's default "parallel" mode,
bench.py:91-93) on the host's physical cores, on the same workload, built by
the oracle's own restatement of the lattice builder -- nothing from the
product package is imported or loaded on that arm.

Keys beyond the driver contract: ``roofline`` (HBM: SURVEY 8d algorithmic
bytes per substep launch / average launch time vs MEASURED_PEAKS.json, and
``frac_dram`` from the kernel's ncu DRAM bytes), ``cpu_baseline``, ``e2e``
(the same metric through the public Engine API with the host state uploaded
and positions read back every step).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SUBSTEPS = 100
HBM_FALLBACK_GBS = 6650.0       # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)
METRIC = "spring updates/sec (springs×steps/s) at 1/2/4/8 B200; HBM GB/s vs peak"   # BASELINE.json
UNIT = "spring-updates/s"
# SURVEY 8d algorithmic bytes: per spring (2 x int32 endpoints + k + l0) and
# per mass (read x and the history vector, write x and v; 16 B or 32 B vectors)
ALGO_BYTES = {"f32": (16, 64), "f64": (24, 128)}


def workload_config(cells: int, springs: int, masses: int, precision: str) -> dict:
    """The ``config`` object both arms print (identical for the same run)."""
    if cells == 91:
        name = "cube_n91_10M_springs_excited_verlet"
    elif cells == 313:
        name = "cube_n313_400M_springs_excited_verlet_x_slabs"
    else:
        name = f"cube_n{cells}_excited_verlet"
    return {"workload": name, "cells": cells, "springs": springs, "masses": masses,
            "integrator": "verlet", "dt": 1e-4, "precision": precision,
            "init": "block_scene(n), velocities N(0,0.05)+(0.3,0.2,0.1), seed 11"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons, 100 ms samples time-stamped on
    arrival; ``summary()`` keeps the samples inside the marked timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.windows: list[tuple[float, float]] = []
        self.t0 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            time.sleep(0.3)              # sampler up before the first timed region
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.windows.append((self.t0, time.time()))
        time.sleep(0.25)                 # let the sample covering the end arrive

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if not any(lo - 0.05 <= ts <= hi + 0.15 for lo, hi in self.windows):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "window_s": round(sum(b - a for a, b in self.windows), 3)}


def profiled_traffic(workload: str, precision: str, fmt: str):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/traffic.json), or None if this config was not profiled."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    entry = json.load(open(p)).get(f"{workload}/{precision}/{fmt}")
    return None if entry is None else entry["bytes"]


# ------------------------------------------------------------ CPU (oracle)

def oracle_module():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc                 # test infrastructure: the CPU checker / baseline only
    return orc


def cpu_workload(cells: int, planes: int | None = None):
    """The bench cube built by the oracle (no product code): the whole
    ``block_scene(cells)`` or, with ``planes``, the slab of its first
    ``planes`` x-cells (a bounded sample of the same lattice)."""
    orc = oracle_module()
    return orc.excite(orc.block_arrays(cells, cells_x=planes), seed=11)


def time_oracle(arrays, mode: str, threads: int, target_s: float, max_steps: int, warmup: int = 1):
    orc = oracle_module()
    eng = orc.OracleEngine(arrays, integrator="verlet", mode=mode, threads=threads)
    eng.step(max(warmup, 1))             # first touch of the slot slab
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps:
        eng.step(1)
        steps += 1
        if time.perf_counter() - t0 >= target_s:
            break
    wall = time.perf_counter() - t0
    return arrays.spring_count * steps / wall, steps, wall


def cpu_baseline(cells: int, planes: int | None = None) -> dict:
    """Bounded CPU sample of the same cube in each of the reference's modes
    (parallel and parallel-det on the physical cores, serial on one);
    ``value`` is the fastest."""
    orc = oracle_module()
    arr = cpu_workload(cells, planes)
    cores = orc.physical_cores()
    what = (f"the {arr.spring_count}-spring cube" if planes is None else
            f"a {planes}-cell x-slab ({arr.spring_count} springs) of the same cube")
    modes = {}
    for mode, threads, budget, cap in (("parallel", cores, 8.0, 40), ("parallel-det", cores, 8.0, 40),
                                       ("serial", 1, 6.0, 20)):
        v, k, w = time_oracle(arr, mode, threads, budget, cap)
        modes[mode] = {"value": v, "threads": threads, "steps": k, "wall_s": round(w, 2)}
    best = max(modes, key=lambda m: modes[m]["value"])
    return {"value": modes[best]["value"], "unit": UNIT, "cores": modes[best]["threads"], "kind": "port",
            "sample": f"{modes[best]['steps']} Verlet steps ({modes[best]['wall_s']} s) of {what} in the fastest "
                      f"of the reference's modes ({best}) restated in C/OpenMP (oracle/); every mode in 'modes'",
            "host_threads": os.cpu_count(), "physical_cores": cores, "modes": modes}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port of
    _kernels.py + engine.py) on the b200 arm's workload, in each of the
    reference's execution modes -- "parallel" (its bench's default,
    bench.py:91-93: the Alg. 1 atomic slot schedule) and "parallel-det" on
    the physical cores, "serial" on one -- reporting the fastest (on the B200
    hosts the serial mode wins: the slot traffic outweighs the threads).
    N>1: rank 0 only, on a bounded x-slab sample of the 400M cube."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    orc = oracle_module()
    cells = args.cells or (313 if world > 1 else 91)
    planes = None
    if cells > 150:                       # 400M: a bounded slab sample of the same lattice
        planes = 16
    arr = cpu_workload(cells, planes)
    cores = orc.physical_cores()
    steps = args.steps
    modes = {}
    for mode, threads in (("parallel", cores), ("parallel-det", cores), ("serial", 1)):
        eng = orc.OracleEngine(arr, integrator="verlet", mode=mode, threads=threads)
        for _ in range(max(args.warmup, 1)):
            eng.step(1)
        t0 = time.perf_counter()
        for _ in range(steps):
            eng.step(1)
        wall = time.perf_counter() - t0
        modes[mode] = {"value": arr.spring_count * steps / wall, "threads": threads, "ms_per_step": 1e3 * wall / steps}
        del eng
    best = max(modes, key=lambda k: modes[k]["value"])
    value, cores_used = modes[best]["value"], modes[best]["threads"]
    n = cells + 1
    s_full = 13 * cells ** 3 + 12 * cells ** 2 + 3 * cells
    sample = (f"{steps} Verlet steps of the {arr.spring_count}-spring cube" if planes is None else
              f"{steps} Verlet steps of a {planes}-cell x-slab ({arr.spring_count} springs) of the "
              f"{s_full}-spring cube")
    sample += (f" per mode; the fastest of the reference's modes ({best}, {cores_used} thread(s)) restated in "
               "C/OpenMP (_kernels.py:44-155, engine.py:261-381); lattice built by the oracle's restatement of "
               "build_voxel_lattice")
    print(json.dumps({
        "metric": METRIC, "impl": "reference", "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": modes[best]["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(cells, s_full, n ** 3, "f64"),
        "substeps_per_step": 1,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores_used, "kind": "port", "sample": sample,
                         "host_threads": os.cpu_count(), "physical_cores": cores, "modes": modes},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------ GPU (b200)

def kernel_of(info: dict) -> tuple[str, str]:
    """(record format, dominant kernel) of an engine (ss_info.tile_kernel)."""
    layout = {1: "csr", 2: "ell", 3: "tile"}[info["layout"]]
    if layout != "tile":
        return layout, "step_kernel"
    fp32 = info["precision"] == 1
    tk = info["tile_kernel"]
    if fp32:
        return {2: ("tile_compact", "tile_lean_kernel"), 6: ("tile_inline", "tile_lean_kernel"),
                7: ("tile_compact_x0", "tile_lean_kernel"),
                1: ("tile_explicit", "tile_lean_kernel")}.get(tk, ("tile_explicit", "step_kernel"))
    return {5: ("tile_inline", "tile_f64_kernel"), 4: ("tile_compact", "tile_f64_kernel"),
            3: ("tile_compact", "step_kernel")}.get(tk, ("tile_explicit", "step_kernel"))


def slab_line(r: dict, precision: str, world: int, peak: float, clocks=None, cpu=None) -> dict:
    """The JSON line (or the scaling_1gpu object) of an x-slab run."""
    S, n = r["springs"], r["masses"]
    per_spring, per_mass = ALGO_BYTES[precision]
    per_sub = r["ms"] / 1e3 / (r["steps"] * r["substeps"])
    achieved = (per_spring * S + per_mass * n) / per_sub / 1e9 / world
    transport = {"p2p": "peer memory (NVLink P2P stores + device flags)", "nccl": "NCCL send/recv"}
    return {
        "metric": METRIC, "value": S * r["substeps"] * r["steps"] / (r["ms"] / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": r["steps"], "warmup": r.get("warmup"),
        "ms_per_step": r["ms"] / r["steps"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": precision, "data": "synthetic",
        "config": workload_config(r["cells"], S, n, precision),
        "substeps_per_step": r["substeps"],
        "parallelism": (f"x-slab x{world}, halo exchange fused into every substep over "
                        + transport.get(r["transport"], r["transport"])) if world > 1
                       else "one GPU through the sharded path (one slab, no neighbours)",
        "l2": "inputs larger than L2",
        "halo_plane_bytes": r["halo_plane_bytes"], "build_s_rank0": round(r["build_s"], 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "note": "per GPU: whole-job SURVEY 8d algorithmic bytes / time / N"},
        "cpu_baseline": cpu,
        "e2e": {"value": S * r["substeps"] * r["e2e_steps"] / r["e2e_wall_s"], "unit": UNIT,
                "h2d_bytes_per_step": r["h2d_bytes_per_step"], "d2h_bytes_per_step": r["d2h_bytes_per_step"]},
        "gpu_launches": r["launches"],
        "clocks": clocks,
    }


def bench_main(args):
    """N>1 under torchrun: the 400M-spring cube (configs[4]) in x-slabs, one
    per rank (sharded.bench_slabs); rank 0 prints the line, time = max over
    ranks, plus a bounded CPU sample of the same lattice."""
    import torch
    import torch.distributed as dist
    from paper_2207_09334_b200 import sharded
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # SS_BENCH_SAME_DEVICE=1 (testing the N>1 path on a one-GPU box): every
    # rank on cuda:0, host coordination over gloo (NCCL refuses duplicate GPUs)
    same_device = os.environ.get("SS_BENCH_SAME_DEVICE") == "1"
    if same_device:
        local = 0
    torch.cuda.set_device(local)
    if same_device:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cells = args.cells or 313
    with ClockSampler(local) as clk:
        r = sharded.bench_slabs(cells, args.precision, args.steps, args.warmup, args.substeps, args.layout,
                                rank, world, dist, local, clk)
    r["warmup"] = args.warmup
    clocks = clk.summary()
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(cells, planes=16 if cells > 150 else None)
    dist.barrier()
    if rank == 0:
        print(json.dumps(slab_line(r, args.precision, world, peaks()[0], clocks, cpu)), flush=True)
    dist.destroy_process_group()


def time_device(eng, steps: int, warmup: int, sub: int, clk: ClockSampler | None):
    """K bench steps of ``sub`` substeps on the engine stream, L2 flushed
    before each (a write of twice its size, outside the per-step events).
    Returns (total ms, launches)."""
    import torch
    stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", 0))
    for _ in range(max(warmup, 3)):
        eng.step_async(sub)
    eng.synchronize()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(2 * max(l2, 64 << 20), dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches0 = eng.launch_count
    torch.cuda.synchronize()
    if clk:
        clk.start()
    for a, b in ev:
        with torch.cuda.stream(stream):
            flush.zero_()
        a.record(stream)
        eng.step_async(sub)
        b.record(stream)
    ev[-1][1].synchronize()
    if clk:
        clk.stop()
    eng.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    return ms, eng.launch_count - launches0


def time_e2e(eng, steps: int, sub: int):
    """Public-API steps: host state (x, v, x_prev) assigned from page-locked
    host arrays, ``step(sub)``, positions read back -- every step."""
    from paper_2207_09334_b200 import pinned_copy
    x_h, v_h, xp_h = (pinned_copy(a) for a in (eng.x, eng.v, eng.x_prev))
    for _ in range(2):                   # untimed: staging buffers, events
        eng.x, eng.v, eng.x_prev = x_h, v_h, xp_h
        eng.step(sub)
        _ = eng.x
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.x, eng.v, eng.x_prev = x_h, v_h, xp_h
        eng.step(sub)
        out = eng.x
    wall = time.perf_counter() - t0
    del out
    return wall


def engine_leg(scene, precision: str, args, clk, workload: str, e2e_steps: int, label: str):
    """Device throughput, roofline and e2e of one Engine on the bench cube."""
    from paper_2207_09334_b200 import Engine
    S, N = scene.spring_count, scene.mass_count
    sub = args.substeps
    eng = Engine(scene, integrator="verlet", precision=precision, layout=args.layout)
    info = eng.info()
    ms, launches = time_device(eng, args.steps, args.warmup, sub, clk)
    value = S * sub * args.steps / (ms / 1e3)
    per_launch_s = ms / 1e3 / launches
    peak, peak_kind = peaks()
    per_spring, per_mass = ALGO_BYTES[precision]
    algo = per_spring * S + per_mass * N
    fmt, kernel = kernel_of(info)
    traffic = profiled_traffic(workload, precision, fmt)
    achieved = algo / per_launch_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "frac_dram": (traffic / per_launch_s / 1e9 / peak) if traffic else None,
            "peak_kind": peak_kind, "algorithmic_bytes_per_launch": algo,
            "algorithmic_model": f"SURVEY 8d: {per_spring} B/spring + {per_mass} B/mass",
            "avg_launch_us": per_launch_s * 1e6, "kernel": kernel,
            "format": fmt, "records_bytes_per_substep": info["tile_blob_bytes"]}
    if traffic and traffic < algo:
        roof["note"] = ("the compact record format streams %.1f B/spring of records instead of the "
                        "model's %d, so measured DRAM bytes (traffic) are below the algorithmic bytes; "
                        "frac_dram is the measured-DRAM fraction of peak" % (info["tile_blob_bytes"] / S,
                                                                               per_spring))
    e2e = None
    if e2e_steps:
        wall = time_e2e(eng, e2e_steps, sub)
        # the caller's (N, 3) f64 arrays: x, v, x_prev in, x out.  fp64 moves
        # exactly these over the bus (permuted on the device); fp32 packs them
        # on the host into 16-byte device slots first
        vec = 3 * 8
        e2e = {"value": S * sub * e2e_steps / wall, "unit": UNIT, "steps": e2e_steps,
               "h2d_bytes_per_step": 3 * N * vec, "d2h_bytes_per_step": N * vec,
               "bus_bytes_per_mass_vector": 24 if precision == "f64" else 16,
               "host_memory": "page-locked numpy arrays (paper_2207_09334_b200.pinned_copy); "
                              "readbacks land in the engine's pooled page-locked buffers"}
    eng.close()
    return {"value": value, "ms_per_step": ms / args.steps, "launches": launches, "roofline": roof,
            "e2e": e2e, "dtype": precision, "label": label,
            "layout_info": {"format": fmt, "tile_halo_ratio": round(info["tile_halo_ratio"], 3),
                            "records_bytes_per_substep": info["tile_blob_bytes"],
                            "device_bytes": info["device_bytes"]}}


def run_single(args):
    import torch  # noqa: F401  (CUDA context, events)
    from paper_2207_09334_b200 import lattice as L
    cells = args.cells or 91
    scene = L.excite(L.block_scene(cells), seed=11)
    S, N = scene.spring_count, scene.mass_count
    cfg = workload_config(cells, S, N, args.precision)
    workload = cfg["workload"]
    e2e_steps = max(2, min(args.steps, 10))
    with ClockSampler(0) as clk:
        head = engine_leg(scene, args.precision, args, clk, workload, e2e_steps, "headline")
        other = None
        if not args.no_extra:
            alt = "f32" if args.precision == "f64" else "f64"
            other = engine_leg(scene, alt, args, clk, workload, e2e_steps, "other precision")
        general = {}
        if not args.no_extra:
            # the general-graph record format (records per incidence, what any
            # scene whose tiles do not fit the compact dictionary runs) on the
            # same cube, in both precisions
            os.environ["SS_TILE_DICT"] = "0"
            try:
                for prec in (args.precision, "f32" if args.precision == "f64" else "f64"):
                    general[prec] = engine_leg(scene, prec, args, clk, workload, 0, "inline records")
            finally:
                del os.environ["SS_TILE_DICT"]
        scaling = None
        if not args.no_400m:
            # the 400M cube on this GPU through the sharded path: the 1-GPU
            # point of the N>1 lines (same workload string)
            from paper_2207_09334_b200 import sharded
            r = sharded.bench_slabs(313, args.precision, max(3, min(args.steps, 10)), 3, args.substeps,
                                    args.layout, clk=clk)
            r["warmup"] = 3
            scaling = slab_line(r, args.precision, 1, peaks()[0])
            scaling.pop("clocks")
    cpu = None if args.no_cpu else cpu_baseline(cells)
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": cfg,
        "substeps_per_step": args.substeps,
        "l2": "L2 flushed before every timed step (a write of twice its size); per-step CUDA events "
              "exclude the flush",
        "parallelism": "single-gpu",
        "roofline": head["roofline"],
        "layout_info": head["layout_info"],
        "e2e": head["e2e"],
        "gpu_launches": head["launches"],
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if other:
        key = "fp32_production" if other["dtype"] == "f32" else "fp64_validation"
        line[key] = {"value": other["value"], "unit": UNIT, "ms_per_step": other["ms_per_step"],
                     "dtype": other["dtype"], "roofline": other["roofline"], "e2e": other["e2e"],
                     "gpu_launches": other["launches"],
                     "note": ("fp32 production mode: displacement form, within 1e-4 relative of the "
                              "reference (DESIGN.md 5)") if other["dtype"] == "f32" else
                             "fp64 validation mode, bitwise equal to the reference's serial engine"}
    for prec, g in general.items():
        key = "general_graph_format" if prec == args.precision else "general_graph_format_" + prec
        line[key] = {
            "value": g["value"], "unit": UNIT, "ms_per_step": g["ms_per_step"],
            "dtype": g["dtype"], "roofline": g["roofline"],
            "note": "SS_TILE_DICT=0: the general-graph record format (records per incidence streamed "
                    "from HBM: fp64 (k, l0), fp32 (k, k*l0) with D formed from the staged X0) -- what a scene whose tiles do not fit "
                    "the 64-entry dictionary runs -- on the same cube"}
    if scaling:
        line["scaling_1gpu"] = scaling
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cells", type=int, default=0)
    ap.add_argument("--substeps", type=int, default=SUBSTEPS)
    ap.add_argument("--precision", default="f64", choices=["f32", "f64"])
    ap.add_argument("--layout", default="auto", choices=["auto", "csr", "ell"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the other-precision and explicit-format measurements")
    ap.add_argument("--no-400m", action="store_true", help="skip the one-GPU 400M (scaling_1gpu) leg")
    ap.add_argument("--sharded", action="store_true",
                    help="run the x-slab sharded path even on one rank (400M cube by default)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29612")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        bench_main(args)
        return
    if args.gpus > 1:
        # not launched under torchrun: launch one process per GPU ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", "--master-port=29611",
               os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    run_single(args)


if __name__ == "__main__":
    main()
