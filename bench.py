"""Throughput benchmark of the B200 relaxation loop (spring updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[3]): the synthetic 10M-spring cube lattice
(``block_scene(91)``: 9,896,068 springs, 778,688 masses, pitch 0.1 m, k=1000/l0,
m=0.1 kg, gravity off), excited like reference tests/test_acceptance.py:75-83
(seed 11), position Verlet (the reference default, engine.py:182), dt=1e-4,
fp32 production mode.  One bench step = ``Engine.step(100)`` — 100 substeps,
the reference bench's MIN_STEPS (bench.py:21) — so value = springs x 100 x K /
time.  N>1 (torchrun): the 400M-spring cube (configs[4]) split into x-slabs
(one per rank) with a halo exchange every substep.

Keys beyond the driver contract: ``roofline`` (HBM: algorithmic bytes per
substep launch / average launch time vs MEASURED_PEAKS.json), ``cpu_baseline``
(the oracle's restatement of the reference's default parallel schedule on the
host's cores, bounded sample), ``e2e`` (the same metric through the public
Engine API with host state uploaded and positions read back every step).
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
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()
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
        lo = (self.t0 or 0.0) - 0.05
        hi = (self.t1 or time.time()) + 0.15
        for ts, ln in self.lines:
            if not lo <= ts <= hi:
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
                "window_s": round((self.t1 or 0) - (self.t0 or 0), 3)}


def profiled_traffic(workload: str, precision: str, layout: str):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/traffic.json), or None if this config was not profiled."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    entry = json.load(open(p)).get(f"{workload}/{precision}/{layout}")
    return None if entry is None else entry["bytes"]


def cpu_sample(scene, target_s=12.0, max_steps=40, threads=None, mode="parallel"):
    """Time the oracle's restatement of the reference's parallel mode (the
    reference bench's default, bench.py:93: Alg. 1 atomic slot schedule,
    OpenMP, all host threads) -- or its serial mode on one core -- on the
    host: bounded sample of Verlet steps."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    from paper_2207_09334_b200.model import scene_arrays
    threads = 1 if mode == "serial" else (threads or orc.max_threads())
    eng = orc.OracleEngine(scene_arrays(scene), integrator="verlet", mode=mode, threads=threads)
    eng.step(1)                          # warm-up (first touch of the slab)
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps:
        eng.step(1)
        steps += 1
        if time.perf_counter() - t0 >= target_s:
            break
    wall = time.perf_counter() - t0
    return scene.spring_count * steps / wall, steps, wall, threads


def build_workload(cells):
    from paper_2207_09334_b200 import lattice as L
    return L.excite(L.block_scene(cells), seed=11)


def run_reference(args):
    """--impl reference: the reference's CPU algorithm in its bench's default
    mode (bench.py:91-93: "parallel", the Alg. 1 atomic slot schedule; oracle
    port, all host threads), same config/metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cells = args.cells or 91
    scene = build_workload(cells)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    from paper_2207_09334_b200.model import scene_arrays
    threads = orc.max_threads()
    eng = orc.OracleEngine(scene_arrays(scene), integrator="verlet", mode="parallel", threads=threads)
    for _ in range(max(args.warmup, 1)):
        eng.step(1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        eng.step(1)
    wall = time.perf_counter() - t0
    value = scene.spring_count * args.steps / wall
    unit = "spring-updates/s"
    print(json.dumps({
        "metric": "spring updates/sec (springs x steps / s)", "impl": "reference",
        "value": value, "unit": unit, "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "none",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cube_n{cells}_excited_verlet", "cells": cells,
                   "springs": scene.spring_count, "masses": scene.mass_count,
                   "step": "one reference Engine.step() (1 substep) per bench step"},
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} Verlet steps of the {scene.spring_count}-spring cube, "
                                   f"the reference bench's default parallel mode (Alg.1 atomic slots) "
                                   f"restated in C/OpenMP"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_single(args):
    import torch
    from paper_2207_09334_b200 import Engine
    cells = args.cells or 91
    scene = build_workload(cells)
    S, N = scene.spring_count, scene.mass_count
    eng = Engine(scene, integrator="verlet", precision=args.precision, layout=args.layout)
    info = eng.info()
    stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", 0))
    sub = args.substeps

    for _ in range(max(args.warmup, 3)):
        eng.step_async(sub)
    eng.synchronize()

    launches0 = eng.launch_count
    # L2 is flushed before every timed step (a write of twice its size on the
    # engine stream); per-step CUDA events bracket only the step itself
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(2 * max(l2, 64 << 20), dtype=torch.uint8, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        time.sleep(0.3)                  # sampler up before the timed region
        clk.start()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            starts[i].record(stream)
            eng.step_async(sub)
            ends[i].record(stream)
        ends[-1].synchronize()
        clk.stop()
    eng.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    del flush
    launches = eng.launch_count - launches0
    substeps = args.steps * sub
    value = S * substeps / (ms / 1e3)
    per_launch_s = ms / 1e3 / launches
    peak, peak_kind = peaks()
    algo = info["algorithmic_bytes_per_step"]
    achieved = algo / per_launch_s / 1e9

    # ---- e2e through the public API: host state in, positions out, every step
    x_host = eng.x.copy()
    v_host = eng.v.copy()
    xp_host = eng.x_prev.copy()
    e2e_steps = max(2, min(args.steps, 10))
    for _ in range(max(1, min(args.warmup, 2))):          # untimed: staging buffers, events
        eng.x = x_host
        eng.v = v_host
        eng.x_prev = xp_host
        eng.step(sub)
        _ = eng.x
    t0 = time.perf_counter()
    marks = []
    for _ in range(e2e_steps):
        eng.x = x_host
        eng.v = v_host
        eng.x_prev = xp_host
        eng.step(sub)
        out = eng.x
        marks.append(time.perf_counter())
    e2e_wall = time.perf_counter() - t0
    if os.environ.get("BENCH_E2E_DEBUG"):
        print("e2e ms per step:", [round(1e3 * (b - a), 2) for a, b in zip([t0] + marks[:-1], marks)],
              file=sys.stderr)
    _ = out
    vec = 16 if args.precision == "f32" else 32
    h2d = 3 * N * vec
    d2h = N * vec

    # configs[3] is a sweep "fp32 vs fp64 validation mode": the fp64 engine
    # (bitwise equal to the reference) on the same cube, same timing rules
    fp64 = None
    if args.precision == "f32" and not args.no_fp64:
        e64 = Engine(scene, integrator="verlet", precision="f64", layout=args.layout)
        st64 = torch.cuda.ExternalStream(e64.stream_ptr, device=torch.device("cuda", 0))
        for _ in range(3):
            e64.step_async(sub)
        e64.synchronize()
        k64 = max(3, min(args.steps, 10))
        flush = torch.empty(2 * max(l2, 64 << 20), dtype=torch.uint8, device="cuda")
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k64)]
        for a64, b64 in ev:                    # same rules: L2 flushed before every timed step
            with torch.cuda.stream(st64):
                flush.zero_()
            a64.record(st64)
            e64.step_async(sub)
            b64.record(st64)
        ev[-1][1].synchronize()
        e64.synchronize()
        ms64 = sum(a.elapsed_time(b) for a, b in ev)
        del flush
        inf64 = e64.info()
        fp64 = {"value": S * sub * k64 / (ms64 / 1e3), "unit": "spring-updates/s", "steps": k64,
                "ms_per_step": ms64 / k64, "dtype": "f64",
                "roofline_frac": inf64["algorithmic_bytes_per_step"] / (ms64 / 1e3 / (k64 * sub)) / 1e9 / peak,
                "note": "fp64 validation mode, bitwise equal to the reference's serial engine"}
        e64.close()

    cpu = None
    if not args.no_cpu:
        cv, csteps, cwall, cthreads = cpu_sample(scene)
        sv, ssteps, swall, _ = cpu_sample(scene, target_s=3.0, max_steps=20, mode="serial")
        cpu = {"value": cv, "unit": "spring-updates/s", "cores": cthreads, "kind": "port",
               "sample": f"{csteps} Verlet steps ({cwall:.1f} s) of the same {S}-spring cube, "
                         f"the reference bench's default parallel mode (Alg.1 atomic slots) restated in C/OpenMP",
               "host_threads": os.cpu_count(),
               "serial_1core": {"value": sv, "unit": "spring-updates/s", "cores": 1,
                                "sample": f"{ssteps} Verlet steps ({swall:.1f} s), the reference's serial mode"}}

    workload = f"cube_n{cells}_10M_springs_excited_verlet" if cells == 91 else f"cube_n{cells}_excited_verlet"
    layout_name = {1: "csr", 2: "ell", 3: "tile"}[info["layout"]]
    line = {
        "metric": "spring updates/sec (springs x steps / s)", "value": value,
        "unit": "spring-updates/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "f32" else "f64",
        "data": "synthetic",
        "config": {"workload": workload,
                   "cells": cells, "springs": S, "masses": N, "substeps_per_step": sub,
                   "integrator": "verlet", "precision": args.precision,
                   "layout": layout_name,
                   "tile_halo_ratio": round(info["tile_halo_ratio"], 3),
                   "tile_foreign_frac": round(info["tile_foreign_frac"], 3),
                   "records_bytes_per_step": info["tile_blob_bytes"],
                   "device_bytes": info["device_bytes"],
                   "l2": "L2 flushed before every timed step (%d MB write); per-step CUDA events exclude "
                         "the flush; per-substep working set ~%.0f MB" % (2 * l2 >> 20,
                                                                           (info["tile_blob_bytes"] + 5 * 16 * N) / 1e6),
                   "parallelism": "single-gpu"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": profiled_traffic(workload, args.precision, layout_name),
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": algo,
                     "avg_launch_us": per_launch_s * 1e6,
                     "note": ("compact tile records: %d record bytes/substep (%.1f B/spring) stream instead of "
                              "the 16 B/spring of the SURVEY 8d model, so measured DRAM traffic is below the "
                              "algorithmic bytes; see DESIGN.md 4" % (info["tile_blob_bytes"],
                                                                      info["tile_blob_bytes"] / S))
                             if info.get("tile_kernel") == 2 else None},
        "fp64_validation": fp64,
        "cpu_baseline": cpu,
        "e2e": {"value": S * sub * e2e_steps / e2e_wall, "unit": "spring-updates/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cells", type=int, default=0)
    ap.add_argument("--substeps", type=int, default=SUBSTEPS)
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--layout", default="auto", choices=["auto", "csr", "ell"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 validation-mode measurement")
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
        from paper_2207_09334_b200 import sharded
        sharded.bench_main(args)
        return
    if args.gpus > 1:
        # not launched under torchrun: launch one process per GPU ourselves
        import sys as _sys
        cmd = [_sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", "--master-port=29611",
               os.path.abspath(__file__)] + _sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    run_single(args)


if __name__ == "__main__":
    main()
