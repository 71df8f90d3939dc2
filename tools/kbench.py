"""Per-substep time of the fp32 tile kernel variants on the 10M cube (dev tool).

    VARIANTS="once:3,once:2,step2,once+SS_DEBUG=1" CELLS=91 python tools/kbench.py

Each variant is SS_KERNEL[:SS_ONCE_MINB][+ENV=VAL...]; the engine reads
these variables at creation.
Also prints max |x - x_first| against the first variant after the timed run
(same inputs, fp32: the variants differ only in summation order)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2207_09334_b200 import Engine, lattice as L

cells = int(os.environ.get("CELLS", "91"))
integ = os.environ.get("INTEG", "verlet")
n_steps = int(os.environ.get("NSTEPS", "200"))
scene = L.excite(L.block_scene(cells), seed=11)
first = None
for var in os.environ.get("VARIANTS", "once:3,once:2,step2").split(","):
    head, *extra = var.split("+")
    name, _, minb = head.partition(":")
    for k in ("SS_DEBUG", "SS_ONCE_MINB", "SS_LEAN_MINB", "SS_TILE_DICT", "SS_TILE_SORT", "SS_PROF", "SS_PDL", "SS_KERNEL"):
        os.environ.pop(k, None)
    os.environ["SS_KERNEL"] = name
    if minb:
        os.environ["SS_ONCE_MINB"] = minb
    for kv in extra:
        k, _, v = kv.partition("=")
        os.environ[k] = v
    eng = Engine(scene, integrator=integ, precision="f32", layout="tile")
    info = eng.info()
    st = torch.cuda.ExternalStream(eng.stream_ptr)
    eng.step_async(20)
    eng.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    eng.step_async(n_steps)
    b.record(st)
    b.synchronize()
    eng.synchronize()
    us = a.elapsed_time(b) * 1e3 / n_steps
    x = eng.x.copy()
    if first is None:
        first = x
    dev = float(np.abs(x - first).max() / np.abs(first).max())
    r = dict(variant=var, integ=integ, cells=cells, us_per_substep=round(us, 2),
             springs_per_s=scene.spring_count / (us * 1e-6),
             algo_GBs=round(info["algorithmic_bytes_per_step"] / (us * 1e-6) / 1e9, 1),
             smem=info["smem_per_block"], rel_dev_vs_first=dev, launches=eng.launch_count)
    if os.environ.get("SS_PROF"):
        import ctypes
        from paper_2207_09334_b200 import _lib
        buf = (ctypes.c_ulonglong * 16)()
        fn = _lib.lib().ss_debug_prof
        fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        fn(eng._h, buf)
        launches = eng.launch_count
        names = ["p_wait_free", "p_issue_own", "p_wait_hdr", "p_issue_halo", "c_wait_states", "c_convert",
                 "c_wait_records", "c_owner", "c_foreign", "c_barrier", "c_refs", "c_epilogue"]
        # per launch, per CTA (148), consumers per group (2): microseconds at 1.965 GHz
        prof = {nm: round(buf[i] / launches / 148 / (2 if nm.startswith("c_") else 1) / 1965.0, 2)
                for i, nm in enumerate(names)}
        r["prof_us_per_cta"] = prof
    print(json.dumps(r), flush=True)
    eng.close()
