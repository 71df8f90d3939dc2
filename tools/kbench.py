"""Per-substep time of the fp32 tile kernel variants on the 10M cube (dev tool).

    VARIANTS="lean,lean+SS_PDL=0,step1,lean+SS_TILE_DICT=0,lean+SS_DEBUG=1" CELLS=91 python tools/kbench.py

Each variant is SS_KERNEL[+ENV=VAL...] (SS_KERNEL: lean = tile_f32.cuh
tile_lean_kernel, step1 = kernels.cuh step_kernel); the engine reads these
variables at creation.
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
for var in os.environ.get("VARIANTS", "lean,step1").split(","):
    head, *extra = var.split("+")
    name, _, minb = head.partition(":")
    for k in ("SS_DEBUG", "SS_ONCE_MINB", "SS_LEAN_MINB", "SS_TILE_DICT", "SS_TILE_SORT", "SS_PDL", "SS_KERNEL"):
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
    print(json.dumps(r), flush=True)
    eng.close()
