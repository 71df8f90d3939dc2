"""fp32 vs fp64 crawler ensemble travel statistics (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_09334_b200 import Engine, crawler_scene, per_instance, replicate

def ens(prec, copies, seed, jitter=1e-9, seconds=8.0, kernel=None):
    if kernel: os.environ["SS_KERNEL"] = kernel
    else: os.environ.pop("SS_KERNEL", None)
    sc = crawler_scene()
    b = replicate(sc, copies, jitter=jitter, seed=seed)
    e = Engine(b, integrator="verlet", precision=prec)
    e.set_damping(2e-4)
    x0 = per_instance(e.x, copies)[:, :, 0].mean(1)
    out = []
    for s in range(int(seconds)):
        e.step(int(round(1.0 / sc.dt)))
        out.append(float((per_instance(e.x, copies)[:, :, 0].mean(1) - x0).mean()))
    tr = per_instance(e.x, copies)[:, :, 0].mean(1) - x0
    return {"prec": prec, "kernel": kernel, "seed": seed, "mean": float(tr.mean()), "std": float(tr.std()), "per_second": out}

for seed in (5, 6):
    for prec, k in (("f64", None), ("f32", None), ("f32", "step1")):
        print(json.dumps(ens(prec, 64, seed, kernel=k)), flush=True)
