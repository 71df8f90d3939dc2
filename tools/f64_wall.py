"""fp64 Engine.step(100) wall time on the 10M cube, at rest and excited (dev tool)."""
import os, time, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
sc = L.block_scene(91)
for exc in (False, True):
    s2 = L.excite(L.block_scene(91), seed=11) if exc else sc
    e = Engine(s2, integrator="verlet", precision="f64")
    e.step(10)
    for _ in range(4):
        t0 = time.perf_counter(); e.step(100); print("excited" if exc else "rest", round((time.perf_counter() - t0) * 1e3, 2), "ms", flush=True)
    e.close()
