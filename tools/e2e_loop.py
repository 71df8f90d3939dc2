import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
if os.environ.get("WITH_TORCH"):
    import torch
    torch.zeros(1, device="cuda")
from paper_2207_09334_b200 import Engine, lattice as L
sc = L.excite(L.block_scene(91), seed=11)
eng = Engine(sc, integrator="verlet", precision="f32")
eng.step(100)
x, v, xp = eng.x.copy(), eng.v.copy(), eng.x_prev.copy()
for rep in range(3):
    ts = []
    for _ in range(6):
        a = time.perf_counter()
        eng.x = x; eng.v = v; eng.x_prev = xp
        b = time.perf_counter(); eng.step(100); c = time.perf_counter()
        out = eng.x
        d = time.perf_counter()
        ts.append((round((b-a)*1e3,2), round((c-b)*1e3,2), round((d-c)*1e3,2)))
    print(ts, flush=True)
