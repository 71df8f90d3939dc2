"""Two x-slab shards of the 10M cube on one GPU, stepped in lockstep: the fused
peer-memory exchange vs plane-copy kernels vs one unsharded engine (dev tool).
PREC=f32|f64, INTEG=verlet|rk4, CELLS=91."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
from paper_2207_09334_b200.sharded import ShardGroup, excited_velocities

cells = int(os.environ.get("CELLS", "91"))
prec = os.environ.get("PREC", "f32")
integ = os.environ.get("INTEG", "verlet")
steps = 200 if integ != "rk4" else 50
full = L.excite(L.block_scene(cells), seed=11)
v = excited_velocities(full.mass_count)
one = Engine(full, precision=prec, integrator=integ)
one.step(10)
t0 = time.perf_counter(); one.step(steps); t1 = time.perf_counter()
print(prec, integ, "single engine", round((t1 - t0) * 1e6 / steps, 2), "us/step", flush=True)
one.close()
for transport in ("copy", "p2p"):
    grp = ShardGroup(cells, 2, precision=prec, v_global=v, transport=transport, integrator=integ)
    grp.step(10)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); grp.step(steps); t1 = time.perf_counter()
    print(prec, integ, "2 shards,", transport, round((t1 - t0) * 1e6 / steps, 2), "us/step (both shards, one stream)",
          flush=True)
    for e in grp.engines:
        e.close()
