"""Two x-slab shards of the 10M cube on one GPU, stepped in lockstep: the fused
peer-memory exchange vs plane-copy kernels vs one unsharded engine (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
from paper_2207_09334_b200.sharded import ShardGroup, excited_velocities

cells = int(os.environ.get("CELLS", "91"))
full = L.excite(L.block_scene(cells), seed=11)
v = excited_velocities(full.mass_count)
one = Engine(full, precision="f32")
one.step(10)
t0 = time.perf_counter(); one.step(200); t1 = time.perf_counter()
print("single engine", round((t1 - t0) * 1e6 / 200, 2), "us/substep", flush=True)
for transport in ("copy", "p2p"):
    grp = ShardGroup(cells, 2, precision="f32", v_global=v, transport=transport)
    grp.step(10)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); grp.step(200); t1 = time.perf_counter()
    print("2 shards,", transport, round((t1 - t0) * 1e6 / 200, 2), "us/substep (both shards, one stream)", flush=True)
