"""Per-step time of each integrator on the 10M cube, fp32 and fp64 (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
sc = L.excite(L.block_scene(int(os.environ.get("CELLS", "91"))), seed=11)
for prec in ("f32", "f64"):
    for integ in ("verlet", "euler", "rk4"):
        e = Engine(sc, integrator=integ, precision=prec)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        e.step_async(5); e.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); e.step_async(50); b.record(st); b.synchronize(); e.synchronize()
        us = a.elapsed_time(b) * 1e3 / 50
        print(prec, integ, round(us, 1), "us/step", e.info()["tile_kernel"], flush=True)
        e.close()
