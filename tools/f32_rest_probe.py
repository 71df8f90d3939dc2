"""fp32 per-substep time on the 10M cube at rest vs excited (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
for name, sc in (("rest", L.block_scene(91)), ("excited", L.excite(L.block_scene(91), seed=11))):
    e = Engine(sc, integrator="verlet", precision="f32")
    st = torch.cuda.ExternalStream(e.stream_ptr)
    e.step_async(20); e.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st); e.step_async(200); b.record(st); b.synchronize(); e.synchronize()
    print(name, round(a.elapsed_time(b) * 1e3 / 200, 2), "us/substep", flush=True)
    e.close()
