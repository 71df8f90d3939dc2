"""Host enqueue time vs device time per step for small multi-tile scenes (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L, crawler_scene, replicate
for name, sc in (("beam40", L.beam_lattice(length=4.0)), ("cube9", L.excite(L.block_scene(9), seed=11)),
                 ("crawler_x64", replicate(crawler_scene(), 64))):
    for prec in ("f32", "f64"):
        e = Engine(sc, integrator="verlet", precision=prec)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        e.step_async(100); e.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        n = 2000
        a.record(st)
        t0 = time.perf_counter(); e.step_async(n); t1 = time.perf_counter()
        b.record(st); b.synchronize(); e.synchronize()
        print(name, prec, "host enqueue", round((t1 - t0) * 1e6 / n, 2), "us/step; device",
              round(a.elapsed_time(b) * 1e3 / n, 2), "us/step", flush=True)
        e.close()
