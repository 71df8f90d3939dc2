"""Host enqueue time vs device time per substep (dev tool): is a mid-size
scene bound by the host's launch rate?"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
for n in (20, 30, 42, 60):
    sc = L.excite(L.block_scene(n), seed=11)
    for prec in ("f64", "f32"):
        e = Engine(sc, integrator="verlet", precision=prec)
        e.step_async(20); e.synchronize()
        st = torch.cuda.ExternalStream(e.stream_ptr)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        k = 400
        a.record(st)
        t0 = time.perf_counter(); e.step_async(k); host = time.perf_counter() - t0
        b.record(st); b.synchronize(); e.synchronize()
        print(json.dumps({"cells": n, "prec": prec, "tiles": e.info()["tile_count"],
                          "host_us_per_step": round(host * 1e6 / k, 2),
                          "device_us_per_step": round(a.elapsed_time(b) * 1e3 / k, 2)}), flush=True)
        e.close()
