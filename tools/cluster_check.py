"""Small multi-tile scenes: per-step time through Engine.step (chunked) and as
one asynchronous batch (CUDA events), launches per batch (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, crawler_scene, lattice as L, replicate
scenes = {"beam40": lambda: L.beam_lattice(length=4.0), "cube9": lambda: L.excite(L.block_scene(9), seed=11),
          "crawler_x64": lambda: replicate(crawler_scene(), 64), "crawler": crawler_scene}
for name, mk in scenes.items():
    for prec in ("f32", "f64"):
        for res in ("16", "0"):
            os.environ["SS_RESIDENT"] = res
            e = Engine(mk(), integrator="verlet", precision=prec)
            e.step(100)
            n = 20000
            l0 = e.launch_count
            t0 = time.perf_counter(); e.step(n); wall = time.perf_counter() - t0
            l1 = e.launch_count
            st = torch.cuda.ExternalStream(e.stream_ptr)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st); e.step_async(n); b.record(st); b.synchronize(); e.synchronize()
            ev = a.elapsed_time(b) * 1e3 / n
            print(json.dumps({"scene": name, "prec": prec, "resident": res, "tiles": e.info()["tile_count"],
                              "us_step_api": round(1e6 * wall / n, 3), "us_step_async_events": round(ev, 3),
                              "launches_api": l1 - l0, "launches_async": e.launch_count - l1}), flush=True)
            e.close()
