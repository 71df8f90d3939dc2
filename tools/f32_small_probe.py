"""fp32 small scenes: resident lanes per mass (default 4-8 vs 1) and launches (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, crawler_scene, lattice as L, replicate
scenes = {"crawler": crawler_scene, "block3": lambda: L.excite(L.block_scene(3), seed=11),
          "crawler_x12": lambda: replicate(crawler_scene(), 12), "beam40": lambda: L.beam_lattice(length=4.0),
          "cube9": lambda: L.excite(L.block_scene(9), seed=11), "crawler_x64": lambda: replicate(crawler_scene(), 64)}
modes = {"launch": {"SS_RESIDENT": "0"}, "lanes": {}, "lanes1": {"SS_RESIDENT_G": "1"}}
for name, mk in scenes.items():
    row = {"scene": name}
    for mode, env in modes.items():
        for k in ("SS_RESIDENT", "SS_RESIDENT_G"):
            os.environ.pop(k, None)
        os.environ.update(env)
        e = Engine(mk(), integrator="verlet", precision="f32")
        e.step(100)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        n = 20000
        a.record(st); e.step_async(n); b.record(st); b.synchronize(); e.synchronize()
        row[mode] = round(a.elapsed_time(b) * 1e3 / n, 3)
        e.close()
    print(json.dumps(row), flush=True)
