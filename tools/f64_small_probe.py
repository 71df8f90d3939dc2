"""fp64 small scenes: per-step time of each stepping mode (launch per step,
resident CTA with 4-8 lanes per mass, resident with one lane per mass, and
the same as clusters for multi-tile scenes) and whether all give the same
bits (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, crawler_scene, lattice as L, replicate
scenes = {"crawler": crawler_scene, "block3": lambda: L.excite(L.block_scene(3), seed=11),
          "crawler_x12": lambda: replicate(crawler_scene(), 12), "beam40": lambda: L.beam_lattice(length=4.0),
          "cube9": lambda: L.excite(L.block_scene(9), seed=11), "crawler_x64": lambda: replicate(crawler_scene(), 64)}
modes = {"launch": {"SS_RESIDENT": "0"}, "lanes": {}, "lanes1": {"SS_RESIDENT_G": "1"},
         "cluster": {"SS_RESIDENT_F64": "16"}, "cluster1": {"SS_RESIDENT_F64": "16", "SS_RESIDENT_G": "1"}}
for name, mk in scenes.items():
    row = {"scene": name}
    ref = None
    for mode, env in modes.items():
        for k in ("SS_RESIDENT", "SS_RESIDENT_G", "SS_RESIDENT_F64"):
            os.environ.pop(k, None)
        os.environ.update(env)
        e = Engine(mk(), integrator="verlet", precision="f64")
        e.step(100)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        n = 20000
        a.record(st); e.step_async(n); b.record(st); b.synchronize(); e.synchronize()
        row[mode] = round(a.elapsed_time(b) * 1e3 / n, 3)
        x = e.x.tobytes() + e.v.tobytes()
        ref = ref or x
        row[mode + "_same"] = x == ref
        e.close()
    print(json.dumps(row), flush=True)
