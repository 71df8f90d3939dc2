"""Small scenes on the CTA/cluster-resident kernel: µs per step for G = 1, 2,
4, 8 lanes per mass (SS_RESIDENT_G), both precisions, and whether every G
gives the fp64 bits of G = 1 (dev tool)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_09334_b200 import Engine, crawler_scene, lattice as L, replicate  # noqa: E402

scenes = {"crawler": crawler_scene, "crawler_x12": lambda: replicate(crawler_scene(), 12),
          "beam40": lambda: L.beam_lattice(length=4.0), "cube9": lambda: L.excite(L.block_scene(9), seed=11),
          "crawler_x64": lambda: replicate(crawler_scene(), 64)}
for prec in ("f64", "f32"):
    for name, mk in scenes.items():
        row = {"scene": name, "prec": prec}
        ref = None
        for g in ("1", "2", "4", "8"):
            os.environ["SS_RESIDENT_G"] = g
            e = Engine(mk(), integrator="verlet", precision=prec)
            e.step(100)
            st = torch.cuda.ExternalStream(e.stream_ptr)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            n = 20000
            a.record(st)
            e.step_async(n)
            b.record(st)
            b.synchronize()
            e.synchronize()
            row["G" + g] = round(a.elapsed_time(b) * 1e3 / n, 3)
            x = e.x.tobytes() + e.v.tobytes()
            ref = ref or x
            if prec == "f64":
                row["G" + g + "_same"] = x == ref
            e.close()
        print(json.dumps(row), flush=True)
