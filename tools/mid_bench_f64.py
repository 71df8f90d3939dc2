"""fp64 and fp32 per-substep time on cubes of 1e5..1e7 springs (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L

for cells in (20, 30, 42, 60, 91):
    sc = L.excite(L.block_scene(cells), seed=11)
    row = {"cells": cells, "springs": sc.spring_count}
    for prec in ("f64", "f32"):
        e = Engine(sc, integrator="verlet", precision=prec)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        e.step_async(20); e.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); e.step_async(200); b.record(st); b.synchronize(); e.synchronize()
        us = a.elapsed_time(b) * 1e3 / 200
        row[prec + "_us"] = round(us, 2)
        row[prec + "_rate"] = float("%.3g" % (sc.spring_count / us * 1e6))
        row["tiles"] = e.info()["tile_count"]
        e.close()
    print(json.dumps(row), flush=True)
