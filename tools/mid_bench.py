"""fp32 per-substep time on mid-size cubes, one vs two lanes per mass (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L

for cells in (20, 30, 42, 60, 91):
    sc = L.excite(L.block_scene(cells), seed=11)
    row = {"cells": cells, "springs": sc.spring_count}
    for lanes in ("1", "2"):
        os.environ["SS_LEAN_LANES"] = lanes
        e = Engine(sc, integrator="verlet", precision="f32")
        st = torch.cuda.ExternalStream(e.stream_ptr)
        e.step_async(20); e.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); e.step_async(200); b.record(st); b.synchronize(); e.synchronize()
        us = a.elapsed_time(b) * 1e3 / 200
        row[f"us_lanes{lanes}"] = round(us, 2)
        row[f"x{lanes}"] = e.x.copy()
        e.close()
    d = float(abs(row.pop("x1") - row.pop("x2")).max())
    row["max_dx"] = d
    print(json.dumps(row), flush=True)
