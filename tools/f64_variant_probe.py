"""fp64 compact-tile kernel instantiations (UNROLL, MINB; SS_F64_VARIANT) against
cube size, µs per substep in graph replays.  CELLS, VARIANTS, INTEG (dev tool)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2207_09334_b200 import Engine, lattice as L
cells_list = [int(c) for c in os.environ.get("CELLS", "20,30,42,60").split(",")]
for cells in cells_list:
    sc = L.excite(L.block_scene(cells), seed=11)
    row = {"cells": cells}
    for v in os.environ.get("VARIANTS", "0,1,2,3,5").split(","):
        if v == "default":
            os.environ.pop("SS_F64_VARIANT", None)
        else:
            os.environ["SS_F64_VARIANT"] = v
        e = Engine(sc, integrator=os.environ.get("INTEG", "verlet"), precision="f64")
        st = torch.cuda.ExternalStream(e.stream_ptr)
        for _ in range(6):
            e.step_async(100)
        e.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(4):
            e.step_async(100)
        b.record(st); b.synchronize(); e.synchronize()
        row["v" + v] = round(a.elapsed_time(b) * 1e3 / 400, 2)
        row["tiles"] = e.info()["tile_count"]
        e.close()
    print(json.dumps(row), flush=True)
