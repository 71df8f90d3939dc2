"""µs per substep of excited cubes (graph replays) under alternative
environment switches, e.g.  PREC=f32 CELLS=42,60 AB="SS_LEAN_LANES=1;SS_LEAN_LANES=2;"
(an empty entry = the defaults); MODE=single times one 400-substep batch
(launches) instead of repeated 100-substep batches (graph replays) -- dev tool."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_09334_b200 import Engine, lattice as L  # noqa: E402

prec = os.environ.get("PREC", "f32")
integ = os.environ.get("INTEG", "verlet")
variants = os.environ.get("AB", ";").split(";")
for cells in [int(c) for c in os.environ.get("CELLS", "42,60").split(",")]:
    sc = L.excite(L.block_scene(cells), seed=11)
    row = {"cells": cells, "prec": prec}
    for var in variants:
        env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
        for k, v in env.items():
            os.environ[k] = v
        e = Engine(sc, integrator=integ, precision=prec)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        single = os.environ.get("MODE") == "single"         # one big batch: launches, no graph replays
        for _ in range(1 if single else 6):
            e.step_async(100)
        e.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        if single:
            e.step_async(400)
        else:
            for _ in range(4):
                e.step_async(100)
        b.record(st)
        b.synchronize()
        e.synchronize()
        row[var or "default"] = round(a.elapsed_time(b) * 1e3 / 400, 2)
        row["tiles"] = e.info()["tile_count"]
        e.close()
        for k in env:
            os.environ.pop(k, None)
    print(json.dumps(row), flush=True)
