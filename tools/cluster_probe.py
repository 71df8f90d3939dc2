"""fp32 per-step time of 2-16-tile scenes: cluster-resident (SS_RESIDENT=16) vs launches (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_09334_b200 import Engine, lattice as L
for cells in (9, 11, 12, 13, 14):
    sc = L.excite(L.block_scene(cells), seed=11)
    row = {"cells": cells, "masses": sc.mass_count}
    for res in ("16", "0"):
        os.environ["SS_RESIDENT"] = res
        e = Engine(sc, integrator="verlet", precision="f32")
        row["tiles"] = e.info()["tile_count"]
        e.step(100)
        t0 = time.perf_counter(); e.step(5000); dt = time.perf_counter() - t0
        row["us_" + res] = round(1e6 * dt / 5000, 2)
        e.close()
    print(json.dumps(row), flush=True)
