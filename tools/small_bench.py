"""Per-step time of small scenes: CTA-resident kernel (default) vs one launch
per step (SS_RESIDENT=0), and whether both give the same bits (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_09334_b200 import Engine, crawler_scene, lattice as L, replicate

scenes = {"crawler": crawler_scene, "crawler_x12": lambda: replicate(crawler_scene(), 12), "beam40": lambda: L.beam_lattice(length=4.0),
          "cube9": lambda: L.excite(L.block_scene(9)), "crawler_x64": lambda: replicate(crawler_scene(), 64)}
if "SS_RESIDENT" not in os.environ:
    os.environ["SS_RESIDENT"] = "16"          # (the default cap; "1" would limit residency to one-tile scenes)
for name, mk in scenes.items():
    for prec in ("f64", "f32"):
        row = {"scene": name, "prec": prec}
        for res in (os.environ.get("RES_ON", "16"), "0"):
            os.environ["SS_RESIDENT"] = res
            e = Engine(mk(), integrator="verlet", precision=prec)
            row["slots"] = e.info()["n_masses"]
            e.step(100)
            n = 20000
            t0 = time.perf_counter(); e.step(n); dt = time.perf_counter() - t0
            row["us_per_step_resident" + ("0" if res == "0" else "1")] = round(1e6 * dt / n, 3)
            row["x_" + ("0" if res == "0" else "1")] = e.x.copy()
            e.close()
        row["same"] = bool(row.pop("x_0").tobytes() == row.pop("x_1").tobytes())
        print(json.dumps(row), flush=True)
