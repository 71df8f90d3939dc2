"""Extended randomised fp64 parity sweep (dev tool): many seeded random scenes
(sizes from one tile to a few hundred, lattice or general graphs, long-range
springs), every integrator, random batch plans and resident/launch/format
switches, bitwise against the oracle.  Prints mismatches; exit code 1 if any."""
import os, sys, json, random
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as orc
from paper_2207_09334_b200 import Engine
from paper_2207_09334_b200.model import scene_arrays
from test_gpu_fuzz import random_scene

n_cases = int(os.environ.get("CASES", "120"))
bad = 0
rnd = random.Random(7)
for case in range(n_cases):
    seed = 100 + case
    n = rnd.choice([20, 60, 200, 500, 1200, 3000, 8000, 20000])
    lattice = rnd.random() < 0.5
    long_range = rnd.choice([0.0, 0.0, 0.0, 0.02])
    integ = rnd.choice(["verlet", "verlet", "euler", "rk4"])
    env = rnd.choice([{}, {"SS_RESIDENT": "0"}, {"SS_TILE_DICT": "0"}, {"SS_TILE_DICT": "explicit"}, {"SS_PDL": "0"}])
    for k in ("SS_RESIDENT", "SS_TILE_DICT", "SS_PDL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    sc = random_scene(seed, n, long_range=long_range, lattice=lattice)
    try:
        eng = Engine(sc, integrator=integ, precision="f64")
    except Exception as exc:
        print(json.dumps({"case": case, "error": repr(exc)})); bad += 1; continue
    ref = orc.OracleEngine(scene_arrays(sc), integrator=integ)
    plan = [rnd.choice([1, 3, 17, 64]) for _ in range(rnd.randint(1, 4))]
    ok = True
    for c in plan:
        try:
            eng.step(c)
        except Exception as exc:
            ok = False
            print(json.dumps({"case": case, "step_error": repr(exc)}))
            break
        ref.step(c)
        if eng.x.tobytes() != ref.x.tobytes() or eng.v.tobytes() != ref.v.tobytes():
            ok = False
            print(json.dumps({"case": case, "seed": seed, "n": sc.mass_count, "lattice": lattice, "lr": long_range,
                              "integ": integ, "env": env, "plan": plan, "tile_kernel": eng.info()["tile_kernel"],
                              "maxdiff": float(np.abs(eng.x - ref.x).max())}), flush=True)
            break
    if ok and eng.degenerate_springs != ref.degenerate_springs:
        ok = False
        print(json.dumps({"case": case, "degenerate": [eng.degenerate_springs, ref.degenerate_springs]}))
    bad += 0 if ok else 1
    eng.close()
print(json.dumps({"cases": n_cases, "mismatches": bad}))
sys.exit(1 if bad else 0)
