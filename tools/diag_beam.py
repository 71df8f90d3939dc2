"""fp32 vs fp64 on the loaded cantilever (dev tool): forces at a perturbed
state and positions after a damped relaxation, for the lean kernel and
SS_KERNEL=step1."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_09334_b200 import Engine, lattice as L

g = json.load(open("tests/golden/observables.json"))["beam_20x4x4"]
def run(prec, kernel, steps):
    os.environ["SS_KERNEL"] = kernel
    sc = L.beam_lattice(length=g["length"])
    e = Engine(sc, integrator="verlet", precision=prec)
    per = g["tip_load"] / len(g["tip_ids"])
    for i in g["tip_ids"]:
        e.set_external_force(i, (0.0, -per, 0.0))
    e.set_damping(g["damping"])
    rng = np.random.default_rng(0)
    xp = sc.x + rng.normal(0, 1e-6, sc.x.shape)
    f = e.forces(xp, np.zeros_like(xp), 0.0)
    e.step(steps)
    return f, e.x.copy(), e.info()
for steps in (100, 2000, 20000):
    f64, x64, _ = run("f64", "lean", steps)
    for k in ("lean", "step1"):
        f32, x32, inf = run("f32", k, steps)
        print(json.dumps({"steps": steps, "kernel": k, "tile_kernel": inf["tile_kernel"],
                          "force_rel_err": float(np.abs(f32 - f64).max() / np.abs(f64).max()),
                          "tip_dy64": float(x64[g["probe"], 1] - 0.2), "tip_dy32": float(x32[g["probe"], 1] - 0.2),
                          "max_dx": float(np.abs(x32 - x64).max())}), flush=True)
