"""fp32 vs fp64 single crawler, short horizons (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_09334_b200 import Engine, crawler_scene

def run(prec, layout, steps_list, damping=2e-4, **mods):
    sc = crawler_scene()
    for k, v in mods.items():
        setattr(sc, k, v)
    e = Engine(sc, integrator="verlet", precision=prec, layout=layout)
    e.set_damping(damping)
    out, done = [], 0
    for s in steps_list:
        e.step(s - done); done = s
        out.append(e.x.copy())
    return out
steps = [200, 2000, 20000]
ref = run("f64", "auto", steps)
for prec, lay in (("f32", "auto"), ("f32", "csr")):
    got = run(prec, lay, steps)
    print(json.dumps({"prec": prec, "layout": lay, "rows": [
        {"steps": s, "max_dx": float(np.abs(g - r).max()), "travel_ref": float(r[:, 0].mean() - crawler_scene().x[:, 0].mean()),
         "travel": float(g[:, 0].mean() - crawler_scene().x[:, 0].mean())} for s, g, r in zip(steps, got, ref)]}), flush=True)
# without actuation / without friction
sc = crawler_scene()
for label, kw in (("no_friction", {}),):
    pass
