"""Randomised sharding sweep (dev tool): random voxel boxes (random extents,
per-spring stiffness / rest-length jitter so some scenes take the inline
record format, fixed masses, f_ext, gravity, damping, a floor with friction,
a sinusoid actuation group), split into 2-5 x-slabs, every integrator, the
plane-copy and fused peer-memory transports, random batch plans: the
assembled fp64 state must equal one engine's bit for bit (PREC=f32: within
1e-4 of the displacement).  Prints mismatches; exit code 1 if any.
CASES=200 by default."""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2207_09334_b200 import DivergenceError, Engine, lattice as L  # noqa: E402
from paper_2207_09334_b200.model import ActuationGroup, ContactPlane  # noqa: E402
from paper_2207_09334_b200.sharded import ShardGroup  # noqa: E402


def random_box(rnd: random.Random, seed: int):
    nx, ny, nz = rnd.randint(4, 14), rnd.randint(1, 5), rnd.randint(1, 5)
    s = L.voxel_box((0.0, 0.0, 0.0), (0.1 * nx, 0.1 * ny, 0.1 * nz), 0.1)
    rng = np.random.default_rng(seed)
    n, m = s.x.shape[0], s.si.shape[0]
    s.v = rng.normal(0.0, 0.05, (n, 3))
    if rnd.random() < 0.5:                                  # per-spring records: the inline format
        s.k = s.k * (1.0 + 1e-3 * rng.standard_normal(m))
        s.l0 = s.l0 * (1.0 + 1e-3 * rng.standard_normal(m))
    if rnd.random() < 0.5:
        s.fixed = rng.random(n) < 0.05
    if rnd.random() < 0.5:
        s.f_ext = rng.normal(0.0, 0.01, (n, 3))
    s.gravity = (0.0, 0.0, -9.81) if rnd.random() < 0.5 else (0.0, 0.0, 0.0)
    s.damping = rnd.choice([0.0, 1e-4, 1e-3])
    if rnd.random() < 0.5:
        s.x[:, 2] -= 0.02                                   # the bottom layer starts in contact
        s.planes = [ContactPlane((0.0, 0.0, 1.0), 0.0, 1e4, rnd.choice([0.0, 0.6]))]
    if rnd.random() < 0.4:
        s.groups = {"m": ActuationGroup("m", mode="sinusoid", amplitude=0.05, frequency=3.0, phase=0.2)}
        s.group = np.where(rng.random(m) < 0.3, 0, -1).astype(np.int32)
    return s


def main():
    n_cases = int(os.environ.get("CASES", "200"))
    rnd = random.Random(11)
    bad = 0
    stats = {"inline": 0, "diverged": 0, "rk4": 0, "p2p": 0}
    for case in range(n_cases):
        scene = random_box(rnd, 1000 + case)
        integ = rnd.choice(["verlet", "euler", "rk4"])
        transport = rnd.choice(["copy", "p2p"])
        nx = len(np.unique(scene.x[:, 0]))
        shards = rnd.randint(2, min(5, nx))
        plan = [rnd.choice([1, 3, 17, 40]) for _ in range(rnd.randint(1, 3))]
        prec = "f32" if os.environ.get("PREC") == "f32" else "f64"
        one = Engine(scene, integrator=integ, precision=prec)
        grp = ShardGroup.from_scene(scene, shards, precision=prec, transport=transport, integrator=integ)
        stats["inline"] += one.info()["tile_kernel"] in (5, 6)
        stats["rk4"] += integ == "rk4"
        stats["p2p"] += transport == "p2p"
        ok = True
        for count in plan:
            err = []
            for target in (one, grp):
                try:
                    target.step(count)
                    err.append(None)
                except DivergenceError as e:
                    err.append((e.mass_id, e.step))
            ok = ok and err[0] == err[1]
            x = np.concatenate([e.x[s.owned] for e, s in zip(grp.engines, grp.slabs)])
            v = np.concatenate([e.v[s.owned] for e, s in zip(grp.engines, grp.slabs)])
            if prec == "f64":
                ok = ok and np.array_equal(x, one.x, equal_nan=True) and np.array_equal(v, one.v, equal_nan=True)
            elif err[0] is None:                            # fp32: within rounding of the displacement
                disp = max(float(np.abs(one.x - scene.x).max()), 1e-12)
                ok = ok and float(np.abs(x - one.x).max()) <= 1e-4 * disp
            if err[0] is not None:
                stats["diverged"] += 1
                break
        if not ok:
            bad += 1
            print(json.dumps({"case": case, "integrator": integ, "transport": transport, "shards": shards,
                              "plan": plan, "masses": int(scene.x.shape[0])}), flush=True)
        one.close()
        for e in grp.engines:
            e.close()
    print(json.dumps({"cases": n_cases, "mismatches": bad, **stats}), flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
