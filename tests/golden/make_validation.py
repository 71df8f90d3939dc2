"""Golden outputs of the reference's validate_scene (dev container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_validation.py

Builds invalid and valid scenes through the reference's raw object model
(model.py:21-204: Mass / Spring / ActuationGroup / ContactPlane / Material
lists, bypassing the add_* guards), runs ``springsim.model.validate_scene``
(model.py:231-327) and stores each scene description with the exact list of
(code, where, message) it returns, in order, as tests/golden/validation.json.
"""

from __future__ import annotations

import json
import math
import os

import numpy as np

from springsim.model import (ActuationGroup, ContactPlane, Mass, Material, Scene, Spring,  # noqa: E402
                             validate_scene)

HERE = os.path.dirname(os.path.abspath(__file__))
NAN, INF = float("nan"), float("inf")


def describe(scene) -> dict:
    return {
        "masses": [[m.id, m.m, list(m.x), list(m.v), list(m.f_ext), m.fixed] for m in scene.masses],
        "springs": [[s.id, s.i, s.j, s.k, s.l0, s.group] for s in scene.springs],
        "groups": [[key, g.label, g.mode, g.amplitude, g.frequency, g.phase] for key, g in scene.groups.items()],
        "planes": [[list(p.normal), p.offset, p.penalty, p.friction] for p in scene.planes],
        "materials": [[m.name, m.k0, m.l_ref, m.density, m.total_mass, m.mass_per_node] for m in scene.materials],
        "gravity": list(scene.gravity), "dt": scene.dt, "damping": scene.damping,
    }


def oscillator():
    s = Scene(gravity=(0.0, -9.81, 0.0))
    a = s.add_mass((0.0, 1.0, 0.0), fixed=True)
    b = s.add_mass((0.0, 0.8, 0.0))
    s.add_spring(a, b, k=100.0)
    return s


def cases():
    out = {"valid_oscillator": oscillator()}
    s = oscillator()
    s.masses.append(Mass(id=7, m=0, x=(0.0, NAN, 0.0), v=(INF, 0.0, 0.0), f_ext=(0.0, 0.0, NAN)))
    s.masses.append(Mass(id=3, m=-1, x=(1.0, 2.0, 3.0)))
    s.masses.append(Mass(id=4, m=NAN, x=(1.0, 2.0, 3.0)))
    out["bad_masses"] = s
    s = oscillator()
    s.masses.append(Mass(id=2, m=0.1, x=(0.0, 0.0, 0.0)))
    s.springs += [Spring(id=5, i=1, j=1, k=0.0, l0=-1.0),
                  Spring(id=2, i=-1, j=3, k=NAN, l0=0.1, group="nope"),
                  Spring(id=3, i=1, j=0, k=10.0, l0=0.2),
                  Spring(id=4, i=2, j=0, k=-5, l0=NAN, group="g"),
                  Spring(id=5, i=0, j=2, k=5.0, l0=INF)]
    s.groups["g"] = ActuationGroup("g")
    out["bad_springs"] = s
    s = oscillator()
    s.groups = {"a": ActuationGroup("b", amplitude=1.0), "c": ActuationGroup("c", mode="square", amplitude=NAN),
                "d": ActuationGroup("d", frequency=INF, amplitude=-0.5), "e": ActuationGroup("e", amplitude=-1.0)}
    out["bad_groups"] = s
    s = oscillator()
    s.planes = [ContactPlane(normal=(0.0, 2.0, 0.0)), ContactPlane(normal=(NAN, 1.0, 0.0), penalty=0.0),
                ContactPlane(normal=(0.6, 0.8, 0.0), friction=-1.0), ContactPlane(normal=(0, 1, 0), penalty=-3)]
    out["bad_planes"] = s
    s = oscillator()
    s.materials = [Material(k0=0.0), Material(l_ref=-1.0), Material(mass_per_node=None),
                   Material(density=-2.0, mass_per_node=None), Material(total_mass=NAN, mass_per_node=0.1),
                   Material(name="ok", l_ref=0.1)]
    out["bad_materials"] = s
    out["bad_dt"] = Scene(dt=0.0, damping=1.0, gravity=(0.0, NAN, 0.0))
    out["bad_dt_nan"] = Scene(dt=NAN, damping=-0.1)
    out["damping_small"] = Scene(damping=0.0001)
    # a larger random mix: many masses and springs, a few of them broken
    rng = np.random.default_rng(3)
    s = Scene(gravity=(0.0, -9.81, 0.0))
    for i in range(400):
        s.add_mass(tuple(rng.normal(0, 1, 3)), m=float(rng.uniform(0.05, 0.2)))
    pairs = set()
    while len(pairs) < 1500:
        a, b = (int(q) for q in rng.integers(0, 400, 2))
        if a != b:
            pairs.add((a, b))
    for a, b in sorted(pairs):
        if (min(a, b), max(a, b)) in s._pairs:
            continue
        s.add_spring(a, b, k=float(rng.uniform(100, 1000)))
    for idx in rng.choice(400, 12, replace=False):
        s.masses[int(idx)].m = float(rng.choice([0.0, -0.5, NAN]))
    for idx in rng.choice(len(s.springs), 20, replace=False):
        sp = s.springs[int(idx)]
        r = int(rng.integers(0, 5))
        if r == 0:
            sp.k = -1.0
        elif r == 1:
            sp.j = sp.i
        elif r == 2:
            sp.j = 400 + int(rng.integers(0, 3))
        elif r == 3:
            sp.l0 = 0.0
        else:
            other = s.springs[int(rng.integers(0, len(s.springs)))]
            sp.i, sp.j = other.j, other.i
    out["random_mix"] = s
    return out


def main():
    res = {}
    for name, scene in cases().items():
        res[name] = {"scene": describe(scene),
                     "violations": [[v.code, v.where, v.message, str(v)] for v in validate_scene(scene)]}
        print(name, len(res[name]["violations"]))
    with open(os.path.join(HERE, "validation.json"), "w") as fh:
        json.dump(res, fh, indent=0)
    _ = math


if __name__ == "__main__":
    main()
