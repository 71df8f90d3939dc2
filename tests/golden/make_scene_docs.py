"""Scene documents rendered by the REFERENCE (sceneio.render_scene) for the
scene-I/O parity tests (tests/test_sceneio.py).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_scene_docs.py
"""
import os
import sys

import numpy as np

from springsim import ActuationGroup, Scene, contact_floor
from springsim.analysis import BeamSpec, beam_lattice
from springsim.sceneio import render_scene

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenes")
sys.path.insert(0, "/root/reference/pkg/demos")
from crawler import build_crawler  # noqa: E402


def random_scene():
    rng = np.random.default_rng(3)
    sc = Scene(gravity=(0.0, -9.81, 0.0), dt=2e-4, damping=0.01)
    for i in range(12):
        sc.add_mass(tuple(rng.normal(0, 0.3, 3)), m=float(rng.uniform(0.05, 0.2)),
                    v=tuple(rng.normal(0, 0.1, 3)), f_ext=tuple(rng.normal(0, 0.01, 3)), fixed=(i == 0))
    sc.add_group(ActuationGroup("pulse", amplitude=0.1, frequency=3.0, phase=0.25))
    sc.add_group(ActuationGroup("grow", mode="constant-expansion", amplitude=0.05))
    pairs = set()
    while len(pairs) < 30:
        a, b = sorted(rng.choice(12, 2, replace=False).tolist())
        pairs.add((a, b))
    for q, (a, b) in enumerate(sorted(pairs, key=lambda p: rng.random())):
        sc.add_spring(a, b, k=float(rng.uniform(500, 2000)),
                      group=("pulse" if q % 5 == 0 else ("grow" if q % 7 == 0 else None)))
    sc.planes.append(contact_floor(y=-1.0, penalty=3e4, friction=0.5))
    return sc


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for name, sc in (("crawler", build_crawler()), ("beam_10x2x2", beam_lattice(BeamSpec(length=1.0, height=0.2, width=0.2))),
                     ("random12", random_scene())):
        with open(os.path.join(OUT, name + ".json"), "w") as fh:
            fh.write(render_scene(sc))
        print(name, sc.mass_count, sc.spring_count)
