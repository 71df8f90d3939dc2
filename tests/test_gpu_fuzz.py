"""Randomised fp64 parity beyond the golden scenes: seeded random scenes of
every shape the engine dispatches on (one-tile CTA-resident, multi-tile
compact, explicit-format fallback, CSR), with gravity, damping, f_ext, fixed
masses, contact planes with friction and both actuation modes, stepped by
every integrator; the GPU state must be bitwise the oracle's (the oracle is
pinned to the reference by tests/test_oracle_golden.py)."""
import os
import sys

import numpy as np
import pytest

from paper_2207_09334_b200 import Engine
from paper_2207_09334_b200.model import ActuationGroup, ArrayScene, ContactPlane, scene_arrays

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))

pytestmark = pytest.mark.gpu


def random_scene(seed, n, neighbours=8, long_range=0.0, lattice=False):
    """n masses in a box, each joined to its nearest neighbours (a lattice-like
    graph with tiles and halos); long_range > 0 adds that fraction of springs
    between random far pairs (huge halos: the explicit/CSR fallbacks).
    lattice=True: jittered lattice points whose springs take their rest length
    and stiffness from a few values (the compact format's dictionary); else
    every spring has its own k and l0 (the explicit format)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    side = 0.1 * n ** (1 / 3)
    if lattice:
        c = int(round(n ** (1 / 3)))
        g = np.stack(np.meshgrid(*[np.arange(c)] * 3, indexing="ij"), -1).reshape(-1, 3) * 0.1
        n = g.shape[0]
        x = g + rng.normal(0.0, 0.004, g.shape)
    else:
        x = rng.uniform(0.0, side, (n, 3))
    _, nb = cKDTree(x).query(x, k=neighbours + 1)
    pairs = {(min(i, j), max(i, j)) for i in range(n) for j in nb[i, 1:] if i != j}
    for _ in range(int(long_range * len(pairs))):
        a, b = (int(q) for q in rng.integers(0, n, 2))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    pairs = sorted(pairs)
    order = rng.permutation(len(pairs)) if seed % 2 else np.arange(len(pairs))   # id order: sorted or random
    si = np.array([pairs[q][0] for q in order], dtype=np.int64)
    sj = np.array([pairs[q][1] for q in order], dtype=np.int64)
    flip = rng.random(si.size) < 0.3
    si[flip], sj[flip] = sj[flip].copy(), si[flip].copy()
    if lattice:
        rest = np.round(np.linalg.norm(g[sj] - g[si], axis=1), 12)
        l0 = rest * rng.choice([0.98, 1.0, 1.02], si.size)
        k = rng.choice([500.0, 1000.0], si.size) / rest
    else:
        l0 = np.linalg.norm(x[sj] - x[si], axis=1) * rng.uniform(0.97, 1.03, si.size)
        k = rng.uniform(200.0, 2000.0, si.size)
    groups = {"a": ActuationGroup("a", amplitude=0.05, frequency=5.0, phase=0.2),
              "b": ActuationGroup("b", mode="constant-expansion", amplitude=-0.03)}
    r = rng.random(si.size)
    group = np.where(r < 0.15, 0, np.where(r < 0.25, 1, -1)).astype(np.int32)
    f_ext = np.where(rng.random((n, 1)) < 0.1, rng.normal(0, 0.05, (n, 3)), 0.0)
    planes = [ContactPlane(normal=(0.0, 1.0, 0.0), offset=0.02 * side, penalty=2e4, friction=0.5)]
    if seed % 3 == 0:
        planes.append(ContactPlane(normal=(1.0, 0.0, 0.0), offset=0.05 * side, penalty=1e4, friction=0.0))
    return ArrayScene(x=x, m=rng.uniform(0.05, 0.2, n), si=si, sj=sj, k=k, l0=l0,
                      v=rng.normal(0.0, 0.05, (n, 3)), f_ext=f_ext, fixed=rng.random(n) < 0.04,
                      gravity=(0.0, -9.81, 0.0) if seed % 4 else (0.0, 0.0, 0.0), dt=1e-4,
                      damping=1e-3 if seed % 5 == 0 else 0.0, groups=groups, group=group, planes=planes)


CASES = [  # (seed, masses, long-range fraction, lattice, layout, expected tile format or None)
    (1, 60, 0.0, False, "auto", None),       # one tile: the CTA-resident kernel
    (2, 216, 0.0, True, "auto", None),
    (3, 1000, 0.0, True, "auto", 3),         # multi-tile compact fp64 (a dictionary per tile)
    (4, 2744, 0.0, True, "auto", 3),
    (5, 700, 0.05, False, "auto", None),     # long-range springs: big halos / fallbacks
    (6, 1500, 0.0, False, "csr", None),
    (7, 1200, 0.0, False, "auto", 5),        # every spring distinct: the inline (general-graph) fp64 format
    (8, 3375, 0.01, True, "auto", None),
]


@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
@pytest.mark.parametrize("seed,n,long_range,lattice,layout,fmt", CASES)
def test_random_scene_fp64_bitwise(seed, n, long_range, lattice, layout, fmt, integrator):
    import oracle as orc
    scene = random_scene(seed, n, long_range=long_range, lattice=lattice)
    eng = Engine(scene, integrator=integrator, precision="f64", layout=layout)
    if fmt is not None and integrator != "rk4":
        # compact fp64 tiles step on tile_f64_kernel (4; 5 with inline records)
        assert eng.info()["tile_kernel"] == (4 if fmt == 3 else fmt)
    ref = orc.OracleEngine(scene_arrays(scene), integrator=integrator)
    steps = (17, 40) if integrator == "rk4" else (37, 120)
    for count in steps:
        eng.step(count)
        ref.step(count)
        assert eng.x.tobytes() == ref.x.tobytes(), (seed, integrator, count, "x")
        assert eng.v.tobytes() == ref.v.tobytes(), (seed, integrator, count, "v")
    assert eng.degenerate_springs == ref.degenerate_springs


@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
@pytest.mark.parametrize("seed,n,long_range,lattice,layout,fmt", CASES)
def test_random_scene_fp32_within_tolerance(seed, n, long_range, lattice, layout, fmt, integrator):
    """The same scenes in fp32 production mode: within 1e-4 of the position
    scale and 1e-3 of the displacement of the fp64 oracle."""
    import oracle as orc
    scene = random_scene(seed, n, long_range=long_range, lattice=lattice)
    eng = Engine(scene, integrator=integrator, precision="f32", layout=layout)
    if fmt == 5:                                            # every spring distinct: fp32 inline records
        assert eng.info()["tile_kernel"] == 6
    ref = orc.OracleEngine(scene_arrays(scene), integrator=integrator)
    count = 60 if integrator == "rk4" else 150
    eng.step(count)
    ref.step(count)
    err = np.abs(eng.x - ref.x).max()
    assert err <= 1e-4 * np.abs(ref.x).max(), (seed, integrator, err)
    assert err <= 1e-3 * np.abs(ref.x - scene.x).max(), (seed, integrator, err)
