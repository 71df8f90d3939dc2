"""Generate golden vectors from the REAL reference (run in the dev container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py

Every case builds a scene through the reference's own API (springsim.Scene /
build_voxel_lattice / bench.block_scene / demos recipes), freezes the exact
arrays ``springsim.Engine.__init__`` sees (engine.py:192-220), runs the
reference ``Engine`` in serial mode (the bit-level oracle, engine.py:3-14) and
stores inputs + checkpointed outputs in ``tests/golden/<case>.npz``.  The
fixtures travel with the repo; /root/reference does not.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import springsim  # noqa: E402  (reference package, from PYTHONPATH)
from springsim import (ActuationGroup, ContactPlane, Engine, LatticeSpec, Scene, box_mesh,  # noqa: E402
                       build_voxel_lattice, contact_floor)
from springsim.bench import block_cells, block_scene  # noqa: E402
from springsim.engine import DivergenceError  # noqa: E402
from springsim.analysis import BeamSpec, beam_lattice  # noqa: E402


def freeze(scene) -> dict:
    """Scene -> the arrays Engine.__init__ builds (engine.py:192-220)."""
    labels = list(scene.groups)
    idx = {l: i for i, l in enumerate(labels)}
    d = {
        "x": np.array([m.x for m in scene.masses], dtype=np.float64),
        "v": np.array([m.v for m in scene.masses], dtype=np.float64),
        "m": np.array([m.m for m in scene.masses], dtype=np.float64),
        "f_ext": np.array([m.f_ext for m in scene.masses], dtype=np.float64),
        "fixed": np.array([m.fixed for m in scene.masses], dtype=bool),
        "si": np.array([s.i for s in scene.springs], dtype=np.int64),
        "sj": np.array([s.j for s in scene.springs], dtype=np.int64),
        "k": np.array([s.k for s in scene.springs], dtype=np.float64),
        "l0": np.array([s.l0 for s in scene.springs], dtype=np.float64),
        "group": np.array([-1 if s.group is None else idx[s.group] for s in scene.springs],
                          dtype=np.int32),
        "group_labels": np.array(labels, dtype=str) if labels else np.zeros(0, dtype="<U1"),
        "group_mode": np.array([scene.groups[l].mode for l in labels], dtype=str)
        if labels else np.zeros(0, dtype="<U1"),
        "group_num": np.array([[scene.groups[l].amplitude, scene.groups[l].frequency,
                                scene.groups[l].phase] for l in labels], dtype=np.float64).reshape(-1, 3),
        "planes": np.array([[*p.normal, p.offset, p.penalty, p.friction] for p in scene.planes],
                           dtype=np.float64).reshape(-1, 6),
        "gravity": np.asarray(scene.gravity, dtype=np.float64),
        "dt": np.float64(scene.dt),
        "damping": np.float64(scene.damping),
    }
    d["x"] = d["x"].reshape(-1, 3)
    d["v"] = d["v"].reshape(-1, 3)
    d["f_ext"] = d["f_ext"].reshape(-1, 3)
    return d


def run_case(name, scene, integrator, checkpoints, setup=None, extra=None):
    eng = Engine(scene, integrator=integrator, mode="serial")
    if setup:
        setup(eng)
    out = {f"in_{k}": v for k, v in freeze(scene).items()}
    # parameters applied through setters after construction (setup) are
    # stored as the engine's live values
    out["in_damping"] = np.float64(eng.damping)
    out["in_f_ext"] = eng.f_ext.copy()
    out["in_gravity"] = np.asarray(eng.gravity, dtype=np.float64)
    out["integrator"] = np.array(integrator)
    done = 0
    ck = []
    for c in checkpoints:
        eng.step(c - done)
        done = c
        ck.append(c)
        out[f"x_{c}"] = eng.x.copy()
        out[f"v_{c}"] = eng.v.copy()
        if eng.x_prev is not None:
            out[f"xp_{c}"] = eng.x_prev.copy()
        out[f"t_{c}"] = np.float64(eng.t)
        out[f"deg_{c}"] = np.int64(eng.degenerate_springs)
    out["checkpoints"] = np.array(ck, dtype=np.int64)
    if extra:
        out.update(extra)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {len(scene.masses)} masses, {len(scene.springs)} springs, {integrator}, "
          f"checkpoints {ck} -> {os.path.getsize(path)} B")


def excited(cells, seed=11):
    """tests/test_acceptance.py:75-83"""
    scene = block_scene(cells)
    rng = np.random.default_rng(seed)
    drift = np.array([0.3, 0.2, 0.1])
    for mass in scene.masses:
        mass.v = tuple(rng.normal(0.0, 0.05, 3) + drift)
    return scene


def anchored_block(cells, dim=0.1):
    """tests/test_parallel.py:42-50"""
    nx, ny, nz = cells
    scene = build_voxel_lattice(box_mesh((0, 0, 0), (nx * dim, ny * dim, nz * dim)), LatticeSpec(dim=dim))
    for mass in scene.masses:
        if mass.x[0] < dim / 2:
            mass.fixed = True
    return scene


def crawler():
    sys.path.insert(0, "/root/reference/pkg/demos")
    import crawler as cr  # demos/crawler.py:27-50
    return cr.build_crawler()


def random_scene(seed=5, n=30, s=90):
    """Springs in random id order (not sorted by endpoint): exercises the
    generic per-mass ordering path."""
    rng = np.random.default_rng(seed)
    scene = Scene(gravity=(0.0, -9.81, 0.0), dt=2e-4, damping=0.0)
    scene.planes.append(contact_floor(y=-0.05, penalty=5e4, friction=0.4))
    scene.planes.append(ContactPlane(normal=(1.0, 0.0, 0.0), offset=-0.5, penalty=3e4, friction=0.0))
    scene.add_group(ActuationGroup("a", amplitude=0.2, frequency=3.0, phase=0.3))
    scene.add_group(ActuationGroup("b", mode="constant-expansion", amplitude=-0.1))
    for i in range(n):
        scene.add_mass(tuple(rng.uniform(-0.3, 0.3, 3)), m=float(rng.uniform(0.05, 0.2)),
                       v=tuple(rng.normal(0, 0.1, 3)), fixed=bool(i == 3))
    pairs = set()
    while len(pairs) < s:
        a, b = (int(q) for q in rng.integers(0, n, 2))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    pairs = list(pairs)
    rng.shuffle(pairs)
    for a, b in pairs:
        if rng.random() < 0.5:
            a, b = b, a
        r = rng.random()
        grp = "a" if r < 0.2 else ("b" if r < 0.3 else None)
        scene.add_spring(a, b, k=float(rng.uniform(200, 2000)), group=grp)
    return scene


def topo_digest(scene) -> str:
    f = freeze(scene)
    h = hashlib.sha256()
    for key in ("x", "m", "si", "sj", "k", "l0"):
        h.update(np.ascontiguousarray(f[key]).tobytes())
    return h.hexdigest()


def main():
    # --- hot-path integrator parity cases
    from springsim.model import Scene as RScene
    osc = RScene(gravity=(0.0, 0.0, 0.0))
    a = osc.add_mass((0.0, 1.0, 0.0), m=0.1, fixed=True)
    b = osc.add_mass((0.0, 0.0, 0.0), m=0.1)
    osc.add_spring(a, b, k=10000.0, l0=1.0)
    osc.masses[1].x = (0.0, -0.05, 0.0)
    for integ in ("euler", "verlet", "rk4"):
        run_case(f"oscillator_{integ}", osc, integ, [1, 10, 100])

    for integ in ("euler", "verlet", "rk4"):
        run_case(f"block3_excited_{integ}", excited(3), integ, [1, 10, 50])

    run_case("block4_anchored_verlet", anchored_block((4, 4, 4)), "verlet", [100, 500, 1000])
    run_case("block9_excited_verlet", excited(9), "verlet", [10, 100, 1000])

    # cantilever 10x2x2, fixed root, gravity, tip load, damping
    cant = beam_lattice(BeamSpec(length=1.0, height=0.2, width=0.2), gravity=(0.0, -9.81, 0.0))
    tip = [i for i, m in enumerate(cant.masses) if m.x[0] > 1.0 - 0.05]

    def cant_setup(eng):
        for t in tip:
            eng.set_external_force(t, (0.0, -0.01, 0.0))
        eng.set_damping(1e-4)
    for integ in ("verlet", "euler"):
        run_case(f"cantilever_10x2x2_{integ}", cant, integ, [1, 50, 200], setup=cant_setup)

    cr = crawler()

    def cr_setup(eng):
        eng.set_damping(2e-4)
    run_case("crawler_verlet", cr, "verlet", [100, 400, 2000], setup=cr_setup)
    run_case("crawler_euler", cr, "euler", [100, 400], setup=cr_setup)
    run_case("crawler_rk4", cr, "rk4", [50, 200], setup=cr_setup)

    rs = random_scene()
    for integ in ("euler", "verlet", "rk4"):
        run_case(f"random_order_{integ}", rs, integ, [1, 50, 300])

    # degenerate spring counted, not faulted (tests/test_engine.py:61-69)
    deg = RScene(gravity=(0.0, 0.0, 0.0))
    deg.add_mass((0, 0, 0))
    deg.add_mass((0, 0, 0))
    deg.add_spring(0, 1, k=100.0, l0=1.0)
    run_case("degenerate_euler", deg, "euler", [3])

    # divergence names mass and step (tests/test_engine.py:253-261)
    dv = RScene(gravity=(0.0, 0.0, 0.0), dt=10.0)
    dv.add_mass((0.0, 0.0, 0.0), fixed=True)
    dv.add_mass((1.5, 0.0, 0.0), m=0.01)
    dv.add_spring(0, 1, k=1e4, l0=1.0)
    e = Engine(dv, integrator="euler")
    try:
        e.step(10000)
        raise SystemExit("expected divergence")
    except DivergenceError as err:
        out = {f"in_{k}": v for k, v in freeze(dv).items()}
        out.update(integrator=np.array("euler"), div_mass=np.int64(err.mass_id),
                   div_step=np.int64(err.step), x_div=e.x.copy(), v_div=e.v.copy())
        np.savez_compressed(os.path.join(HERE, "divergence_euler.npz"), **out)
        print("divergence:", err.mass_id, err.step)

    # forces at a perturbed state (SURVEY App. A probe)
    blk = block_scene(6)
    eng = Engine(blk)
    rng = np.random.default_rng(0)
    xp = eng.x + rng.normal(0, 0.01, eng.x.shape)
    vp = rng.normal(0, 0.1, eng.x.shape)
    acc = eng.forces(xp, vp, 0.0)
    out = {f"in_{k}": v for k, v in freeze(blk).items()}
    out.update(px=xp, pv=vp, acc=acc)
    np.savez_compressed(os.path.join(HERE, "forces_block6.npz"), **out)

    # topology digests / small topologies (lattice.py:89-136)
    topo = {}
    for n in (1, 2, 3, 9, 20):
        topo[f"block_{n}"] = topo_digest(block_scene(n))
    topo["beam_20x4x4"] = topo_digest(beam_lattice(BeamSpec()))
    topo["beam_40x4x4"] = topo_digest(beam_lattice(BeamSpec(length=4.0)))
    topo["box_0.3x0.2x0.1"] = topo_digest(build_voxel_lattice(box_mesh((0, 0, 0), (0.3, 0.2, 0.1)),
                                                              LatticeSpec(dim=0.1)))
    topo["crawler"] = topo_digest(cr)
    topo["crawler_groups"] = [-1 if s.group is None else list(cr.groups).index(s.group)
                              for s in cr.springs]
    ex = excited(9)
    topo["excited9_v_sha256"] = hashlib.sha256(
        np.array([m.v for m in ex.masses], dtype=np.float64).tobytes()).hexdigest()
    topo["beam_40x4x4_mass"] = beam_lattice(BeamSpec(length=4.0)).masses[0].m
    topo["beam_40x4x4_counts"] = [len(beam_lattice(BeamSpec(length=4.0)).masses),
                                  len(beam_lattice(BeamSpec(length=4.0)).springs)]
    topo["block_springs"] = {str(n): springsim.bench.block_springs(n) for n in (1, 2, 3, 9, 42, 91, 313)}
    topo["block_cells"] = {str(s): block_cells(s) for s in (28, 500, 10_000, 1_000_000, 10_000_000,
                                                             400_000_000)}
    with open(os.path.join(HERE, "topology.json"), "w") as fh:
        json.dump(topo, fh, indent=1, sort_keys=True)
    print("topology digests written")


if __name__ == "__main__":
    main()
