"""Array-native voxel lattices and the synthetic workloads of the benchmarks.

``voxel_box`` is bit-identical to the reference's
``build_voxel_lattice(box_mesh(lo, hi), LatticeSpec(dim), material)``
(lattice.py:89-136) — same mass ids, same spring order, same rest lengths
(the fma-ddot rounding of ``np.linalg.norm``, lattice.py:84) and stiffness
(model.py:87-92) — but is built by the C++ builder in the shared library
(``ss_lattice_box``) into an :class:`~.model.ArrayScene`, in O(S) time
with no per-spring Python objects.

The workload helpers mirror reference bench.py:60-89 (``block_springs``,
``block_cells``, ``block_scene``), analysis.py:435-452 (``beam_lattice``)
and demos/crawler.py:27-50 (``crawler_scene``).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .model import ActuationGroup, ArrayScene, Material, contact_floor

PITCH = 0.1


def lattice_counts(lo, hi, dim: float) -> tuple[int, int, int]:
    """Grid node counts along each axis (lattice.py:104-107)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    counts = np.floor((hi - lo) / dim + 1e-9).astype(int) + 1
    return tuple(int(c) for c in counts)


def voxel_arrays(lo, hi, dim: float, k0: float = 1e4, l_ref: float | None = None,
                 plane_range: tuple[int, int] | None = None):
    """Raw builder output: (counts, x, si, sj, k, l0, spring_ids).

    ``plane_range=(i_lo, i_hi)`` restricts to the masses of x-planes
    [i_lo, i_hi) and the springs touching them (global ids kept)."""
    lib = _lib.lib()
    lo_a = (C.c_double * 3)(*[float(c) for c in lo])
    hi_a = (C.c_double * 3)(*[float(c) for c in hi])
    lref = float(dim if l_ref is None else l_ref)
    i_lo, i_hi = plane_range if plane_range is not None else (0, 0)
    counts = np.zeros(3, dtype=np.int64)
    nm = C.c_int64(0)
    ns = C.c_int64(0)
    _lib.check(lib.ss_lattice_box(lo_a, hi_a, float(dim), float(k0), lref, i_lo, i_hi,
                                  _lib.i64ptr(counts), C.byref(nm), C.byref(ns),
                                  None, None, None, None, None, None), "ss_lattice_box")
    x = np.empty((nm.value, 3), dtype=np.float64)
    si = np.empty(ns.value, dtype=np.int64)
    sj = np.empty(ns.value, dtype=np.int64)
    k = np.empty(ns.value, dtype=np.float64)
    l0 = np.empty(ns.value, dtype=np.float64)
    ids = np.empty(ns.value, dtype=np.int64)
    _lib.check(lib.ss_lattice_box(lo_a, hi_a, float(dim), float(k0), lref, i_lo, i_hi,
                                  _lib.i64ptr(counts), C.byref(nm), C.byref(ns),
                                  _lib.dptr(x), _lib.i64ptr(si), _lib.i64ptr(sj),
                                  _lib.dptr(k), _lib.dptr(l0), _lib.i64ptr(ids)), "ss_lattice_box")
    return tuple(int(c) for c in counts), x, si, sj, k, l0, ids


def voxel_box(lo, hi, dim: float, material: Material | None = None) -> ArrayScene:
    """``build_voxel_lattice(box_mesh(lo, hi), LatticeSpec(dim=dim), material)``."""
    material = material or Material()
    l_ref = material.l_ref if material.l_ref is not None else dim
    lo_a = np.asarray(lo, dtype=np.float64)
    hi_a = np.asarray(hi, dtype=np.float64)
    if np.any(hi_a <= lo_a):
        raise ValueError("box must have positive extent on every axis")
    _, x, si, sj, k, l0, _ = voxel_arrays(lo_a, hi_a, dim, material.k0, l_ref)
    volume = float(np.prod(hi_a - lo_a))
    node_mass = material.node_mass(x.shape[0], volume=volume or None)
    mat = material if material.l_ref is not None else Material(
        name=material.name, k0=material.k0, l_ref=dim, density=material.density,
        total_mass=material.total_mass, mass_per_node=material.mass_per_node)
    return ArrayScene(x=x, m=node_mass, si=si, sj=sj, k=k, l0=l0, materials=[mat])


# ----------------------------------------------------------- workloads

def block_springs(cells: int) -> int:
    """13 n^3 + 12 n^2 + 3 n (reference bench.py:60-69)."""
    if cells < 1:
        raise ValueError("cells must be >= 1")
    return 13 * cells ** 3 + 12 * cells ** 2 + 3 * cells


def block_cells(spring_count: int) -> int:
    """Cube edge whose block is closest to ``spring_count`` (bench.py:72-80)."""
    if spring_count < 1:
        raise ValueError("spring_count must be >= 1")
    guess = max(1, round((spring_count / 13) ** (1 / 3)))          # 13 n^3 dominates
    near = [c for c in range(guess - 1, guess + 3) if c >= 1]       # first minimum wins ties, as the reference
    return near[int(np.argmin([abs(block_springs(c) - spring_count) for c in near]))]


def block_scene(cells: int) -> ArrayScene:
    """Free solid block, gravity off (bench.py:83-89): the throughput workload."""
    side = cells * PITCH
    scene = voxel_box((0.0, 0.0, 0.0), (side, side, side), PITCH)
    scene.gravity = (0.0, 0.0, 0.0)
    return scene


def excite(scene: ArrayScene, seed: int = 11, sigma: float = 0.05,
           drift=(0.3, 0.2, 0.1)) -> ArrayScene:
    """Seeded velocities N(0, sigma) + drift, drawn mass by mass exactly like
    ``_excited_block`` (reference tests/test_acceptance.py:75-83)."""
    rng = np.random.default_rng(seed)
    drift = np.asarray(drift, dtype=np.float64)
    n = scene.mass_count
    # rng.normal(0, s, 3) per mass consumes the stream in mass order, which is
    # exactly one normal(0, s, (n, 3)) draw.
    scene.v = rng.normal(0.0, sigma, (n, 3)) + drift
    return scene


def beam_lattice(length=2.0, height=0.4, width=0.4, density=100.0, pitch=PITCH,
                 gravity=(0.0, 0.0, 0.0), material: Material | None = None) -> ArrayScene:
    """Anchored cantilever, root layer fixed (reference analysis.py:435-452)."""
    if material is None:
        material = Material(mass_per_node=density * pitch ** 3)
    scene = voxel_box((0.0, 0.0, 0.0), (length, height, width), pitch, material)
    scene.fixed = scene.x[:, 0] < pitch / 2.0
    scene.gravity = tuple(float(c) for c in gravity)
    return scene


def crawler_scene() -> ArrayScene:
    """The actuated two-segment crawler (reference demos/crawler.py:27-50)."""
    scene = voxel_box((0.0, 0.0, 0.0), (4 * PITCH, PITCH, PITCH), PITCH)
    scene.gravity = (0.0, -9.81, 0.0)
    scene.dt = 5e-5
    scene.planes.append(contact_floor(y=0.0, penalty=2e4, friction=0.8))
    scene.add_group(ActuationGroup("rear", amplitude=0.25, frequency=2.0, phase=0.5 * np.pi))
    scene.add_group(ActuationGroup("front", amplitude=0.25, frequency=2.0, phase=0.0))
    a = scene.x[scene.si]
    b = scene.x[scene.sj]
    on_floor = (a[:, 1] == 0.0) & (b[:, 1] == 0.0)
    longitudinal = np.abs(a[:, 0] - b[:, 0]) > 1e-12
    center = 0.5 * (a[:, 0] + b[:, 0])
    sel = on_floor & longitudinal
    mid = 2 * PITCH
    scene.assign_group(np.nonzero(sel & (center < mid))[0], "rear")
    scene.assign_group(np.nonzero(sel & ~(center < mid))[0], "front")
    return scene


def multi_material_cube(cells: int, stiff_factor: float = 10.0, stretch: float = 1e-3) -> ArrayScene:
    """Config 2: free cube, k x ``stiff_factor`` where both endpoints have
    x < side/2, released from a uniaxial x-stretch about the centroid with
    zero velocity."""
    scene = block_scene(cells)
    side = cells * PITCH
    both = (scene.x[scene.si, 0] < side / 2) & (scene.x[scene.sj, 0] < side / 2)
    scene.k = np.where(both, scene.k * stiff_factor, scene.k)
    cx = scene.x[:, 0].mean()
    scene.x = scene.x.copy()
    scene.x[:, 0] = cx + (scene.x[:, 0] - cx) * (1.0 + stretch)
    return scene


__all__ = ["voxel_box", "voxel_arrays", "lattice_counts", "block_springs", "block_cells",
           "block_scene", "excite", "beam_lattice", "crawler_scene", "multi_material_cube",
           "PITCH"]
_ = math
