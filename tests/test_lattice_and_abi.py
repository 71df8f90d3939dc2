"""CPU-only checks: array-native lattice builder vs reference topology digests,
workload helpers, and the C ABI surface of the shared library."""

import hashlib
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

from paper_2207_09334_b200 import _lib
from paper_2207_09334_b200 import lattice as L
from paper_2207_09334_b200.model import ActuationGroup, Scene, scene_arrays, validate_scene

TOPO = json.load(open(os.path.join(GOLDEN, "topology.json")))


def digest(scene) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(scene.x).tobytes())
    h.update(np.ascontiguousarray(scene.m).tobytes())
    for a in (scene.si, scene.sj, scene.k, scene.l0):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("n", [1, 2, 3, 9, 20])
def test_block_scene_bit_identical_to_reference(n):
    s = L.block_scene(n)
    assert digest(s) == TOPO[f"block_{n}"]
    assert s.spring_count == L.block_springs(n)
    assert s.mass_count == (n + 1) ** 3
    assert s.gravity == (0.0, 0.0, 0.0)


def test_beams_bit_identical_to_reference():
    assert digest(L.beam_lattice()) == TOPO["beam_20x4x4"]
    b40 = L.beam_lattice(length=4.0)
    assert digest(b40) == TOPO["beam_40x4x4"]
    assert [b40.mass_count, b40.spring_count] == TOPO["beam_40x4x4_counts"]
    assert b40.m[0] == TOPO["beam_40x4x4_mass"]
    assert int(b40.fixed.sum()) == 25


def test_box_with_inexact_extent_keeps_surface_nodes():
    s = L.voxel_box((0, 0, 0), (0.3, 0.2, 0.1), 0.1)
    assert digest(s) == TOPO["box_0.3x0.2x0.1"]


def test_crawler_topology_and_groups():
    c = L.crawler_scene()
    assert digest(c) == TOPO["crawler"]
    assert c.group.tolist() == TOPO["crawler_groups"]
    assert list(c.groups) == ["rear", "front"]


def test_excited_velocities_match_reference_stream():
    s = L.excite(L.block_scene(9), seed=11)
    assert hashlib.sha256(s.v.tobytes()).hexdigest() == TOPO["excited9_v_sha256"]


def test_block_sizing_matches_reference():
    for n, s in TOPO["block_springs"].items():
        assert L.block_springs(int(n)) == s
    for s, n in TOPO["block_cells"].items():
        assert L.block_cells(int(s)) == n
    with pytest.raises(ValueError):
        L.block_springs(0)
    with pytest.raises(ValueError):
        L.block_cells(0)


def test_slab_emission_partitions_the_lattice():
    """Spatial slabs (multi-GPU sharding) carry global spring ids; the union of
    the slabs' owned springs is the whole lattice, each exactly once."""
    counts, x, si, sj, k, l0, ids = L.voxel_arrays((0, 0, 0), (0.7, 0.4, 0.5), 0.1)
    nx = counts[0]
    plane = counts[1] * counts[2]
    seen = np.zeros(si.shape[0], dtype=np.int64)
    cuts = [0, 3, 5, nx]
    for a, b in zip(cuts[:-1], cuts[1:]):
        c2, xs, si2, sj2, k2, l02, ids2 = L.voxel_arrays((0, 0, 0), (0.7, 0.4, 0.5), 0.1, plane_range=(a, b))
        assert xs.tobytes() == x[a * plane:b * plane].tobytes()
        assert np.array_equal(si2, si[ids2]) and np.array_equal(sj2, sj[ids2])
        assert k2.tobytes() == k[ids2].tobytes() and l02.tobytes() == l0[ids2].tobytes()
        own = (si2 >= a * plane) & (si2 < b * plane)          # lower endpoint in slab
        seen[ids2[own]] += 1
        touches = ((si >= a * plane) & (si < b * plane)) | ((sj >= a * plane) & (sj < b * plane))
        assert set(ids2.tolist()) == set(np.nonzero(touches)[0].tolist())
    assert (seen == 1).all()


def test_scene_api_and_freeze():
    sc = Scene(gravity=(0.0, 0.0, 0.0))
    a = sc.add_mass((0, 0, 0), fixed=True)
    b = sc.add_mass((1.2, 0, 0))
    sc.add_group(ActuationGroup("g", amplitude=0.1))
    s = sc.add_spring(a, b, k=10.0, group="g")
    assert sc.springs[s].l0 == 1.2
    with pytest.raises(ValueError):
        sc.add_spring(b, a, k=1.0)
    with pytest.raises(ValueError):
        sc.add_group(ActuationGroup("g"))
    assert validate_scene(sc) == []
    arr = scene_arrays(sc)
    assert arr.group.tolist() == [0]
    assert arr.fixed.tolist() == [True, False]
    assert sc.degrees() == [1, 1]


# ------------------------------------------------------------- C ABI


def header_symbols():
    text = open(os.path.join(ROOT, "include", "springsim_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert lib.ss_abi_version() == 2


def test_tile_plan_statistics_on_host():
    """The tiled layout of a brick-aligned cube: tiles follow 4x8x8 bricks,
    so the halo ratio and the foreign-reference fraction stay near the
    brick's geometric values (6*10*10/256 = 2.34; 4.05 of 13 references = 31%)."""
    from paper_2207_09334_b200.engine import plan
    info = plan(L.block_scene(31))          # 32^3 masses: exact bricks
    assert info["tile_count"] == 32 ** 3 // 256
    assert info["canonical_order"] == 1
    assert info["tile_halo_ratio"] <= 2.4
    assert info["tile_foreign_frac"] <= 0.32
    ragged = plan(L.block_scene(29))        # 30^3 masses: partial bricks
    assert ragged["tile_halo_ratio"] <= 2.6
    assert ragged["tile_foreign_frac"] <= 0.32
    assert ragged["smem_per_block"] <= 76 * 1024


def test_fp64_compact_tile_plan_on_host(monkeypatch):
    """fp64 tiles use the compact format (spring-id ordered incidence lists
    over a per-tile (k, l0, group) dictionary) when every tile has at most 64
    distinct records; a tile with more falls back to the inline format ((k,
    l0) per incidence), which SS_TILE_DICT=0 forces; SS_TILE_DICT=explicit
    forces the older explicit format."""
    from paper_2207_09334_b200.engine import plan
    cube = L.block_scene(15)
    info = plan(cube, precision="f64")
    assert info["tile_kernel"] == 3
    assert info["tile_foreign_frac"] == 0.0
    assert info["smem_per_block"] <= 56 * 1024          # 4 CTAs per SM
    rnd = L.block_scene(15)
    rnd.k = rnd.k * (1.0 + 1e-6 * np.arange(rnd.k.size))    # every spring distinct
    inl = plan(rnd, precision="f64")
    assert inl["tile_kernel"] == 5
    assert inl["tile_blob_bytes"] >= 16 * 2 * rnd.spring_count      # (k, l0) at both endpoints
    monkeypatch.setenv("SS_TILE_DICT", "0")
    assert plan(cube, precision="f64")["tile_kernel"] == 5
    monkeypatch.setenv("SS_TILE_DICT", "explicit")
    assert plan(cube, precision="f64")["tile_kernel"] == 0
    assert plan(cube, precision="f32")["tile_kernel"] == 1
    monkeypatch.delenv("SS_TILE_DICT")
    assert plan(cube, precision="f32")["tile_kernel"] == 2
    f32i = plan(rnd, precision="f32")
    assert f32i["tile_kernel"] == 6 and f32i["tile_blob_bytes"] >= 8 * 2 * rnd.spring_count   # (k, k*l0)
    # positions off the lattice, materials shared: the (k, k*l0, group)
    # dictionary with rest vectors formed from X0 (7); fp64 keys never held D
    from paper_2207_09334_b200 import crawler_scene, replicate
    pop = replicate(crawler_scene(), 96, jitter=1e-6, seed=3)
    assert plan(pop, precision="f32")["tile_kernel"] == 7
    assert plan(pop, precision="f64")["tile_kernel"] == 3


def test_engine_without_gpu_fails_loudly():
    """No CPU fallback: on a host without a device, construction raises."""
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_2207_09334_b200 import Engine
    with pytest.raises(_lib.CudaError):
        Engine(L.block_scene(1))


def test_bad_arguments_are_value_errors():
    from paper_2207_09334_b200 import Engine
    with pytest.raises(ValueError):
        Engine(L.block_scene(1), integrator="leapfrog")
    with pytest.raises(ValueError):
        Engine(L.block_scene(1), mode="turbo")
    with pytest.raises(ValueError):
        Engine(L.block_scene(1), precision="f16")


@pytest.mark.parametrize("n", [42, 91])
def test_bench_size_cubes_bit_identical_to_reference(n):
    """configs[1] (984,438 springs) and configs[3] (9,896,068 springs): the
    array builder reproduces the reference's block_scene(n) digests
    (tests/golden/make_topology_big.py built them through the reference
    object model)."""
    s = L.block_scene(n)
    assert digest(s) == TOPO[f"block_{n}"]
    assert s.spring_count == L.block_springs(n)


def test_bench_cube_excited_velocities_match_reference_stream():
    s = L.excite(L.block_scene(91), seed=11)
    assert hashlib.sha256(np.ascontiguousarray(s.v).tobytes()).hexdigest() == TOPO["excited91_v_sha256"]


def _validation_scene(desc):
    from paper_2207_09334_b200.model import ContactPlane, Mass, Material, Spring
    sc = Scene(gravity=tuple(desc["gravity"]), dt=desc["dt"], damping=desc["damping"])
    sc.masses = [Mass(i, m, tuple(x), tuple(v), tuple(f), fx) for i, m, x, v, f, fx in desc["masses"]]
    sc.springs = [Spring(i, a, b, k, l0, g) for i, a, b, k, l0, g in desc["springs"]]
    sc.groups = {key: ActuationGroup(lab, mode, amp, freq, ph) for key, lab, mode, amp, freq, ph in desc["groups"]}
    sc.planes = [ContactPlane(tuple(nrm), off, pen, fr) for nrm, off, pen, fr in desc["planes"]]
    sc.materials = [Material(*m) for m in desc["materials"]]
    return sc


@pytest.mark.parametrize("case", sorted(json.load(open(os.path.join(GOLDEN, "validation.json")))))
def test_validate_scene_matches_reference_output(case):
    """Codes, field paths, messages and order identical to the reference's
    validate_scene on the same (broken) scenes (tests/golden/make_validation.py)."""
    want = json.load(open(os.path.join(GOLDEN, "validation.json")))[case]
    got = validate_scene(_validation_scene(want["scene"]))
    assert [[v.code, v.where, v.message, str(v)] for v in got] == want["violations"]


def test_validate_scene_vectorised_on_array_scenes():
    s = L.block_scene(30)
    assert validate_scene(s) == []
    s.k = s.k.copy()
    s.k[[5, 70000]] = [-1.0, np.nan]
    s.si = s.si.copy()
    s.si[9] = s.sj[9]
    got = validate_scene(s)
    assert [(v.where, v.code) for v in got] == [("springs[5].k", "nonpositive-stiffness"),
                                               ("springs[9]", "self-loop"),
                                               ("springs[70000].k", "nonpositive-stiffness")]
