"""GPU parity: the sm_100a kernels through the C ABI vs the reference.

fp64 mode must be BITWISE equal to the reference's serial mode (the golden
vectors were produced by the real reference; the oracle reproduces them, see
test_oracle_golden.py).  fp32 mode must stay within the stated tolerance
max|x - x_ref| / max|x_ref| <= 1e-4 over <= 1000 steps.
"""

import numpy as np
import pytest

from conftest import golden_arrays, golden_cases, golden_scene, load_golden

from paper_2207_09334_b200 import DivergenceError, Engine
from paper_2207_09334_b200 import lattice as L

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4     # relative position tolerance of the fp32 production mode


def run_engine(case, layout, precision="f64"):
    d = load_golden(case)
    eng = Engine(golden_scene(d), integrator=str(d["integrator"]), precision=precision,
                 layout=layout)
    return d, eng


@pytest.mark.parametrize("layout", ["csr", "ell", "tile"])
@pytest.mark.parametrize("case", golden_cases())
def test_fp64_bitwise_vs_reference(case, layout):
    d, eng = run_engine(case, layout)
    done = 0
    for c in d["checkpoints"]:
        eng.step(int(c) - done)
        done = int(c)
        assert eng.x.tobytes() == d[f"x_{c}"].tobytes(), (case, layout, c, "x")
        assert eng.v.tobytes() == d[f"v_{c}"].tobytes(), (case, layout, c, "v")
        if f"xp_{c}" in d.files:
            assert eng.x_prev.tobytes() == d[f"xp_{c}"].tobytes(), (case, layout, c, "x_prev")
        assert eng.t == float(d[f"t_{c}"]) and eng.n == int(c)
        assert eng.degenerate_springs == int(d[f"deg_{c}"])


@pytest.mark.parametrize("fmt,kernel", [("0", 5), ("explicit", 0)])
@pytest.mark.parametrize("case", golden_cases())
def test_fp64_general_tile_formats_bitwise(case, fmt, kernel, monkeypatch):
    """The fp64 formats for graphs whose tiles do not fit the 64-entry
    (k, l0, group) dictionary are bitwise equal to the reference too: the
    inline format (the general-graph path; SS_TILE_DICT=0 forces it) and the
    older explicit format (SS_TILE_DICT=explicit)."""
    monkeypatch.setenv("SS_TILE_DICT", fmt)
    d, eng = run_engine(case, "tile")
    assert eng.info()["tile_kernel"] == kernel
    done = 0
    for c in d["checkpoints"]:
        eng.step(int(c) - done)
        done = int(c)
        assert eng.x.tobytes() == d[f"x_{c}"].tobytes(), (case, c, "x")
        assert eng.v.tobytes() == d[f"v_{c}"].tobytes(), (case, c, "v")
        assert eng.degenerate_springs == int(d[f"deg_{c}"])


def test_fp64_compact_format_is_the_default():
    """Compact fp64 tiles, stepped by tile_f64_kernel (4) for Euler, Verlet
    and the four RK4 stages."""
    d, eng = run_engine("block9_excited_verlet", "tile")
    assert eng.info()["tile_kernel"] == 4
    rk = Engine(L.block_scene(9), integrator="rk4", precision="f64", layout="tile")
    assert rk.info()["tile_kernel"] == 4


@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
def test_fp64_compact_equals_explicit_on_a_crawler_batch(integrator, monkeypatch):
    """The three fp64 tile formats on 48 jittered crawlers (2 actuation
    groups, ground contact with friction): identical bits after 600 steps."""
    from paper_2207_09334_b200 import crawler_scene, replicate
    batch = replicate(crawler_scene(), 48, jitter=1e-6, seed=3)
    runs = []
    for fmt, kernel in (("1", 4), ("0", 5), ("explicit", 0)):
        monkeypatch.setenv("SS_TILE_DICT", fmt)
        eng = Engine(batch, integrator=integrator, precision="f64", layout="tile")
        assert eng.info()["tile_kernel"] == kernel
        eng.set_damping(1e-4)
        eng.step(600)
        runs.append((eng.x.copy(), eng.v.copy(), eng.degenerate_springs))
        eng.close()
    for other in runs[1:]:
        assert runs[0][0].tobytes() == other[0].tobytes()
        assert runs[0][1].tobytes() == other[1].tobytes()
        assert runs[0][2] == other[2]


def test_fp64_compact_equals_explicit_on_a_multi_tile_cube(monkeypatch):
    """An excited 13^3-cell cube (11 tiles with halos), all three formats:
    identical bits."""
    scene = L.excite(L.block_scene(13), seed=5)
    runs = []
    for fmt in ("1", "0", "explicit"):
        monkeypatch.setenv("SS_TILE_DICT", fmt)
        eng = Engine(scene, integrator="verlet", precision="f64", layout="tile")
        eng.step(300)
        runs.append((eng.x.copy(), eng.v.copy()))
        eng.close()
    for other in runs[1:]:
        assert runs[0][0].tobytes() == other[0].tobytes()
        assert runs[0][1].tobytes() == other[1].tobytes()


@pytest.mark.parametrize("layout", ["csr", "ell", "tile"])
@pytest.mark.parametrize("case", [c for c in golden_cases() if "degenerate" not in c])
def test_fp32_within_tolerance(case, layout):
    run_case_fp32(case, layout)


def run_case_fp32(case, layout):
    d, eng = run_engine(case, layout, precision="f32")
    done = 0
    for c in d["checkpoints"]:
        if int(c) > 1000:
            break
        eng.step(int(c) - done)
        done = int(c)
        ref = d[f"x_{c}"]
        err = np.abs(eng.x - ref).max() / max(np.abs(ref).max(), 1e-300)
        assert err <= FP32_TOL, (case, layout, c, err)


@pytest.mark.parametrize("layout", ["csr", "ell", "tile"])
def test_divergence_names_mass_and_step(layout):
    d = load_golden("divergence_euler")
    eng = Engine(golden_scene(d), integrator="euler", layout=layout)
    with pytest.raises(DivergenceError) as err:
        eng.step(10000)
    assert err.value.mass_id == int(d["div_mass"])
    assert err.value.step == int(d["div_step"])
    assert "smaller dt" in str(err.value)
    assert eng.n == int(d["div_step"])
    assert eng.x.tobytes() == d["x_div"].tobytes()
    assert eng.v.tobytes() == d["v_div"].tobytes()


@pytest.mark.parametrize("layout", ["csr", "ell", "tile"])
def test_forces_bitwise(layout):
    d = load_golden("forces_block6")
    eng = Engine(golden_scene(d), layout=layout)
    acc = eng.forces(d["px"], d["pv"], 0.0)
    assert acc.tobytes() == d["acc"].tobytes()


def test_batched_equals_single_steps():
    """step(n) in one device batch == n calls of step(1) (bitwise)."""
    d = load_golden("crawler_verlet")
    a = Engine(golden_scene(d))
    b = Engine(golden_scene(d))
    a.step(123)
    for _ in range(123):
        b.step(1)
    assert a.x.tobytes() == b.x.tobytes() and a.v.tobytes() == b.v.tobytes()


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_large_block_against_oracle(precision):
    """Full-size property check beyond the golden sizes: 42^3-cell excited
    block (984,438 springs), 20 Verlet steps, GPU vs the C oracle (itself
    pinned to the reference): bitwise in fp64, 1e-4 in fp32."""
    import oracle as orc
    from paper_2207_09334_b200.model import scene_arrays
    scene = L.excite(L.block_scene(42), seed=11)
    eng = Engine(scene, precision=precision)
    eng.step(20)
    ref = orc.OracleEngine(scene_arrays(scene), integrator="verlet", mode="parallel-det", threads=8)
    ref.step(20)
    if precision == "f64":
        assert eng.x.tobytes() == ref.x.tobytes()
        assert eng.v.tobytes() == ref.v.tobytes()
    else:
        disp = np.abs(ref.x - scene.x).max()
        err = np.abs(eng.x - ref.x).max()
        assert err / np.abs(ref.x).max() <= FP32_TOL
        assert err / disp <= 1e-3     # displacement-relative error


def test_full_size_10m_cube():
    """BASELINE configs[3] at full size (block_scene(91): 9,896,068 springs,
    the bench workload): fp64 bitwise vs the C oracle (pinned to the
    reference) after 3 Verlet steps; fp32 vs fp64 after 100 substeps within
    1e-3 of the displacement; total momentum of the free cube conserved."""
    import oracle as orc
    from paper_2207_09334_b200.model import scene_arrays
    scene = L.excite(L.block_scene(91), seed=11)
    arr = scene_arrays(scene)
    e64 = Engine(scene, precision="f64")
    e64.step(3)
    ref = orc.OracleEngine(arr, integrator="verlet", mode="parallel-det", threads=16)
    ref.step(3)
    assert e64.x.tobytes() == ref.x.tobytes()
    assert e64.v.tobytes() == ref.v.tobytes()
    del ref
    e64.step(97)
    e32 = Engine(scene, precision="f32")
    e32.step(100)
    disp = np.abs(e64.x - scene.x).max()
    assert np.abs(e32.x - e64.x).max() <= 1e-3 * disp
    p0 = (arr.m[:, None] * scene.v).sum(axis=0)
    for eng, tol in ((e64, 1e-9), (e32, 1e-5)):
        p1 = (arr.m[:, None] * eng.v).sum(axis=0)
        assert np.linalg.norm(p1 - p0) <= tol * np.linalg.norm(p0)


def test_momentum_conserved_free_block():
    """tests/test_acceptance.py:169-195 momentum criterion on the GPU."""
    scene = L.excite(L.block_scene(9), seed=11)
    eng = Engine(scene)
    p0 = (eng.m[:, None] * scene.v).sum(axis=0)
    eng.step(1000)
    p1 = (eng.m[:, None] * eng.v).sum(axis=0)
    assert np.linalg.norm(p1 - p0) / np.linalg.norm(p0) <= 1e-9


@pytest.mark.parametrize("fmt,kernels", [("0", (6,)), ("explicit", (0, 1))])
@pytest.mark.parametrize("case", ["crawler_verlet", "block9_excited_verlet", "cantilever_10x2x2_verlet",
                                  "random_order_verlet", "block3_excited_rk4", "crawler_rk4", "random_order_euler"])
def test_fp32_general_tile_formats(case, fmt, kernels, monkeypatch):
    """The fp32 formats for tiles with more than 64 distinct spring records --
    inline records on tile_lean_kernel (6; SS_TILE_DICT=0 forces it) and the
    older explicit format (SS_TILE_DICT=explicit) -- within the fp32
    tolerance of the reference."""
    monkeypatch.setenv("SS_TILE_DICT", fmt)
    run_case_fp32(case, "tile")
    d, eng = run_engine(case, "tile", precision="f32")
    assert eng.info()["tile_kernel"] in kernels


def test_fp32_inline_records_on_a_jittered_population(monkeypatch):
    """48 crawlers whose every spring has its own stiffness (every tile
    overflows the dictionary): the inline format by default, within the fp32
    tolerance of the fp64 engine over 2000 steps, groups and contact
    included, and the same bits whatever the batching."""
    from paper_2207_09334_b200 import crawler_scene, replicate
    batch = replicate(crawler_scene(), 48, jitter=1e-6, seed=3)
    batch.k = batch.k * (1.0 + 1e-6 * np.arange(batch.k.size))
    monkeypatch.setenv("SS_RESIDENT", "0")                  # (the resident kernel has its own image)
    e64 = Engine(batch, precision="f64")
    e32 = Engine(batch, precision="f32")
    assert e64.info()["tile_kernel"] == 5 and e32.info()["tile_kernel"] == 6
    e64.step(2000)
    e32.step(1000)
    e32.step(1000)
    span = np.abs(e64.x - batch.x).max()
    assert np.abs(e32.x - e64.x).max() <= 1e-3 * span


@pytest.mark.parametrize("integrator", ["verlet", "rk4"])
def test_fp32_inline_rest_vectors_equal_the_dictionary(integrator, monkeypatch):
    """The fp32 inline format forms each rest vector D = fp32(X0_o - X0_m)
    on the device from the staged fp64 X0; the dictionary stores the same
    value.  With one lane per mass both formats sum the same incidences in
    the same order, so steps and forces agree bit for bit."""
    scene = L.excite(L.block_scene(12), seed=11)
    monkeypatch.setenv("SS_RESIDENT", "0")
    monkeypatch.setenv("SS_LEAN_LANES", "1")
    comp = Engine(scene, integrator=integrator, precision="f32")
    monkeypatch.setenv("SS_TILE_DICT", "0")
    inl = Engine(scene, integrator=integrator, precision="f32")
    assert comp.info()["tile_kernel"] == 2 and inl.info()["tile_kernel"] == 6
    comp.step(40)
    inl.step(40)
    assert inl.x.tobytes() == comp.x.tobytes() and inl.v.tobytes() == comp.v.tobytes()
    rng = np.random.default_rng(5)
    xp = scene.x + 1e-3 * rng.standard_normal(scene.x.shape)
    assert inl.forces(xp, scene.v, 0.0).tobytes() == comp.forces(xp, scene.v, 0.0).tobytes()


@pytest.mark.parametrize("integrator", ["verlet", "rk4"])
def test_fp32_dictionary_with_rest_vectors_from_x0(integrator, monkeypatch):
    """Walkers jittered in place (positions off the lattice, shared materials):
    a rest-vector-keyed dictionary overflows, a (k, k*l0, group) one does not
    (tile_kernel 7: D formed from the staged X0).  Same D and the same order as
    the inline records, so the two formats agree bit for bit; within the fp32
    tolerance of the fp64 engine over 2000 steps (groups and contact)."""
    from paper_2207_09334_b200 import crawler_scene, replicate
    batch = replicate(crawler_scene(), 96, jitter=1e-6, seed=3)
    monkeypatch.setenv("SS_RESIDENT", "0")
    x0 = Engine(batch, integrator=integrator, precision="f32")
    monkeypatch.setenv("SS_TILE_DICT", "0")
    inl = Engine(batch, integrator=integrator, precision="f32")
    monkeypatch.delenv("SS_TILE_DICT")
    assert x0.info()["tile_kernel"] == 7 and inl.info()["tile_kernel"] == 6
    x0.step(100)
    inl.step(100)
    assert x0.x.tobytes() == inl.x.tobytes() and x0.v.tobytes() == inl.v.tobytes()
    rng = np.random.default_rng(9)
    xp = batch.x + 1e-3 * rng.standard_normal(batch.x.shape)
    assert x0.forces(xp, batch.v, 0.0).tobytes() == inl.forces(xp, batch.v, 0.0).tobytes()
    e64 = Engine(batch, integrator=integrator, precision="f64")
    e64.step(2000 if integrator == "verlet" else 500)
    x0.step(1900 if integrator == "verlet" else 400)
    span = np.abs(e64.x - batch.x).max()
    assert np.abs(x0.x - e64.x).max() <= 1e-3 * span


@pytest.mark.parametrize("lanes", ["1", "2"])
def test_degenerate_springs_in_tiled_fp32(lanes, monkeypatch):
    """Coincident endpoints in a multi-tile fp32 scene: the spring is skipped
    and counted once per step by either lean-kernel shape (one or two lanes
    per mass), like the reference (_kernels.py:58-60)."""
    monkeypatch.setenv("SS_LEAN_LANES", lanes)
    scene = L.block_scene(12)
    s0 = 5000
    i, j = int(scene.si[s0]), int(scene.sj[s0])
    scene.x[j] = scene.x[i]                   # spring s0 now has L = 0
    eng = Engine(scene, integrator="verlet", precision="f32")
    assert eng.info()["tile_kernel"] == 2
    eng.step(1)
    assert eng.degenerate_springs == 1
    assert np.isfinite(eng.x).all()
