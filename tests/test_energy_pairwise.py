"""The energy reduction restates numpy's pairwise summation (sampling.cuh),
so an fp64 engine's energies are bitwise the reference's energy_breakdown
(engine.py:148-170) at the same state.

CPU: the restatement (and the per-row orders of np.linalg.norm and einsum)
against numpy itself.  GPU: Engine.energies(), snapshots and simulate()'s
on-device samples against the host formulas, bit for bit in fp64."""
import numpy as np
import pytest


def pairwise(a, lo=0, n=None):
    """numpy's pairwise_sum over a[lo:lo+n] (what sampling.cuh restates)."""
    n = len(a) if n is None else n
    if n < 8:
        r = 0.0
        for i in range(n):
            r += a[lo + i]
        return r
    if n <= 128:
        r = [a[lo + j] for j in range(8)]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += a[lo + i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for q in range(i, n):
            res += a[lo + q]
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise(a, lo, n2) + pairwise(a, lo + n2, n - n2)


@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 257, 1000, 4095, 8192, 8193, 65537, 300007])
def test_restatement_is_np_sum(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n)
    assert 0.0 + pairwise(list(a)) == np.sum(a)


def test_signed_zeros_and_row_orders():
    """np.sum of negative zeros is +0 (the 0.0 + pairwise form); the row
    reductions the reference uses: norm(axis=1) sums (d0^2 + d1^2) + d2^2,
    einsum('ij,ij->i') sums (v0^2 + v2^2) + v1^2 (numpy's 2-lane SIMD
    accumulator), x @ up is exact for an axis-aligned up."""
    for n in (1, 7, 8, 200):
        assert np.sum(np.full(n, -0.0)) == 0.0 and not np.signbit(np.sum(np.full(n, -0.0)))
    rng = np.random.default_rng(3)
    d = rng.standard_normal((50000, 3)) * 10.0 ** rng.integers(-3, 3, (50000, 3))
    s = d * d
    assert np.array_equal(np.linalg.norm(d, axis=1), np.sqrt((s[:, 0] + s[:, 1]) + s[:, 2]))
    assert np.array_equal(np.einsum("ij,ij->i", d, d), (s[:, 0] + s[:, 2]) + s[:, 1])
    for g in ((0.0, 0.0, -9.81), (0.0, -9.81, 0.0), (-2.0, 0.0, 0.0)):
        g = np.asarray(g)
        up = -g / float(np.linalg.norm(g))
        assert np.array_equal(d @ up, (d[:, 0] * up[0] + d[:, 1] * up[1]) + d[:, 2] * up[2])


def _host_energies(eng):
    from paper_2207_09334_b200.engine import energy_breakdown
    x, v = eng.x.copy(), eng.v.copy()
    epe, gpe, ke = energy_breakdown(x, v, eng.m, eng._si, eng._sj, eng._sk, eng._rest_lengths(eng.t),
                                    eng.gravity, eng.gpe_datum)
    return epe, gpe, ke, epe + gpe + ke


def _scenes():
    from paper_2207_09334_b200 import crawler_scene, lattice as L, replicate
    yield "crawler_x8", replicate(crawler_scene(), 8, jitter=1e-6, seed=1)     # gravity, 2 groups, contact
    yield "cube20", L.excite(L.block_scene(20), seed=11)                       # 109,260 springs: deep trees
    beam = L.beam_lattice(length=2.0)
    yield "beam20", beam


@pytest.mark.gpu
@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
def test_device_energies_are_bitwise_the_reference_formulas(integrator):
    from paper_2207_09334_b200 import Engine
    for name, sc in _scenes():
        eng = Engine(sc, integrator=integrator, precision="f64")
        eng.gpe_datum = 0.05
        eng.step(123)
        got = eng.energies()
        want = _host_energies(eng)
        assert [g.hex() for g in got] == [w.hex() for w in want], (name, got, want)
        eng.close()


@pytest.mark.gpu
def test_sampled_energies_are_bitwise_the_host_path():
    """simulate(): on-device samples against the host path (one chunk per
    sample, download, numpy) -- identical in fp64."""
    import paper_2207_09334_b200.engine as E
    from paper_2207_09334_b200 import crawler_scene, simulate
    out = {}
    for device in (True, False):
        E.DEVICE_SAMPLING = device
        try:
            out[device] = simulate(crawler_scene(), 0.05, traces=[0, 19], sample_every=13, precision="f64")
        finally:
            E.DEVICE_SAMPLING = True
    assert out[True].energies.tobytes() == out[False].energies.tobytes()


@pytest.mark.gpu
def test_oblique_gravity_agrees_to_rounding():
    """For gravity off the axes the reference's x @ up goes through BLAS gemv
    (its order is the BLAS kernel's); the device sums x.up in index order, so
    GPE agrees to rounding, EPE and KE stay bitwise."""
    from paper_2207_09334_b200 import Engine, crawler_scene
    eng = Engine(crawler_scene(), precision="f64")
    eng.set_gravity((1.0, -9.0, 2.5))
    eng.step(50)
    got, want = eng.energies(), _host_energies(eng)
    assert got[0] == want[0] and got[2] == want[2]
    assert abs(got[1] - want[1]) <= 1e-13 * abs(want[1])
