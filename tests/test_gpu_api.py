"""Engine API behaviour on the GPU, against the reference's hand-derived oracles
(the known-answer tests of reference tests/test_engine.py:38-437, restated)."""

import math
import threading

import numpy as np
import pytest

from paper_2207_09334_b200 import (ActuationGroup, ContactPlane, DivergenceError, Engine, Scene,
                                   contact_floor, contact_force, simulate, spring_force,
                                   total_force)

pytestmark = pytest.mark.gpu


def drop(dt=0.01, m=1.0):
    sc = Scene(dt=dt)
    sc.add_mass((0.0, 0.0, 0.0), m=m)
    return sc


def axial(dt, u0=0.5, k=1.0, m=1.0):
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=dt)
    a = sc.add_mass((0.0, 0.0, 0.0), fixed=True)
    b = sc.add_mass((1.0 + u0, 0.0, 0.0), m=m)
    sc.add_spring(a, b, k=k, l0=1.0)
    return sc, b


# ---------------------------------------------------------- scalar oracles

def test_spring_force_kats():
    np.testing.assert_allclose(spring_force((0, 0, 0), (2, 0, 0), 100.0, 1.0), [100, 0, 0])
    np.testing.assert_allclose(spring_force((0, 0, 0), (0.5, 0, 0), 100.0, 1.0), [-50, 0, 0])
    fi = spring_force((0.2, -0.4, 1.0), (1.1, 0.3, -0.2), 37.0, 0.8)
    fj = spring_force((1.1, 0.3, -0.2), (0.2, -0.4, 1.0), 37.0, 0.8)
    np.testing.assert_array_equal(fi, -fj)
    np.testing.assert_array_equal(spring_force((1, 1, 1), (1, 1, 1), 1e4, 1.0), np.zeros(3))


def test_contact_force_kats():
    pl = ContactPlane(normal=(0.0, 1.0, 0.0), offset=0.0, penalty=1e5, friction=0.5)
    np.testing.assert_array_equal(contact_force((0, 0.1, 0), (0, -1, 0), 0.1, pl, 1e-4), np.zeros(3))
    np.testing.assert_allclose(contact_force((0, -0.01, 0), (0, 0, 0), 0.1, pl, 1e-4), [0, 1000, 0])
    np.testing.assert_allclose(contact_force((0, -0.01, 0), (2.0, 0, 0), 10.0, pl, 1e-4), [-500, 1000, 0])
    np.testing.assert_allclose(contact_force((0, -0.01, 0), (0.001, 0, 0), 0.1, pl, 1.0), [-0.0001, 1000, 0])


# ----------------------------------------------------------------- device

def test_degenerate_spring_counted_not_faulted():
    sc = Scene(gravity=(0.0, 0.0, 0.0))
    sc.add_mass((0, 0, 0))
    sc.add_mass((0, 0, 0))
    sc.add_spring(0, 1, k=100.0, l0=1.0)
    eng = Engine(sc, integrator="euler")
    eng.step(3)
    assert eng.degenerate_springs == 3
    np.testing.assert_array_equal(eng.v, np.zeros((2, 3)))


def test_total_force_kats():
    sc = Scene()
    sc.add_mass((5.0, 2.0, 1.0), m=0.1)
    np.testing.assert_allclose(total_force(sc, 0), [0.0, -0.981, 0.0])
    sc = Scene(gravity=(0.0, 0.0, 0.0))
    sc.add_mass((0, 0, 0), f_ext=(1.0, 2.0, 3.0))
    np.testing.assert_allclose(total_force(sc, 0), [1.0, 2.0, 3.0])
    sc = Scene()
    a = sc.add_mass((0, 1, 0), fixed=True)
    b = sc.add_mass((0, -0.5, 0), m=0.1)
    sc.add_spring(a, b, k=10.0, l0=1.0)
    np.testing.assert_allclose(total_force(sc, b), [0.0, 5.0 - 0.981, 0.0])


def test_sliding_block_decelerates():
    sc = Scene(planes=[contact_floor(penalty=1e6, friction=0.3)], dt=1e-4)
    sc.add_mass((0.0, -1e-5, 0.0), m=0.1, v=(1.0, 0.0, 0.0))
    eng = Engine(sc, integrator="euler")
    eng.step(2000)
    assert eng.v[0, 0] < 1.0


def test_euler_kats():
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=0.1)
    sc.add_mass((0, 0, 0), v=(1.0, 0.0, 0.0))
    eng = Engine(sc, integrator="euler")
    eng.step()
    np.testing.assert_allclose(eng.x[0], [0.1, 0, 0])
    eng = Engine(drop(dt=0.01), integrator="euler")
    eng.step()
    assert eng.x[0, 1] == 0.0
    assert eng.v[0, 1] == pytest.approx(-0.0981)
    sc = Scene()
    sc.add_mass((1.0, 2.0, 3.0), fixed=True, f_ext=(1e6, 0, 0))
    eng = Engine(sc, integrator="euler")
    eng.step(10)
    np.testing.assert_array_equal(eng.x[0], [1.0, 2.0, 3.0])
    np.testing.assert_array_equal(eng.v[0], np.zeros(3))
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=0.1, damping=0.1)
    sc.add_mass((0, 0, 0), v=(1.0, 0.0, 0.0))
    eng = Engine(sc, integrator="euler")
    eng.step()
    assert eng.v[0, 0] == pytest.approx(0.9)


def test_verlet_kats():
    eng = Engine(drop(dt=0.01), integrator="verlet")
    assert eng.state.prev_positions is None
    eng.step()
    assert eng.x[0, 1] == pytest.approx(-4.905e-4)
    assert eng.state.prev_positions is not None
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=1.0)
    sc.add_mass((1.0, 0.0, 0.0))
    eng = Engine(sc, integrator="verlet")
    eng.x_prev = np.array([[0.9, 0.0, 0.0]])            # host write-through
    eng.step()
    assert eng.x[0, 0] == pytest.approx(1.1)
    eng = Engine(drop(dt=0.01), integrator="verlet")
    eng.step(100)
    assert eng.t == pytest.approx(1.0)
    assert eng.x[0, 1] == pytest.approx(-0.5 * 9.81 * eng.t ** 2, abs=1e-10)


def test_verlet_velocity_is_central_difference():
    sc, b = axial(dt=0.01)
    eng = Engine(sc, integrator="verlet")
    eng.step(5)
    replay = Engine(sc, integrator="verlet")
    xs = [replay.x.copy()]
    for _ in range(5):
        replay.step()
        xs.append(replay.x.copy())
    central = (xs[5] - xs[3]) / (2 * 0.01)
    np.testing.assert_allclose(eng.v[b], central[b], rtol=0, atol=0)


def test_verlet_damped_form_decays():
    sc, b = axial(dt=0.001, u0=0.5)
    sc.damping = 0.01
    eng = Engine(sc, integrator="verlet")
    eng.step(2000)
    assert abs(eng.x[b, 0] - 1.0) < 0.5


def test_rk4_kats():
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=0.1)
    sc.add_mass((0, 0, 0), v=(1.0, 0.0, 0.0))
    eng = Engine(sc, integrator="rk4")
    eng.step()
    np.testing.assert_allclose(eng.x[0], [0.1, 0.0, 0.0])
    eng = Engine(drop(dt=0.02), integrator="rk4")
    eng.step(50)
    assert eng.x[0, 1] == pytest.approx(-0.5 * 9.81, abs=1e-12)
    sc, b = axial(dt=0.01)
    eng = Engine(sc, integrator="rk4")
    eng.step(628)
    assert abs(eng.x[b, 0] - (1.0 + 0.5 * math.cos(6.28))) < 1e-8
    sc, _ = axial(dt=0.01, u0=0.4)
    eng = Engine(sc, integrator="rk4")
    eng.step(50)
    np.testing.assert_array_equal(eng.x[0], [0.0, 0.0, 0.0])


def test_time_is_step_count_times_dt():
    eng = Engine(drop(dt=0.1), integrator="euler")
    for n in range(1, 6):
        eng.step()
        assert eng.t == n * 0.1 and eng.n == n


def test_divergence_reports_mass_and_step():
    sc, b = axial(dt=10.0, k=1e4, m=0.01)
    eng = Engine(sc, integrator="euler")
    with pytest.raises(DivergenceError) as err:
        eng.step(10000)
    assert err.value.mass_id == b and err.value.step > 0


def test_anchor_bit_identical_over_run():
    sc = Scene()
    a = sc.add_mass((0.1, 0.2, 0.3), fixed=True)
    b = sc.add_mass((0.1, -0.9, 0.3), m=0.1)
    sc.add_spring(a, b, k=1000.0)
    eng = Engine(sc, integrator="verlet")
    eng.step(500)
    assert eng.x[a].tobytes() == np.array(sc.masses[a].x).tobytes()


def test_actuation():
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=1e-3)
    a = sc.add_mass((0, 0, 0), fixed=True)
    b = sc.add_mass((1, 0, 0), m=0.1)
    sc.add_group(ActuationGroup("muscle", amplitude=0.1, frequency=5.0))
    sc.add_spring(a, b, k=100.0, group="muscle")
    res = simulate(sc, 1.0, traces=[b], integrator="verlet")
    x = res.positions[b][:, 0]
    assert x.max() > 1.02 and x.min() < 0.98
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=1e-3, damping=0.05)
    a = sc.add_mass((0, 0, 0), fixed=True)
    b = sc.add_mass((1, 0, 0), m=0.1)
    sc.add_group(ActuationGroup("grow", mode="constant-expansion", amplitude=0.2))
    sc.add_spring(a, b, k=100.0, group="grow")
    eng = Engine(sc, integrator="verlet")
    eng.step(5000)
    assert eng.x[b, 0] == pytest.approx(1.2, abs=1e-3)


def test_simulate_sampling_rules(tmp_path):
    res = simulate(drop(), 0.0, traces=[0], integrator="euler")
    assert res.engine.n == 0 and len(res.times) == 1
    res = simulate(drop(dt=1e-3), 1.0, traces=[0], integrator="verlet")
    assert res.engine.x[0, 1] == pytest.approx(-4.905, abs=1e-3)
    res = simulate(drop(dt=0.01), 0.05, traces=[0], integrator="verlet")
    assert res.engine.n == 5
    np.testing.assert_allclose(res.times, [0.0, 0.01, 0.02, 0.03, 0.04])
    res = simulate(drop(dt=0.01), 0.1, traces=[0], integrator="euler", sample_every=5)
    np.testing.assert_allclose(res.times, [0.0, 0.05, 0.1])
    sc = drop(dt=0.01)
    first = simulate(sc, 0.05, traces=[0], integrator="euler")
    second = simulate(sc, 0.05, traces=[0], engine=first.engine)
    assert second.times[0] == pytest.approx(0.06) and second.engine.n == 10
    res = simulate(drop(dt=0.01), 0.03, traces=[0], integrator="euler")
    path = tmp_path / "trace.csv"
    res.write_csv(path)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == "t,0.x,0.y,0.z,epe,gpe,ke,total" and len(lines) == 5
    assert float(lines[2].split(",")[2]) == res.positions[0][1, 1]


def test_commands_and_pause_resume():
    eng = Engine(drop(dt=0.01), integrator="euler")
    eng.post_command({"op": "set-damping", "value": 0.5})
    eng.step()
    assert eng.damping == 0.5
    sc = drop(dt=0.01)
    eng = Engine(sc, integrator="euler")
    eng.post_command({"op": "stop"})
    assert simulate(sc, 1.0, engine=eng).engine.n == 1
    eng = Engine(sc, integrator="euler")
    eng.post_command({"op": "pause"})
    eng.step()
    assert eng.paused
    done = threading.Event()

    def finish():
        simulate(sc, 0.05, engine=eng)
        done.set()

    th = threading.Thread(target=finish)
    th.start()
    assert not done.wait(0.1)
    eng.post_command({"op": "resume"})
    assert done.wait(10.0)
    th.join()
    assert eng.n == 6
    eng = Engine(drop(), integrator="euler")
    eng.post_command({"op": "warp-reality"})
    eng.step()
    assert eng.command_errors and "warp-reality" in eng.command_errors[0]


def test_momentum_isolated_pair():
    sc = Scene(gravity=(0.0, 0.0, 0.0))
    sc.add_mass((0.0, 0.0, 0.0), m=0.1)
    sc.add_mass((1.2, 0.0, 0.0), m=0.1)
    sc.add_spring(0, 1, k=10000.0, l0=1.0)
    eng = Engine(sc, integrator="euler")
    p0 = (eng.m[:, None] * eng.v).sum(axis=0)
    for _ in range(50):
        f = eng.forces(eng.x, eng.v, eng.t)
        eng.step()
    p1 = (eng.m[:, None] * eng.v).sum(axis=0)
    assert np.abs(f.sum(axis=0)).max() <= 1e-9 * max(np.abs(f).sum(), 1.0)
    np.testing.assert_allclose(p1, p0, atol=1e-9 * 2400)


def test_host_inplace_edits_reach_the_device():
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=0.1)
    sc.add_mass((0.0, 0.0, 0.0))
    eng = Engine(sc, integrator="euler")
    eng.v[0, 0] = 2.0                 # in-place edit of the host mirror
    eng.f_ext[0] = (0.0, 1.0, 0.0)
    eng.set_external_force(0, (0.0, 1.0, 0.0))
    eng.step()
    assert eng.x[0, 0] == pytest.approx(0.2)
    assert eng.v[0, 1] == pytest.approx(1.0)


@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_device_sampling_matches_host_sampling(integrator, precision):
    """simulate() with on-device sampling (ss_step_sampled) against the
    reference-style host path (step per sampling chunk, download, numpy
    energy_breakdown): identical sample times and positions; energies
    bitwise in fp64 (the device restates numpy's pairwise sums), to 1e-12 in
    fp32 (its fp64 reconstruction of a sampled x_prev may round differently)."""
    import paper_2207_09334_b200.engine as E
    from paper_2207_09334_b200 import crawler_scene
    out = {}
    for device in (True, False):
        E.DEVICE_SAMPLING = device
        try:
            sc = crawler_scene()
            res = simulate(sc, 0.02, traces=[0, 7, 19], integrator=integrator, sample_every=7,
                           precision=precision)
        finally:
            E.DEVICE_SAMPLING = True
        out[device] = res
    a, b = out[True], out[False]
    np.testing.assert_array_equal(a.times, b.times)
    for i in (0, 7, 19):
        if precision == "f64":
            assert a.positions[i].tobytes() == b.positions[i].tobytes()
        else:   # fp32 Verlet samples x_prev = X0 + (r - u): same value, fp64 rounding path may differ
            np.testing.assert_allclose(a.positions[i], b.positions[i], rtol=1e-14, atol=1e-16)
    if precision == "f64":
        assert a.energies.tobytes() == b.energies.tobytes()
    else:
        np.testing.assert_allclose(a.energies, b.energies, rtol=1e-12, atol=1e-15)
    assert a.engine.n == b.engine.n


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("integrator", ["verlet", "euler"])
def test_persistent_small_scene_stepping_is_bitwise_identical(precision, integrator, monkeypatch):
    """The opt-in cooperative persistent stepping (SS_PERSIST=1; the resident
    kernel off) against back-to-back launches, actuation and contact
    included: the same bits in fp64; in fp32 the launches split each mass's
    incidences over two lanes on a scene this small (a different summation
    order), so agreement is to fp32 rounding."""
    from paper_2207_09334_b200 import crawler_scene
    monkeypatch.setenv("SS_RESIDENT", "0")
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("SS_PERSIST", flag)
        eng = Engine(crawler_scene(), integrator=integrator, precision=precision)
        eng.set_damping(2e-4)
        eng.step(777)
        out.append((eng.x.copy(), eng.v.copy(), eng.n))
    if precision == "f64":
        assert out[0][0].tobytes() == out[1][0].tobytes()
        assert out[0][1].tobytes() == out[1][1].tobytes()
    else:
        assert np.abs(out[0][0] - out[1][0]).max() <= 1e-4 * np.abs(out[0][0]).max()
    assert out[0][2] == out[1][2] == 777


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_steering_snapshot_from_device(precision):
    """Engine.snapshot (service.py:378-389): decimated positions bitwise equal
    to the host mirror, energies equal to the host formulas at the mirror
    (bitwise in fp64); the message keeps the reference's layout."""
    from paper_2207_09334_b200 import crawler_scene, replicate
    batch = replicate(crawler_scene(), 8, jitter=1e-6, seed=1)      # gravity, contact, 2 actuation groups
    eng = Engine(batch, integrator="verlet", precision=precision)
    eng.step(777)
    ids, pos, en = eng.snapshot(decimate=3)
    assert ids.tolist() == list(range(0, eng.mass_count, 3))
    assert pos.tobytes() == np.ascontiguousarray(eng.x[ids]).tobytes()
    ref = eng.energies(x=eng.x, v=eng.v)                  # host path: numpy at the downloaded state
    for got, want in zip(en, ref):
        if precision == "f64":
            assert got == want
        else:
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
    msg = eng.snapshot_message(decimate=5, throughput=1.0)
    assert list(msg) == ["type", "t", "n", "positions", "energies", "throughput"]
    assert msg["n"] == 777 and msg["positions"][1][0] == 5 and len(msg["energies"]) == 3


@pytest.mark.parametrize("integrator", ["verlet", "euler"])
def test_resident_kernel_matches_per_step_launches(integrator, monkeypatch):
    """One-tile scenes run the CTA-resident kernel (resident.cuh) for whole
    batches; fp64 is bitwise the per-step launches (SS_RESIDENT=0), fp32
    agrees to rounding (its summation order differs)."""
    from paper_2207_09334_b200 import crawler_scene, replicate
    batch = replicate(crawler_scene(), 12, jitter=1e-6, seed=2)     # 240 masses, contact, 2 groups
    out = {}
    for prec in ("f64", "f32"):
        for res in ("1", "0"):
            monkeypatch.setenv("SS_RESIDENT", res)
            eng = Engine(batch, integrator=integrator, precision=prec)
            eng.set_damping(1e-4)
            eng.step(1)
            eng.step(1500)
            eng.x_prev                                              # noqa: B018  (mirror refresh)
            out[prec, res] = (eng.x.copy(), eng.v.copy(), eng.n)
            eng.close()
    assert out["f64", "1"][0].tobytes() == out["f64", "0"][0].tobytes()
    assert out["f64", "1"][1].tobytes() == out["f64", "0"][1].tobytes()
    assert out["f64", "1"][2] == out["f64", "0"][2] == 1501
    span = np.abs(out["f64", "0"][0] - batch.x).max()
    assert np.abs(out["f32", "1"][0] - out["f32", "0"][0]).max() <= 1e-3 * span


def test_engines_release_their_device_memory():
    """Creating and destroying engines (all kernels: resident, tiled, with
    staging buffers, sampling and snapshots) does not leak device memory."""
    import torch
    from paper_2207_09334_b200 import crawler_scene, lattice as L

    def cycle():
        for prec in ("f32", "f64"):
            for sc in (crawler_scene(), L.excite(L.block_scene(10), seed=1)):
                e = Engine(sc, precision=prec)
                e.step(20)
                e.x = e.x                                       # host round trip through the staging buffers
                e.step(3)
                e.snapshot(decimate=7)
                e.close()

    cycle()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(5):
        cycle()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 8 << 20, (free0, free1)


def test_cluster_resident_fp32_matches_per_step_launches(monkeypatch):
    """fp32 scenes of 2-8 tiles run one thread-block cluster for a whole batch
    (positions in shared memory, halos through distributed shared memory):
    same physics as one launch per step to fp32 rounding, same divergence
    step and mass."""
    from paper_2207_09334_b200 import crawler_scene, lattice as L, replicate
    for scene in (L.beam_lattice(length=4.0), replicate(crawler_scene(), 64, jitter=1e-6, seed=4)):
        out = {}
        for res in ("8", "0"):
            monkeypatch.setenv("SS_RESIDENT", res)
            eng = Engine(scene, integrator="verlet", precision="f32")
            eng.step(3)
            eng.step(2000)
            out[res] = eng.x.copy()
            eng.close()
        assert np.abs(out["8"] - out["0"]).max() <= 1e-4 * np.abs(out["0"]).max()   # the fp32 tolerance
    # divergence inside a cluster batch: the reference's step and lowest mass
    blown = L.excite(L.block_scene(9), seed=11)
    blown.dt = 0.05
    got = {}
    for res in ("8", "0"):
        monkeypatch.setenv("SS_RESIDENT", res)
        eng = Engine(blown, integrator="euler", precision="f32")
        with pytest.raises(DivergenceError) as err:
            eng.step(10000)
        got[res] = (err.value.mass_id, err.value.step, eng.n)
        eng.close()
    assert got["8"][1:] == got["0"][1:]


@pytest.mark.parametrize("integrator", ["verlet", "euler"])
def test_cluster_resident_fp64_is_bitwise_the_launches(integrator, monkeypatch):
    """fp64 scenes of 2-16 tiles run one thread-block cluster, one lane per
    mass adding in list order (resident.cuh): bitwise the per-step launches
    of tile_f64_kernel and the reference's order, including the divergence
    step and mass, and the 4/8-lane variants."""
    from paper_2207_09334_b200 import crawler_scene, lattice as L, replicate
    for scene in (L.beam_lattice(length=4.0), replicate(crawler_scene(), 64, jitter=1e-6, seed=4)):
        out = {}
        for res, g in (("16", ""), ("0", ""), ("16", "4")):
            monkeypatch.setenv("SS_RESIDENT", res)
            monkeypatch.setenv("SS_RESIDENT_G", g)
            eng = Engine(scene, integrator=integrator, precision="f64")
            eng.set_damping(1e-4)
            eng.step(3)
            eng.step(1500)
            out[res, g] = (eng.x.tobytes(), eng.v.tobytes(), eng.n)
            eng.close()
        assert out["16", ""] == out["0", ""] == out["16", "4"]
    monkeypatch.setenv("SS_RESIDENT_G", "")
    blown = L.excite(L.block_scene(9), seed=11)
    blown.dt = 0.05
    got = {}
    for res in ("16", "0"):
        monkeypatch.setenv("SS_RESIDENT", res)
        eng = Engine(blown, integrator=integrator, precision="f64")
        with pytest.raises(DivergenceError) as err:
            eng.step(10000)
        got[res] = (err.value.mass_id, err.value.step, eng.n, eng.x.tobytes())
        eng.close()
    assert got["16"] == got["0"]


def test_command_posted_mid_batch_lands_within_the_batch():
    """The reference drains the command queue before every step
    (engine.py:366-370).  A command posted by another thread while one long
    step(N) runs must take effect inside that batch (within ~two drain
    chunks), not N steps late."""
    from paper_2207_09334_b200 import lattice as L
    scene = L.excite(L.block_scene(20), seed=4)
    a = Engine(scene, integrator="verlet", precision="f64")
    b = Engine(scene, integrator="verlet", precision="f64")
    a.step(20)                      # measured step time sizes the drain chunks
    b.step(20)
    steps = max(4000, int(0.25 / max(a._step_s, 1e-7)))      # a batch of ~0.25 s
    seen = {}

    def post():
        import time as _t
        _t.sleep(0.05)
        a.post_command({"op": "set-gravity", "value": [0.0, -9.81, 0.0]})
        seen["posted"] = True
    th = threading.Thread(target=post)
    th.start()
    a.step(steps)
    th.join()
    b.step(steps)
    assert seen.get("posted") and np.allclose(a.gravity, [0.0, -9.81, 0.0])
    # gravity acted for part of the batch: the centre of mass fell
    drop_a = float(b.x[:, 1].mean() - a.x[:, 1].mean())
    assert drop_a > 0.0
    # and not from the very first step (it was posted 50 ms into the batch)
    full = 0.5 * 9.81 * (steps * scene.dt) ** 2
    assert drop_a < full


def test_divergence_behind_an_async_batch_is_not_dropped():
    """A divergence found while another call settles asynchronously
    enqueued steps is raised by the next step (never silently continued)."""
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=1.0)
    a = sc.add_mass((0.0, 0.0, 0.0))
    b = sc.add_mass((1.0, 0.0, 0.0))
    sc.add_spring(a, b, k=1e6, l0=0.5)      # dt far too large: blows up
    eng = Engine(sc, integrator="euler")
    ref = Engine(sc, integrator="euler")
    with pytest.raises(DivergenceError) as want:
        ref.step(2000)
    eng.step_async(2000)
    _ = eng.x                               # settles the batch behind this read
    with pytest.raises(DivergenceError) as err:
        eng.step(1)
    assert (err.value.mass_id, err.value.step) == (want.value.mass_id, want.value.step)
    assert eng.n == ref.n


def test_kept_f_ext_reference_edits_reach_the_device():
    """f_ext is a live array (the reference's forces() reads it every step):
    an edit through a reference kept across steps takes effect."""
    sc = Scene(gravity=(0.0, 0.0, 0.0), dt=1e-3)
    sc.add_mass((0.0, 0.0, 0.0), m=2.0)
    eng = Engine(sc, integrator="euler")
    fe = eng.f_ext
    eng.step(10)
    fe[0] = (4.0, 0.0, 0.0)
    eng.step(10)
    # v = (F/m) * 10 dt after the edit
    assert eng.v[0, 0] == pytest.approx(4.0 / 2.0 * 10 * 1e-3, rel=1e-12)
    with pytest.raises(ValueError):
        eng.m[0] = 1.0                      # masses are part of the device state


def test_gpe_datum_change_reaches_device_sampling():
    sc = Scene(gravity=(0.0, -9.81, 0.0), dt=1e-3)
    sc.add_mass((0.0, 1.0, 0.0), m=2.0, fixed=True)
    eng = Engine(sc, integrator="euler")
    r0 = simulate(sc, 0.005, engine=eng)
    eng.gpe_datum = eng.gpe_datum - 1.0
    r1 = simulate(sc, 0.005, engine=eng)
    assert r1.energies[-1, 1] == pytest.approx(r0.energies[-1, 1] + 2.0 * 9.81 * 1.0, rel=1e-12)
    assert eng.energies()[1] == pytest.approx(r1.energies[-1, 1], rel=1e-12)


@pytest.mark.parametrize("precision", ["f32", "f64"])
@pytest.mark.parametrize("scene", ["crawler", "cube9", "cube20"])
def test_results_do_not_depend_on_batching(precision, scene):
    """step(1) x N, uneven batches and step(N) give the same bits in both
    precisions (reference tests/test_service.py's idle-viewer check: a viewer
    that splits the run into batches changes nothing).  Covers the
    CTA-resident kernel (crawler), the resident cluster (cube9) and the
    per-step tile kernels (cube20)."""
    from paper_2207_09334_b200 import crawler_scene, lattice as L
    make = {"crawler": crawler_scene, "cube9": lambda: L.excite(L.block_scene(9), seed=11),
            "cube20": lambda: L.excite(L.block_scene(20), seed=11)}[scene]
    runs = []
    for plan in ([60], [1] * 60, [7, 1, 13, 2, 37]):
        eng = Engine(make(), integrator="verlet", precision=precision)
        for c in plan:
            eng.step(c)
        runs.append((eng.x.tobytes(), eng.v.tobytes()))
        eng.close()
    assert runs[0] == runs[1] == runs[2]


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_page_locked_state_arrays(precision):
    """State assigned from page-locked arrays (one DMA) and from ordinary
    numpy arrays (staged) gives the same bits; readbacks land in pooled
    page-locked buffers and stay valid while the caller holds them."""
    from paper_2207_09334_b200 import lattice as L, pinned_copy
    from paper_2207_09334_b200 import _lib
    sc = L.excite(L.block_scene(12), seed=11)
    out = []
    for pin in (False, True):
        eng = Engine(sc, integrator="verlet", precision=precision)
        eng.step(5)
        x, v, xp = eng.x.copy(), eng.v.copy(), eng.x_prev.copy()
        x[:, 0] += 1e-3
        if pin:
            x, v, xp = pinned_copy(x), pinned_copy(v), pinned_copy(xp)
        held = []
        for _ in range(3):
            eng.x, eng.v, eng.x_prev = x, v, xp
            eng.step(7)
            held.append(eng.x)                            # a readback the caller keeps
        assert all(h.tobytes() == held[0].tobytes() for h in held)
        out.append((held[-1].tobytes(), eng.v.tobytes(), eng.x_prev.tobytes()))
        eng.close()
    assert out[0] == out[1]
    a = _lib.pinned_empty((1000, 3))
    a[:] = 1.5
    assert a.flags.c_contiguous and float(a.sum()) == 4500.0


def _graph_pair(make, monkeypatch, **kw):
    """The same scene in two engines: batches replayed as CUDA graphs
    (default) and launched one by one (SS_GRAPH=0)."""
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SS_GRAPH", flag)
        out.append(Engine(make(), **kw))
    monkeypatch.delenv("SS_GRAPH")
    return out


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
def test_graph_replays_are_bitwise_the_launches(precision, integrator, monkeypatch):
    """Repeated batches of one shape are captured once and replayed as CUDA
    graphs (step numbers from a device word, actuation tables re-uploaded
    per batch); a parameter change between batches makes a new graph.  The
    replays give the bits of one launch per substep, in both precisions."""
    from paper_2207_09334_b200 import crawler_scene, lattice as L, replicate
    monkeypatch.setenv("SS_RESIDENT", "0")
    def general():                                          # every tile on the inline general-graph format
        c = L.excite(L.block_scene(14), seed=5)
        c.k = c.k * (1.0 + 1e-7 * np.arange(c.k.size))
        return c
    for make in (lambda: L.excite(L.block_scene(20), seed=3),
                 lambda: replicate(crawler_scene(), 48, jitter=1e-6, seed=2),     # 2 groups, contact
                 general):
        g, n = _graph_pair(make, monkeypatch, integrator=integrator, precision=precision)
        for eng in (g, n):
            for b in range(6):
                if b == 3:
                    eng.set_damping(2e-3)                   # new launch parameters: a new graph
                eng.step(25)
            eng.step(7)
            eng.step(25)
        assert g.x.tobytes() == n.x.tobytes() and g.v.tobytes() == n.v.tobytes()
        assert g.n == n.n == 182 and g.t == n.t
        assert g.launch_count == n.launch_count
        g.close()
        n.close()


def test_graph_replays_report_divergence_like_the_launches(monkeypatch):
    """A step that diverges inside a replayed batch: the same DivergenceError
    (step and lowest mass) and the same state as one launch per substep."""
    from paper_2207_09334_b200 import lattice as L
    monkeypatch.setenv("SS_RESIDENT", "0")
    blown = L.excite(L.block_scene(20), seed=11)
    blown.dt = 0.004
    got = []
    for eng in _graph_pair(lambda: blown, monkeypatch, integrator="euler", precision="f64"):
        eng.step(10)
        with pytest.raises(DivergenceError) as err:
            for _ in range(200):
                eng.step(10)
        got.append((err.value.mass_id, err.value.step, eng.n, eng.x.tobytes()))
        eng.close()
    assert got[0] == got[1]
    assert got[0][1] > 30                                   # (diverged inside a replayed batch)


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("integrator", ["verlet", "rk4"])
def test_pdl_autotune_leaves_no_trace(precision, integrator, monkeypatch):
    """Engine creation times both PDL choices on mid-size scenes (one to eight
    tiles per SM) on the engine's own buffers: afterwards the state, step
    counter, launch and degenerate counters are the untuned engine's, and so
    are the results."""
    from paper_2207_09334_b200 import lattice as L
    scene = L.excite(L.block_scene(40), seed=4)
    engines = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SS_AUTOTUNE", flag)
        engines.append(Engine(scene, integrator=integrator, precision=precision))
    monkeypatch.delenv("SS_AUTOTUNE")
    tuned, plain = engines
    assert 148 <= tuned.info()["tile_count"] <= 8 * 148
    for e in engines:
        assert e.n == 0 and e.launch_count == 0 and e.degenerate_springs == 0
        assert e.x.tobytes() == scene.x.tobytes()
        e.step(30)
        e.step(30)
    assert tuned.x.tobytes() == plain.x.tobytes() and tuned.v.tobytes() == plain.v.tobytes()
    assert tuned.n == plain.n == 60 and tuned.launch_count == plain.launch_count
    for e in engines:
        e.close()
