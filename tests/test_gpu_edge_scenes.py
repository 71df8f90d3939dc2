"""GPU edge scenes against the oracle, fp64 bitwise: no springs at all, one
mass, springs only between fixed masses, a mass whose every spring is
degenerate -- through every layout and integrator, plus on-device sampling
of a spring-less scene (EPE from an empty sum)."""

import os
import sys

import numpy as np
import pytest

from paper_2207_09334_b200 import Engine, simulate
from paper_2207_09334_b200.model import ArrayScene, ContactPlane, scene_arrays

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))

pytestmark = pytest.mark.gpu

FLOOR = [ContactPlane((0.0, 0.0, 1.0), 0.0, 1e4, 0.5)]


def _no_springs():
    rng = np.random.default_rng(3)
    x = rng.uniform(0.0, 1.0, (40, 3))
    x[:5, 2] = -0.01                                    # in contact with the floor
    v = rng.normal(0.0, 0.2, (40, 3))
    fixed = np.zeros(40, dtype=bool)
    fixed[7] = True
    e = np.zeros(0, dtype=np.int64)
    return ArrayScene(x=x, m=0.1, si=e, sj=e, k=np.zeros(0), l0=np.zeros(0), v=v, fixed=fixed,
                      gravity=(0.0, 0.0, -9.81), planes=FLOOR, damping=1e-3)


def _one_mass():
    e = np.zeros(0, dtype=np.int64)
    return ArrayScene(x=[[0.0, 0.0, 0.5]], m=2.0, si=e, sj=e, k=np.zeros(0), l0=np.zeros(0), v=[[0.1, 0.0, 0.0]],
                      gravity=(0.0, 0.0, -9.81), planes=FLOOR)


def _fixed_springs():
    x = np.array([[0.0, 0.0, 0.0], [0.1, 0.0, 0.0], [0.0, 0.1, 0.0], [0.3, 0.3, 0.3]])
    return ArrayScene(x=x, m=0.1, si=[0, 0, 1], sj=[1, 2, 2], k=[1e3, 2e3, 3e3], l0=[0.12, 0.08, 0.15],
                      fixed=[True, True, True, False], gravity=(0.0, 0.0, -9.81))


def _degenerate_star():
    x = np.zeros((5, 3))
    x[1:, 0] = [0.0, 0.0, 0.1, 0.2]                     # masses 1 and 2 coincide with mass 0
    return ArrayScene(x=x, m=0.1, si=[0, 0, 0, 0, 3], sj=[1, 2, 3, 4, 4], k=1e3 * np.ones(5),
                      l0=[0.0, 0.05, 0.1, 0.2, 0.1], gravity=(0.0, 0.0, 0.0), v=np.full((5, 3), 0.01))


SCENES = {"no_springs": _no_springs, "one_mass": _one_mass, "fixed_springs": _fixed_springs,
          "degenerate_star": _degenerate_star}


@pytest.mark.parametrize("integrator", ["verlet", "euler", "rk4"])
@pytest.mark.parametrize("layout", ["auto", "csr", "ell", "tile"])
@pytest.mark.parametrize("name", list(SCENES))
def test_edge_scene_fp64_bitwise(name, layout, integrator, monkeypatch):
    import oracle as orc
    for resident in ("16", "0"):                        # the resident kernel and per-step launches
        monkeypatch.setenv("SS_RESIDENT", resident)
        scene = SCENES[name]()
        eng = Engine(scene, integrator=integrator, precision="f64", layout=layout)
        ref = orc.OracleEngine(scene_arrays(scene), integrator=integrator)
        for count in (1, 30):
            eng.step(count)
            ref.step(count)
            assert eng.x.tobytes() == ref.x.tobytes(), (name, layout, integrator, resident, count)
            assert eng.v.tobytes() == ref.v.tobytes(), (name, layout, integrator, resident, count)
        assert eng.degenerate_springs == ref.degenerate_springs
        eng.close()


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_edge_scene_fp32_and_sampling(precision):
    """The spring-less scene through simulate(): positions traced on the
    device, EPE exactly 0 (an empty sum), the trace of a free-falling mass."""
    scene = _no_springs()
    run = simulate(scene, 0.01, traces=(20,), sample_every=10, precision=precision)
    e = np.asarray(run.energies)
    assert e.shape[1] == 4 and (e[:, 0] == 0.0).all()
    tr = run.position_series(20, axis=2)
    assert len(tr.values) > 5 and np.isfinite(tr.values).all()
