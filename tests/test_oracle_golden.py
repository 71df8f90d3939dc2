"""Pin the C oracle to the real reference: byte-for-byte on every golden vector.

The golden fixtures were produced by running the reference itself
(tests/golden/make_golden.py).  If these pass, the oracle is a faithful
restatement of reference engine.py / _kernels.py and can be trusted as the
checker for the GPU path at sizes the reference is too slow for.
"""

import numpy as np
import pytest

from conftest import golden_arrays, golden_cases, load_golden

import oracle as orc


@pytest.mark.parametrize("mode", ["serial", "parallel-det"])
@pytest.mark.parametrize("case", golden_cases())
def test_oracle_matches_reference_bitwise(case, mode):
    d = load_golden(case)
    integ = str(d["integrator"])
    eng = orc.OracleEngine(golden_arrays(d), integrator=integ, mode=mode, threads=4)
    done = 0
    for c in d["checkpoints"]:
        eng.step(int(c) - done)
        done = int(c)
        assert eng.x.tobytes() == d[f"x_{c}"].tobytes(), (case, c, "x")
        assert eng.v.tobytes() == d[f"v_{c}"].tobytes(), (case, c, "v")
        if f"xp_{c}" in d.files:
            assert eng.x_prev.tobytes() == d[f"xp_{c}"].tobytes(), (case, c, "x_prev")
        assert eng.t == float(d[f"t_{c}"])
        assert eng.degenerate_springs == int(d[f"deg_{c}"])


def test_oracle_divergence_names_mass_and_step():
    d = load_golden("divergence_euler")
    eng = orc.OracleEngine(golden_arrays_div(d), integrator="euler")
    with pytest.raises(orc.OracleDiverged) as err:
        eng.step(10000)
    assert err.value.mass_id == int(d["div_mass"])
    assert err.value.step == int(d["div_step"])
    assert eng.x.tobytes() == d["x_div"].tobytes()


def golden_arrays_div(d):
    # divergence fixture stores only inputs (no checkpoints)
    return golden_arrays(d)


def test_oracle_forces_bitwise():
    d = load_golden("forces_block6")
    eng = orc.OracleEngine(golden_arrays(d), integrator="verlet")
    acc = eng.forces(d["px"], d["pv"], 0.0)
    assert acc.tobytes() == d["acc"].tobytes()


def test_oracle_parallel_det_is_thread_count_invariant():
    d = load_golden("block9_excited_verlet")
    outs = []
    for threads in (1, 3, 8):
        eng = orc.OracleEngine(golden_arrays(d), integrator="verlet", mode="parallel-det",
                               threads=threads)
        eng.step(10)
        outs.append(eng.x.tobytes())
    assert outs[0] == outs[1] == outs[2] == d["x_10"].tobytes()
