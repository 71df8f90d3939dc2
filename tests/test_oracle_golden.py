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


def _digest(a) -> str:
    import hashlib
    h = hashlib.sha256()
    for arr in (a.x, a.m, a.si, a.sj, a.k, a.l0):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("n", [1, 2, 3, 9, 20, 42, 91])
def test_oracle_lattice_builder_matches_reference(n):
    """oracle_voxel_box (the reference arm's workload builder, a restatement
    of lattice.py:89-136) against the reference's block_scene digests."""
    import json
    import os
    from conftest import GOLDEN
    topo = json.load(open(os.path.join(GOLDEN, "topology.json")))
    a = orc.block_arrays(n)
    assert _digest(a) == topo[f"block_{n}"]


def test_oracle_excite_matches_reference_stream():
    import hashlib
    import json
    import os
    from conftest import GOLDEN
    topo = json.load(open(os.path.join(GOLDEN, "topology.json")))
    a = orc.excite(orc.block_arrays(91), seed=11)
    assert hashlib.sha256(np.ascontiguousarray(a.v).tobytes()).hexdigest() == topo["excited91_v_sha256"]


def test_oracle_box_with_inexact_extent():
    import json
    import os
    from conftest import GOLDEN
    topo = json.load(open(os.path.join(GOLDEN, "topology.json")))
    _, x, si, sj, k, l0 = orc.voxel_box((0, 0, 0), (0.3, 0.2, 0.1), 0.1)
    a = orc.Arrays(x, si, sj, k, l0)
    assert _digest(a) == topo["box_0.3x0.2x0.1"]
