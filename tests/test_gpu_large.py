"""Parity at the full bench sizes (BASELINE.json configs[3] and configs[4]).

* configs[4], the 399,812,428-spring cube: the oracle (serial mode, pinned
  to the reference) against the fp64 engine on the whole cube, and the
  x-slab sharded path (two shards, fused peer-memory exchange) against that
  engine -- all bitwise -- plus total momentum.
* configs[3], the 9,896,068-spring cube: the fp32 production mode against
  the fp64 engine (bitwise the reference, test_gpu_parity.py) over 1000
  substeps, within the stated 1e-4 relative position tolerance.

SS_TEST_400M_CELLS shrinks the configs[4] cube for a quicker run.
"""

import os

import numpy as np
import pytest

from paper_2207_09334_b200 import Engine
from paper_2207_09334_b200 import lattice as L
from paper_2207_09334_b200.model import scene_arrays
from paper_2207_09334_b200.sharded import ShardGroup

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4


@pytest.mark.timeout(1800)
def test_configs4_oracle_engine_and_shards_bitwise():
    import oracle as orc
    cells = int(os.environ.get("SS_TEST_400M_CELLS", "313"))
    full = L.excite(L.block_scene(cells), seed=11)
    assert full.spring_count == L.block_springs(cells)
    steps = 2
    one = Engine(full, precision="f64")
    one.step(steps)
    x1, v1 = one.x.copy(), one.v.copy()
    one.close()
    ref = orc.OracleEngine(scene_arrays(full), integrator="verlet")
    ref.step(steps)
    assert ref.x.tobytes() == x1.tobytes() and ref.v.tobytes() == v1.tobytes()
    del ref
    grp = ShardGroup(cells, 2, precision="f64", v_global=full.v, transport="p2p")
    grp.step(steps)
    assert grp.positions().tobytes() == x1.tobytes()
    assert grp.velocities().tobytes() == v1.tobytes()
    # a free cube keeps its momentum (masses equal, no external force)
    p0 = full.v.sum(axis=0)
    assert np.abs(v1.sum(axis=0) - p0).max() <= 1e-9 * np.abs(p0).max() * full.mass_count ** 0.5


@pytest.mark.timeout(900)
def test_configs3_fp32_within_tolerance_over_1000_substeps():
    full = L.excite(L.block_scene(91), seed=11)
    e64 = Engine(full, precision="f64")
    e32 = Engine(full, precision="f32")
    for _ in range(10):
        e64.step(100)
        e32.step(100)
    x64, x32 = e64.x, e32.x
    err = np.abs(x32 - x64).max() / np.abs(x64).max()
    assert err <= FP32_TOL, err
    disp = np.abs(x64 - full.x).max()
    assert np.abs(x32 - x64).max() <= 1e-3 * disp
