"""Add the bench-size topology pins to topology.json (dev container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_topology_big.py

Builds ``springsim.bench.block_scene(42)`` (984,438 springs, configs[1]) and
``block_scene(91)`` (9,896,068 springs, configs[3]) through the REAL
reference object model (13 s and 110 s, ~5 GB) and stores the digest of the
arrays ``Engine.__init__`` freezes (engine.py:192-220) as ``block_42`` /
``block_91``, plus the excited-velocity digest of the bench cube
(tests/test_acceptance.py:75-83, seed 11) as ``excited91_v_sha256``.
The existing keys are kept.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import excited, topo_digest  # noqa: E402  (imports the reference package)
from springsim.bench import block_scene  # noqa: E402


def main():
    path = os.path.join(HERE, "topology.json")
    topo = json.load(open(path))
    topo["block_42"] = topo_digest(block_scene(42))
    print("block_42", topo["block_42"], flush=True)
    ex = excited(91)
    topo["block_91"] = topo_digest(ex)
    topo["excited91_v_sha256"] = hashlib.sha256(
        np.array([m.v for m in ex.masses], dtype=np.float64).tobytes()).hexdigest()
    print("block_91", topo["block_91"], flush=True)
    with open(path, "w") as fh:
        json.dump(topo, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
