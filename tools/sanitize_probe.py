"""compute-sanitizer target: a few substeps of each tiled kernel family on
small scenes (fp64/fp32 compact and inline records, RK4, sharded RK4 and
Verlet).  Run as
  compute-sanitizer --tool memcheck python tools/sanitize_probe.py
  compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2207_09334_b200 import lattice as L  # noqa: E402
from paper_2207_09334_b200.engine import Engine  # noqa: E402
from paper_2207_09334_b200.sharded import ShardGroup, excited_velocities  # noqa: E402


def main():
    cube = L.excite(L.block_scene(12), seed=11)
    rnd = L.excite(L.block_scene(12), seed=11)
    rnd.k = rnd.k * (1.0 + 1e-6 * np.arange(rnd.k.size))       # every tile overflows the dictionary
    os.environ["SS_RESIDENT"] = "0"                               # the tile kernels, not the resident one
    for scene, name in ((cube, "compact"), (rnd, "inline")):
        for prec in ("f64", "f32"):
            for integ in ("verlet", "euler", "rk4"):
                e = Engine(scene, precision=prec, integrator=integ)
                e.step(3)
                assert np.isfinite(e.x).all()
                print(name, prec, integ, e.info()["tile_kernel"], flush=True)
    for integ in ("verlet", "rk4"):
        for transport in ("copy", "p2p"):
            g = ShardGroup(9, 2, precision="f64", v_global=excited_velocities(1000), integrator=integ,
                           transport=transport)
            g.step(3)
            print("shards", integ, transport, flush=True)


if __name__ == "__main__":
    main()
