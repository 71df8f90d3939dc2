"""Two shards of the 10M cube in one process, a few steps: target for ncu (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_09334_b200 import lattice as L
from paper_2207_09334_b200.sharded import ShardGroup, excited_velocities
full = L.excite(L.block_scene(91), seed=11)
grp = ShardGroup(91, 2, precision="f32", v_global=excited_velocities(full.mass_count),
                 transport=os.environ.get("TRANSPORT", "p2p"))
grp.step(6)
