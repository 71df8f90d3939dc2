"""10M cube at rest, fp64: target for ncu of the validation-mode kernel (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_09334_b200 import Engine, lattice as L
sc = L.block_scene(91)
e = Engine(sc, integrator="verlet", precision="f64")
e.step(10)
e.step(5)
