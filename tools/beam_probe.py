"""40x4x4 beam, 50 fp32 Verlet steps: target for ncu launch timing (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_09334_b200 import Engine, lattice as L
e = Engine(L.beam_lattice(length=4.0), integrator="verlet", precision="f32")
e.step(50)
