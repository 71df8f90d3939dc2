import sys
sys.path.insert(0, "/root/repo")
from paper_2207_09334_b200 import Engine, lattice as L
e = Engine(L.beam_lattice(length=4.0), integrator="verlet", precision="f32")
e.step(50)
