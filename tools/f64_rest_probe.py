import sys
sys.path.insert(0, "/root/repo")
from paper_2207_09334_b200 import Engine, lattice as L
sc = L.block_scene(91)
e = Engine(sc, integrator="verlet", precision="f64")
e.step(10)
e.step(5)
