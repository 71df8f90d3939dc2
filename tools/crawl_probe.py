import os, sys
sys.path.insert(0, "/root/repo")
from paper_2207_09334_b200 import Engine, crawler_scene
prec = os.environ.get("PREC", "f32")
e = Engine(crawler_scene(), integrator="verlet", precision=prec)
e.step(100)
e.step(5000)
