"""Crawler, 5100 Verlet steps: target for ncu captures of the resident kernel (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_09334_b200 import Engine, crawler_scene
prec = os.environ.get("PREC", "f32")
e = Engine(crawler_scene(), integrator="verlet", precision=prec)
e.step(100)
e.step(5000)
