"""The reference's Fig-9-style benchmark grid through the drop-in harness
(paper_2207_09334_b200.benchmark.profile): 100 Verlet steps per point, wall
clock around Engine.step, fp32 and fp64 (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_09334_b200 import benchmark as B
for prec in ("f64", "f32"):
    reps = B.profile(spring_counts=(10_000, 100_000, 1_000_000, 10_000_000), integrators=("verlet",),
                     precision=prec)
    print(prec)
    print(B.profile_table(reps), flush=True)
