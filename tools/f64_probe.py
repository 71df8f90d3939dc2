"""fp64 validation-mode timing on the 10M cube (dev tool): us per substep."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2207_09334_b200 import Engine, lattice as L

cells = int(os.environ.get("CELLS", "91"))
n = int(os.environ.get("NSTEPS", "20"))
scene = L.excite(L.block_scene(cells), seed=11)
eng = Engine(scene, integrator=os.environ.get("INTEG", "verlet"), precision="f64", layout="tile")
st = torch.cuda.ExternalStream(eng.stream_ptr)
eng.step_async(3)
eng.synchronize()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record(st)
eng.step_async(n)
b.record(st)
b.synchronize()
us = a.elapsed_time(b) * 1e3 / n
print(json.dumps(dict(cells=cells, us_per_substep=round(us, 2), springs_per_s=scene.spring_count / (us * 1e-6),
                      info={k: v for k, v in eng.info().items() if isinstance(v, (int, float))})))
