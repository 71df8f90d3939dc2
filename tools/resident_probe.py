"""One-tile scenes on the CTA-resident kernel: what a step costs with and
without actuation groups, contact planes and gravity (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, crawler_scene, lattice as L


def variant(name):
    sc = crawler_scene()
    if "nogroups" in name:
        sc.group = None
        sc.groups = {}
    if "noplanes" in name:
        sc.planes = []
    if "nogravity" in name:
        sc.gravity = (0.0, 0.0, 0.0)
    return sc


for name in ("full", "nogroups", "noplanes", "nogroups_noplanes", "nogroups_noplanes_nogravity", "block3"):
    for prec in ("f32", "f64"):
        sc = L.excite(L.block_scene(3), seed=11) if name == "block3" else variant(name)
        e = Engine(sc, integrator="verlet", precision=prec)
        e.step(100)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        n = 20000
        a.record(st); e.step_async(n); b.record(st); b.synchronize(); e.synchronize()
        print(json.dumps({"scene": name, "prec": prec, "us_step": round(a.elapsed_time(b) * 1e3 / n, 3),
                          "masses": sc.mass_count}), flush=True)
        e.close()
