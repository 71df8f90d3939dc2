"""Would CUDA graphs remove the per-launch floor of mid-size scenes?  Capture
one batch of substeps on the engine stream and replay it (timing only: the
replayed launches reuse their captured step numbers) (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
for n in (20, 30, 42):
    sc = L.excite(L.block_scene(n), seed=11)
    for prec in ("f64", "f32"):
        e = Engine(sc, integrator="verlet", precision=prec)
        e.step_async(20); e.synchronize()
        st = torch.cuda.ExternalStream(e.stream_ptr)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        k = 100
        a.record(st); e.step_async(k); b.record(st); b.synchronize(); e.synchronize()
        plain = a.elapsed_time(b) * 1e3 / k
        row = {"cells": n, "prec": prec, "plain_us": round(plain, 2)}
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(st):
                g.capture_begin()
                e.step_async(k)
                g.capture_end()
            e.synchronize()
            g.replay(); torch.cuda.synchronize()
            a.record(st); g.replay(); b.record(st); b.synchronize()
            row["graph_us"] = round(a.elapsed_time(b) * 1e3 / k, 2)
        except Exception as exc:
            row["graph_error"] = repr(exc)[:200]
        print(json.dumps(row), flush=True)
        try:
            e.close()
        except Exception:
            pass
