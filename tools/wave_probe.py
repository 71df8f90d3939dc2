"""One-wave cubes (n = 30, 42): per-substep time from CUDA events, with and
without programmatic dependent launch and the persistent kernel (dev tool;
run under ncu for the kernels' own durations)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L
cells = [int(c) for c in os.environ.get("CELLS", "30,42").split(",")]
modes = {"default": {}, "nopdl": {"SS_PDL": "0"}, "persist": {"SS_PERSIST": "1"}}
if os.environ.get("MODES"):
    modes = {k: v for k, v in modes.items() if k in os.environ["MODES"].split(",")}
for n in cells:
    sc = L.excite(L.block_scene(n), seed=11)
    for prec in os.environ.get("PRECS", "f64,f32").split(","):
        row = {"cells": n, "prec": prec, "springs": sc.spring_count}
        for mode, env in modes.items():
            for k in ("SS_PDL", "SS_PERSIST"):
                os.environ.pop(k, None)
            os.environ.update(env)
            e = Engine(sc, integrator="verlet", precision=prec)
            st = torch.cuda.ExternalStream(e.stream_ptr)
            k = int(os.environ.get("STEPS", "200"))
            for _ in range(4):                                      # (a batch shape seen twice is replayed as a graph)
                e.step_async(k)
            e.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st); e.step_async(k); b.record(st); b.synchronize(); e.synchronize()
            row[mode] = round(a.elapsed_time(b) * 1e3 / k, 2)
            row["tiles"] = e.info()["tile_count"]
            e.close()
        print(json.dumps(row), flush=True)
