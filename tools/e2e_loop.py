"""Per-iteration timing of the public-API loop (set state, step 100, read x) on the 10M cube;
WITH_TORCH=1 adds a device timeline of one step (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if os.environ.get("WITH_TORCH"):
    import torch
    torch.zeros(1, device="cuda")
from paper_2207_09334_b200 import Engine, lattice as L
sc = L.excite(L.block_scene(91), seed=11)
eng = Engine(sc, integrator="verlet", precision="f32")
eng.step(100)
x, v, xp = eng.x.copy(), eng.v.copy(), eng.x_prev.copy()
for rep in range(3):
    ts = []
    for _ in range(6):
        a = time.perf_counter()
        eng.x = x; eng.v = v; eng.x_prev = xp
        b = time.perf_counter(); eng.step(100); c = time.perf_counter()
        out = eng.x
        d = time.perf_counter()
        ts.append((round((b-a)*1e3,2), round((c-b)*1e3,2), round((d-c)*1e3,2)))
    print(ts, flush=True)

if os.environ.get("WITH_TORCH"):
    # device-side timeline of one public-API step: uploads, kernels, download
    from paper_2207_09334_b200 import _lib
    import ctypes as C
    st = torch.cuda.ExternalStream(eng.stream_ptr)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for _ in range(3):
        eng.x = x; eng.v = v; eng.x_prev = xp
        h0 = time.perf_counter()
        ev[0].record(st)
        eng._upload_lent(); eng._push_params()
        h1 = time.perf_counter()
        ev[1].record(st)
        res = _lib.StepResult()
        for _i in range(100):
            _lib.lib().ss_step_async(eng._h, 1)
        ev[2].record(st)
        h2 = time.perf_counter()
        _lib.lib().ss_sync(eng._h, C.byref(res))
        h3 = time.perf_counter()
        eng._mark_stepped()
        print("host ms: upload", round(1e3 * (h1 - h0), 2), "launch", round(1e3 * (h2 - h1), 2),
              "sync", round(1e3 * (h3 - h2), 2), "| device ms: uploads", round(ev[0].elapsed_time(ev[1]), 2),
              "kernels", round(ev[1].elapsed_time(ev[2]), 2), flush=True)
