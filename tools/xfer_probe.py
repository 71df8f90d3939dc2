"""Host<->device transfer rates of the state path (dev tool): pinned DMA
ceiling (torch), and ss_set_state / ss_get_state of one (N,3) f64 array."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2207_09334_b200 import Engine, lattice as L, _lib

def best(f, n=7):
    f(); ts = []
    for _ in range(n):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return min(ts)

nb = 778688 * 24
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True); d = torch.empty(nb, dtype=torch.uint8, device="cuda")
pg = torch.empty(nb, dtype=torch.uint8)
out = {"pinned_h2d_GBs": nb / best(lambda: d.copy_(h, non_blocking=True)) / 1e9,
       "pinned_d2h_GBs": nb / best(lambda: h.copy_(d, non_blocking=True)) / 1e9,
       "pageable_h2d_GBs": nb / best(lambda: d.copy_(pg)) / 1e9,
       "host_memcpy_GBs": nb / best(lambda: pg.copy_(h)) / 1e9}
sc = L.excite(L.block_scene(91), seed=11)
eng = Engine(sc, precision="f64")
x = np.ascontiguousarray(sc.x); lib = _lib.lib()
out["set_x_GBs"] = nb / best(lambda: _lib.check(lib.ss_set_state(eng._h, _lib.dptr(x), None, None))) / 1e9
y = np.empty_like(x)
out["get_x_GBs"] = nb / best(lambda: _lib.check(lib.ss_get_state(eng._h, _lib.dptr(y), None, None, None))) / 1e9
print(os.environ.get("SS_CHUNK_MB", "4"), {k: round(v, 1) for k, v in out.items()}, flush=True)
