"""Where the e2e (host buffers in, positions out) time goes (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_09334_b200 import Engine, lattice as L
from paper_2207_09334_b200 import _lib
import ctypes as C

sc = L.excite(L.block_scene(int(os.environ.get("CELLS", "91"))), seed=11)
eng = Engine(sc, integrator="verlet", precision=os.environ.get("PREC", "f64"))
eng.step(100)
x, v, xp = eng.x.copy(), eng.v.copy(), eng.x_prev.copy()
lib = _lib.lib()
def t(f, n=5):
    f(); ts = []
    for _ in range(n):
        a = time.perf_counter(); f(); ts.append(time.perf_counter() - a)
    return round(1e3 * min(ts), 2)
res = {}
res["set_x_v_xprev_ms"] = t(lambda: _lib.check(lib.ss_set_state(eng._h, _lib.dptr(x), _lib.dptr(v), _lib.dptr(xp))))
res["set_x_ms"] = t(lambda: _lib.check(lib.ss_set_state(eng._h, _lib.dptr(x), None, None)))
res["set_v_ms"] = t(lambda: _lib.check(lib.ss_set_state(eng._h, None, _lib.dptr(v), None)))
out = np.empty_like(x)
res["get_x_ms"] = t(lambda: _lib.check(lib.ss_get_state(eng._h, _lib.dptr(out), None, None, None)))
res["get_xprev_ms"] = t(lambda: _lib.check(lib.ss_get_state(eng._h, None, None, _lib.dptr(out), None)))
st = _lib.StepResult()
res["step100_ms"] = t(lambda: lib.ss_step(eng._h, 100, C.byref(st)))
def api():
    eng.x = x; eng.v = v; eng.x_prev = xp; eng.step(100); _ = eng.x
res["api_e2e_ms"] = t(api)
print(res, flush=True)

# the public-API step, piece by piece
def piece(name, f, acc):
    a = time.perf_counter(); f(); acc[name] = acc.get(name, 0.0) + time.perf_counter() - a
acc = {}
reps = 5
for _ in range(reps):
    eng.x = x; eng.v = v; eng.x_prev = xp
    piece("drain", eng.drain_commands, acc)
    piece("upload_lent", eng._upload_lent, acc)
    piece("push_params", eng._push_params, acc)
    res = _lib.StepResult()
    piece("ss_step", lambda: lib.ss_step(eng._h, 100, C.byref(res)), acc)
    eng._mark_stepped()
    piece("get_x", lambda: eng.x, acc)
print({k: round(1e3 * v / reps, 3) for k, v in acc.items()}, flush=True)
