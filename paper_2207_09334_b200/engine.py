"""Drop-in ``Engine`` / ``simulate`` for the B200 relaxation loop.

Call-compatible with the reference (pkg/src/springsim/engine.py): the same
constructor ``Engine(scene, integrator="verlet", mode="serial", threads=None)``,
the same methods (``step``, ``forces``, ``total_force``, ``energies``,
``state``, setters, command queue) and the same public attributes
(``x, v, x_prev, m, f_ext, t, n, dt, damping, gravity, integrator, mode,
threads, gpe_datum, degenerate_springs, paused, stopped, command_errors``).

What changes underneath: the per-step work (engine.py:261-354, 366-381) runs
as hand-written sm_100a kernels behind the C ABI of
``include/springsim_b200.h`` (bound in :mod:`._lib`).  There is no CPU
fallback — constructing an Engine without the built library or without a
GPU raises.

Two extra keyword arguments select the arithmetic and the incidence layout:

* ``precision="f64"`` (default) — validation mode, bitwise identical to the
  reference's serial mode; ``"f32"`` — production mode (displacement form,
  1e-4 relative over short horizons).
* ``layout="auto" | "csr" | "ell"`` — device incidence structure.

Host mirrors.  ``x, v, x_prev, f_ext`` read as numpy arrays downloaded
lazily after each batch of steps; callers may edit them in place or assign
them (reference code does both: tests/test_engine.py:170, service.py:442),
and any array handed out is re-uploaded before the next step.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import queue
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .model import CONSTANT_EXPANSION, ActuationGroup, actuation_scale, scene_arrays
from .traces import TraceSeries

SERIAL = "serial"
PARALLEL = "parallel"
PARALLEL_DET = "parallel-det"
EXEC_MODES = (SERIAL, PARALLEL, PARALLEL_DET)

EULER = "euler"
VERLET = "verlet"
RK4 = "rk4"
INTEGRATORS = (EULER, VERLET, RK4)

PRECISIONS = ("f64", "f32")
LAYOUTS = {"auto": _lib.SS_LAYOUT_AUTO, "csr": _lib.SS_LAYOUT_CSR, "ell": _lib.SS_LAYOUT_ELL,
           "tile": _lib.SS_LAYOUT_TILE}

DEGENERATE_LENGTH = 1e-12          # _kernels.py:23
_INTEG = {EULER: _lib.SS_EULER, VERLET: _lib.SS_VERLET, RK4: _lib.SS_RK4}


class DivergenceError(RuntimeError):
    """Non-finite position or velocity; the run is halted (engine.py:44-52)."""

    MESSAGE = ("simulation diverged at step {step}: mass {mass_id} has a "
               "non-finite position or velocity (try a smaller dt)")

    def __init__(self, mass_id: int, step: int):
        super().__init__(self.MESSAGE.format(step=step, mass_id=mass_id))
        self.mass_id, self.step = mass_id, step


def spring_force(x_i, x_j, k: float, l0: float) -> np.ndarray:
    """Force on mass i from one spring; the force on j is its exact negation
    (engine.py:55-65).  ``np.linalg.norm`` of the 1-D offset, as the
    reference, so the length rounds the same way; coincident endpoints
    (L < 1e-12) give zero force."""
    d = np.subtract(x_j, x_i, dtype=np.float64)
    length = float(np.linalg.norm(d))
    return np.zeros(3) if length < DEGENERATE_LENGTH else (k * (length - l0) / length) * d


def _friction(v, normal, f_n: float, mu: float, m: float, dt: float):
    """Clamped Coulomb friction opposing the tangential velocity: at most
    |v_t| m / dt, so one step can stop the sliding but never reverse it."""
    v_t = v - (v @ normal) * normal
    speed = float(np.linalg.norm(v_t))
    if not (mu > 0.0 and speed > 1e-15):
        return None
    return (min(mu * f_n, speed * m / dt) / speed) * v_t


def _penetration(x, plane, normal) -> float:
    """How far x lies inside the plane's solid side (<= 0: outside)."""
    return plane.offset - x @ normal


def contact_force(x, v, m: float, plane, dt: float) -> np.ndarray:
    """Penalty normal force plus friction of one plane on one mass
    (engine.py:68-89); zero outside the half-space."""
    x, v, normal = (np.asarray(a, dtype=np.float64) for a in (x, v, plane.normal))
    depth = _penetration(x, plane, normal)
    if depth <= 0.0:
        return np.zeros(3)
    push = plane.penalty * depth
    tangential = _friction(v, normal, push, plane.friction, m, dt)
    return push * normal if tangential is None else push * normal - tangential


@dataclass
class EngineState:
    """Snapshot between steps (engine.py:135-145)."""

    positions: np.ndarray
    velocities: np.ndarray
    prev_positions: np.ndarray | None
    t: float
    n: int
    integrator: str
    mode: str


def _elastic(x, si, sj, k, l0_eff) -> float:
    """1/2 sum k (L - l0_eff)^2 over the springs (L by np.linalg.norm, as the reference)."""
    if not si.size:
        return 0.0
    stretch = np.linalg.norm(x[sj] - x[si], axis=1) - l0_eff
    return float(0.5 * np.sum(k * stretch ** 2))


def _gravitational(x, m, gravity, datum: float) -> float:
    """sum m |g| (height above datum), height measured against gravity; 0 without gravity."""
    g = np.asarray(gravity, dtype=np.float64)
    g_mag = float(np.linalg.norm(g))
    if not g_mag > 0.0:
        return 0.0
    return float(np.sum(m * g_mag * (x @ (-g / g_mag) - datum)))


def _kinetic(v, m) -> float:
    return float(0.5 * np.sum(m * np.einsum("ij,ij->i", v, v)))


def energy_breakdown(x, v, m, si, sj, k, l0_eff, gravity, datum: float):
    """(elastic, gravitational, kinetic) energy of a raw state on the host
    (engine.py:148-170, same formulas and reductions); overflow reads as inf
    (the stepper's divergence check reports the blow-up)."""
    with np.errstate(over="ignore", invalid="ignore"):
        return _elastic(x, si, sj, k, l0_eff), _gravitational(x, m, gravity, datum), _kinetic(v, m)


PINNED_MIRROR_BYTES = 256 << 20      # state readbacks up to this size land in page-locked memory


def _host_state(n: int) -> np.ndarray:
    """A fresh (n, 3) f64 host array for a readback: page-locked (one DMA,
    pooled, no first-touch page faults) up to PINNED_MIRROR_BYTES, else
    ordinary memory."""
    if n * 24 <= PINNED_MIRROR_BYTES:
        try:
            return _lib.pinned_empty((n, 3))
        except _lib.CudaError:           # page-locked memory exhausted
            pass
    return np.empty((n, 3))


class _Mirror:
    """Lazy host copy of one (N,3) device array with lend/upload tracking."""

    __slots__ = ("arr", "stale", "lent")

    def __init__(self, arr):
        self.arr = arr
        self.stale = False
        self.lent = False


class Engine:
    """GPU engine, call-compatible with reference engine.py:173-466."""

    _divergence_error = DivergenceError      # (reference_backend raises the host package's class)

    def __init__(self, scene, integrator: str = VERLET, mode: str = SERIAL,
                 threads: int | None = None, *, precision: str = "f64",
                 layout: str = "auto", device: int = 0):
        if integrator not in INTEGRATORS:
            raise ValueError(f"unknown integrator {integrator!r}")
        if mode not in EXEC_MODES:
            raise ValueError(f"unknown execution mode {mode!r}")
        if precision not in PRECISIONS:
            raise ValueError(f"unknown precision {precision!r}")
        if layout not in LAYOUTS:
            raise ValueError(f"unknown layout {layout!r}")
        if scene.mass_count == 0:
            raise ValueError("scene has no masses")
        self.integrator = integrator
        self.mode = mode
        self.precision = precision
        self.device = int(device)
        arr = scene_arrays(scene)
        self.dt = float(arr.dt)
        self.damping = float(arr.damping)
        self.gravity = np.asarray(arr.gravity, dtype=np.float64)
        self._m = arr.m
        self._m.setflags(write=False)      # masses live in the device state: fixed at construction
        self._fixed = arr.fixed
        self._fixed_idx = np.nonzero(arr.fixed)[0]
        self._si = arr.si
        self._sj = arr.sj
        self._sk = arr.k
        self._l0 = arr.l0
        self._l0_eff = arr.l0.copy()
        self._group_of = arr.group
        self._groups: dict[str, dict] = {}
        for gi, (label, mode_, amp, freq, phase) in enumerate(arr.group_params):
            self._groups[label] = {"indices": np.nonzero(arr.group == gi)[0].astype(np.int64),
                                   "mode": mode_, "amplitude": amp, "frequency": freq,
                                   "phase": phase}
        self._planes = arr.planes
        self.paused = False
        self.stopped = False
        self._commands: queue.Queue = queue.Queue()
        self.command_errors: list[str] = []
        self.threads = 1
        if mode != SERIAL:
            available = os.cpu_count() or 1
            self.threads = max(1, min(threads or available, available))
        g_mag = float(np.linalg.norm(self.gravity))
        self._gpe_datum = float((arr.x @ (-self.gravity / g_mag)).min()) if g_mag else 0.0
        self._degenerate_offset = 0
        self._host_prev_nonverlet = None

        self._h = C.c_void_p()
        self._create(arr, LAYOUTS[layout])
        self._x = _Mirror(arr.x)
        self._v = _Mirror(arr.v)
        self._xp = _Mirror(None)
        self._f = _Mirror(arr.f_ext)
        self._f_sent = None                # f_ext as last uploaded (once handed out, edits are watched)
        # seconds per step: sizes the command-drain chunks of long batches;
        # measured after every step() call, first guessed from the size
        self._step_s = 2e-6 + 1e-11 * arr.si.shape[0]

    # ------------------------------------------------------------ plumbing

    def _create(self, arr, layout: int) -> None:
        lib = _lib.lib()
        n, s = arr.x.shape[0], arr.si.shape[0]
        self._keep = keep = {}
        keep["x"] = np.ascontiguousarray(arr.x, dtype=np.float64)
        keep["v"] = np.ascontiguousarray(arr.v, dtype=np.float64)
        keep["m"] = np.ascontiguousarray(arr.m, dtype=np.float64)
        keep["f"] = np.ascontiguousarray(arr.f_ext, dtype=np.float64)
        keep["fixed"] = np.ascontiguousarray(arr.fixed, dtype=np.uint8)
        keep["si"] = np.ascontiguousarray(arr.si, dtype=np.int64)
        keep["sj"] = np.ascontiguousarray(arr.sj, dtype=np.int64)
        keep["k"] = np.ascontiguousarray(arr.k, dtype=np.float64)
        keep["l0"] = np.ascontiguousarray(arr.l0, dtype=np.float64)
        keep["group"] = np.ascontiguousarray(arr.group, dtype=np.int32)
        G = len(arr.group_params)
        keep["gmode"] = np.array([_lib.SS_CONSTANT_EXPANSION if g[1] == CONSTANT_EXPANSION
                                  else _lib.SS_SINUSOID for g in arr.group_params] or [0],
                                 dtype=np.int32)
        keep["gamp"] = np.array([g[2] for g in arr.group_params] or [0.0])
        keep["gfreq"] = np.array([g[3] for g in arr.group_params] or [0.0])
        keep["gphase"] = np.array([g[4] for g in arr.group_params] or [0.0])
        planes = np.array([[*p[0], p[1], p[2], p[3]] for p in arr.planes] or [[0.0] * 6],
                          dtype=np.float64).reshape(-1)
        keep["planes"] = planes
        d = _lib.SceneDesc()
        d.n_masses = n
        d.n_springs = s
        d.x = _lib.dptr(keep["x"])
        d.v = _lib.dptr(keep["v"])
        d.m = _lib.dptr(keep["m"])
        d.f_ext = _lib.dptr(keep["f"])
        d.fixed = _lib.u8ptr(keep["fixed"])
        d.si = _lib.i64ptr(keep["si"])
        d.sj = _lib.i64ptr(keep["sj"])
        d.k = _lib.dptr(keep["k"])
        d.l0 = _lib.dptr(keep["l0"])
        d.group = _lib.i32ptr(keep["group"])
        d.n_groups = G
        d.group_mode = _lib.i32ptr(keep["gmode"])
        d.group_amplitude = _lib.dptr(keep["gamp"])
        d.group_frequency = _lib.dptr(keep["gfreq"])
        d.group_phase = _lib.dptr(keep["gphase"])
        d.n_planes = len(arr.planes)
        d.planes = _lib.dptr(planes)
        for c in range(3):
            d.gravity[c] = float(arr.gravity[c])
        d.dt = self.dt
        d.damping = self.damping
        d.integrator = _INTEG[self.integrator]
        d.precision = _lib.SS_F32 if self.precision == "f32" else _lib.SS_F64
        d.layout = layout
        d.device = self.device
        _lib.check(lib.ss_create(C.byref(d), C.byref(self._h)), "ss_create")
        # the engine copied everything it needs
        for key in ("x", "v", "f", "fixed", "group", "gmode", "gamp", "gfreq", "gphase", "planes"):
            keep.pop(key, None)

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib().ss_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self) -> "Engine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = _lib.Info()
        _lib.check(_lib.lib().ss_get_info(self._h, C.byref(inf)), "ss_get_info")
        return {f: getattr(inf, f) for f, _ in _lib.Info._fields_}

    def _download(self, which: str) -> None:
        """Refresh the host mirror ``which`` ("x", "v" or "x_prev") if stale;
        only that one crosses the bus."""
        lib = _lib.lib()
        n = self.mass_count
        need_x = which == "x" and self._x.stale
        need_v = which == "v" and self._v.stale
        need_p = which == "x_prev" and self._xp.stale and self.integrator == VERLET
        if not (need_x or need_v or need_p):
            return
        has_prev = C.c_int(0)
        x = _host_state(n) if need_x else None
        v = _host_state(n) if need_v else None
        p = _host_state(n) if need_p else None
        _lib.check(lib.ss_get_state(self._h, _lib.dptr(x), _lib.dptr(v), _lib.dptr(p),
                                    C.byref(has_prev)), "ss_get_state")
        if need_x:
            self._x.arr, self._x.stale = x, False
        if need_v:
            self._v.arr, self._v.stale = v, False
        if need_p:
            self._xp.arr = p if has_prev.value else None
            self._xp.stale = False

    def _upload_lent(self) -> None:
        """Push host-side edits (assignments or in-place writes) to the device."""
        lib = _lib.lib()
        x = self._x.arr if self._x.lent else None
        v = self._v.arr if self._v.lent else None
        p = None
        clear_prev = False
        if self.integrator == VERLET and self._xp.lent:
            if self._xp.arr is None:
                clear_prev = True
            else:
                p = self._xp.arr
        if x is not None or v is not None or p is not None:
            x = None if x is None else np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
            v = None if v is None else np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3)
            p = None if p is None else np.ascontiguousarray(p, dtype=np.float64).reshape(-1, 3)
            for a in (x, v, p):
                if a is not None and a.shape[0] != self.mass_count:
                    raise ValueError("state array has the wrong number of masses")
            _lib.check(lib.ss_set_state(self._h, _lib.dptr(x), _lib.dptr(v), _lib.dptr(p)),
                       "ss_set_state")
        if clear_prev:
            _lib.check(lib.ss_clear_prev(self._h), "ss_clear_prev")
        # f_ext is a live array in the reference (forces() reads it every
        # step): once handed out it stays watched, and any change -- through
        # the attribute, a kept reference or set_external_force -- goes down
        if self._f.lent and (self._f_sent is None or not np.array_equal(self._f.arr, self._f_sent)):
            f = np.ascontiguousarray(self._f.arr, dtype=np.float64).reshape(-1, 3)
            _lib.check(lib.ss_set_f_ext(self._h, _lib.dptr(f)), "ss_set_f_ext")
            self._f_sent = f.copy()
        self._x.lent = self._v.lent = self._xp.lent = False

    def _push_params(self) -> None:
        """Scalars the reference reads fresh every step (damping, gravity,
        actuation parameters) go down before each batch."""
        lib = _lib.lib()
        _lib.check(lib.ss_set_damping(self._h, float(self.damping)), "ss_set_damping")
        g = np.ascontiguousarray(self.gravity, dtype=np.float64).reshape(3)
        _lib.check(lib.ss_set_gravity(self._h, _lib.dptr(g)), "ss_set_gravity")
        for gi, g_ in enumerate(self._groups.values()):
            mode = _lib.SS_CONSTANT_EXPANSION if g_["mode"] == CONSTANT_EXPANSION else _lib.SS_SINUSOID
            _lib.check(lib.ss_set_group(self._h, gi, mode, float(g_["amplitude"]),
                                        float(g_["frequency"]), float(g_["phase"])),
                       "ss_set_group")

    def _mark_stepped(self) -> None:
        self._x.stale = self._v.stale = True
        self._x.lent = self._v.lent = False
        if self.integrator == VERLET:
            self._xp.stale = True
            self._xp.lent = False

    # ------------------------------------------------------- state mirrors

    @property
    def x(self) -> np.ndarray:
        self._download("x")
        self._x.lent = True
        return self._x.arr

    @x.setter
    def x(self, value) -> None:
        # like the reference's plain attribute: keep the caller's array (no
        # copy when it is already (N,3) float64); uploaded before the next step
        self._x.arr = np.asarray(value, dtype=np.float64).reshape(-1, 3)
        self._x.stale, self._x.lent = False, True

    @property
    def v(self) -> np.ndarray:
        self._download("v")
        self._v.lent = True
        return self._v.arr

    @v.setter
    def v(self, value) -> None:
        self._v.arr = np.asarray(value, dtype=np.float64).reshape(-1, 3)
        self._v.stale, self._v.lent = False, True

    @property
    def x_prev(self):
        if self.integrator != VERLET:
            return self._host_prev_nonverlet
        self._download("x_prev")
        self._xp.lent = True
        return self._xp.arr

    @x_prev.setter
    def x_prev(self, value) -> None:
        if self.integrator != VERLET:
            self._host_prev_nonverlet = None if value is None else np.array(value, dtype=np.float64)
            return
        self._xp.arr = None if value is None else np.asarray(value, dtype=np.float64).reshape(-1, 3)
        self._xp.stale, self._xp.lent = False, True

    @property
    def m(self) -> np.ndarray:
        """Node masses (read-only: they are part of the device state)."""
        return self._m

    @property
    def gpe_datum(self) -> float:
        return self._gpe_datum

    @gpe_datum.setter
    def gpe_datum(self, value: float) -> None:
        """Height GPE is measured from (engine.py:240-242); every later energy
        sample uses the new datum, as the reference reads it per call."""
        self._gpe_datum = float(value)
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.check(_lib.lib().ss_set_gpe_datum(self._h, self._gpe_datum), "ss_set_gpe_datum")

    @property
    def f_ext(self) -> np.ndarray:
        self._f.lent = True
        return self._f.arr

    @f_ext.setter
    def f_ext(self, value) -> None:
        self._f.arr = np.array(value, dtype=np.float64).reshape(-1, 3)
        self._f.lent = True

    @property
    def t(self) -> float:
        t = C.c_double()
        _lib.check(_lib.lib().ss_get_time(self._h, C.byref(t), None), "ss_get_time")
        return t.value

    @t.setter
    def t(self, value: float) -> None:
        _lib.check(_lib.lib().ss_set_time(self._h, float(value), self.n), "ss_set_time")

    @property
    def n(self) -> int:
        n = C.c_int64()
        _lib.check(_lib.lib().ss_get_time(self._h, None, C.byref(n)), "ss_get_time")
        return n.value

    @n.setter
    def n(self, value: int) -> None:
        _lib.check(_lib.lib().ss_set_time(self._h, self.t, int(value)), "ss_set_time")

    @property
    def degenerate_springs(self) -> int:
        c = C.c_int64()
        _lib.check(_lib.lib().ss_degenerate_count(self._h, C.byref(c)), "ss_degenerate_count")
        return int(c.value) + self._degenerate_offset

    @degenerate_springs.setter
    def degenerate_springs(self, value: int) -> None:
        self._degenerate_offset = 0
        self._degenerate_offset = int(value) - self.degenerate_springs

    @property
    def mass_count(self) -> int:
        return int(self.m.shape[0])

    @property
    def spring_count(self) -> int:
        return int(self._sk.shape[0])

    # ------------------------------------------------------------- forces

    def _rest_lengths(self, t: float) -> np.ndarray:
        """Actuated rest lengths at time t on the host (engine.py:250-259;
        energies of a supplied state only -- the device scales l0 per group
        inside the spring kernels)."""
        for g in self._groups.values():
            signal = ActuationGroup("", g["mode"], g["amplitude"], g["frequency"], g["phase"])
            self._l0_eff[g["indices"]] = self._l0[g["indices"]] * actuation_scale(signal, t)
        return self._l0_eff

    def forces(self, x: np.ndarray, v: np.ndarray, t: float) -> np.ndarray:
        """Total force on every mass at a trial state (engine.py:261-289), on the GPU."""
        self._upload_lent()
        self._push_params()
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
        v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3)
        acc = np.empty_like(x)
        deg = C.c_int64()
        _lib.check(_lib.lib().ss_forces(self._h, _lib.dptr(x), _lib.dptr(v), float(t),
                                        _lib.dptr(acc), C.byref(deg)), "ss_forces")
        return acc

    def total_force(self, mass_id: int) -> np.ndarray:
        return self.forces(self.x, self.v, self.t)[mass_id]

    # ------------------------------------------------------------ stepping

    # A batch longer than this much device time is enqueued in chunks with
    # the command queue drained before each one (the reference drains before
    # every step, engine.py:366-370): the host stays one chunk ahead of the
    # device, so a command posted mid-batch lands within about two chunks.
    COMMAND_LATENCY_S = 2e-3
    MIN_CHUNK_STEPS = 16

    def _chunk_steps(self) -> int:
        return max(self.MIN_CHUNK_STEPS, int(self.COMMAND_LATENCY_S / max(self._step_s, 1e-8)))

    def _raise_step(self, rc: int, res, what: str) -> None:
        if rc == _lib.SS_EDIVERGED:
            raise self._divergence_error(int(res.diverged_mass), int(res.diverged_step))
        _lib.check(rc, what)

    def step(self, count: int = 1) -> None:
        """Advance ``count`` steps (engine.py:366-373).

        Short batches go down as one device batch; long ones in chunks of
        about COMMAND_LATENCY_S of device time, draining queued commands and
        re-reading damping, gravity, f_ext and actuation before each chunk.
        DivergenceError is raised for the first non-finite step, the state
        being the diverged state, as in the reference."""
        if count <= 0:
            return
        lib = _lib.lib()
        res = _lib.StepResult()
        chunk = self._chunk_steps()
        t0 = time.perf_counter()
        if count <= chunk:
            self.drain_commands()
            self._upload_lent()
            self._push_params()
            rc = lib.ss_step(self._h, int(count), C.byref(res))
            self._mark_stepped()
            self._raise_step(rc, res, "ss_step")
        else:
            done = 0
            try:
                while done < count:
                    self.drain_commands()
                    self._upload_lent()
                    self._push_params()
                    k = min(chunk, count - done)
                    rc = lib.ss_step_async(self._h, k)
                    if rc != _lib.SS_OK:
                        self._raise_step(rc, res, "ss_step_async")
                    done += k
                    _lib.check(lib.ss_pending_wait(self._h, chunk), "ss_pending_wait")
            finally:
                self._mark_stepped()
            self._raise_step(lib.ss_sync(self._h, C.byref(res)), res, "ss_sync")
        self._step_s = 0.5 * (self._step_s + (time.perf_counter() - t0) / count)

    def step_sampled(self, count: int, sample_every: int, traces=()):
        """Advance ``count`` steps recording, on the device, the samples
        ``simulate`` takes (engine.py:546-559): after every step whose index
        d (Verlet: n-1, at x_prev with the lagged v; otherwise n) is a
        multiple of ``sample_every``, the traced positions and the energy
        breakdown at t = d*dt.  Returns (times (R,), positions (R, n, 3),
        energies (R, 4)).  One host synchronisation per call."""
        count = int(count)
        sample_every = max(1, int(sample_every))
        ids = np.ascontiguousarray(list(traces), dtype=np.int64)
        if count <= 0:
            return np.zeros(0), np.zeros((0, ids.size, 3)), np.zeros((0, 4))
        self.drain_commands()
        self._upload_lent()
        self._push_params()
        lib = _lib.lib()
        self._energy_setup()
        max_rows = count // sample_every + 2
        times = np.empty(max_rows)
        pos = np.empty((max_rows, max(ids.size, 1), 3))
        en = np.empty((max_rows, 4))
        rows = C.c_int64()
        res = _lib.StepResult()
        rc = lib.ss_step_sampled(self._h, count, sample_every, _lib.i64ptr(ids) if ids.size else None,
                                 int(ids.size), max_rows, _lib.dptr(times), _lib.dptr(pos), _lib.dptr(en),
                                 C.byref(rows), C.byref(res))
        self._mark_stepped()
        if rc == _lib.SS_EDIVERGED:
            raise self._divergence_error(int(res.diverged_mass), int(res.diverged_step))
        _lib.check(rc, "ss_step_sampled")
        r = int(rows.value)
        return times[:r], pos[:r, :ids.size], en[:r]

    def _energy_setup(self) -> None:
        """Spring list for the device energy reduction, uploaded once."""
        if getattr(self, "_energy_ready", False):
            return
        grp = np.ascontiguousarray(self._group_of, dtype=np.int32)
        _lib.check(_lib.lib().ss_energy_setup(self._h, self.spring_count, _lib.i64ptr(self._si),
                                              _lib.i64ptr(self._sj), _lib.dptr(self._sk), _lib.dptr(self._l0),
                                              grp.ctypes.data_as(C.POINTER(C.c_int32)),
                                              float(self.gpe_datum)), "ss_energy_setup")
        self._energy_ready = True

    def snapshot(self, decimate: int = 1, ids=None):
        """Steering snapshot from the device (service.py:378-389): positions
        of every ``decimate``-th mass (or of ``ids``) and (epe, gpe, ke, total)
        at the current state -- ``Engine.energies()`` reduced on the device,
        without downloading the full state.  Returns (ids, positions (n,3),
        energies (4,))."""
        if ids is None:
            if decimate < 1:
                raise ValueError("decimate must be >= 1")
            ids = np.arange(0, self.mass_count, int(decimate), dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        self._upload_lent()
        self._push_params()
        self._energy_setup()
        pos = np.empty((ids.size, 3))
        en = np.empty(4)
        _lib.check(_lib.lib().ss_snapshot(self._h, _lib.i64ptr(ids) if ids.size else None, int(ids.size),
                                          float(self.gpe_datum), _lib.dptr(pos), _lib.dptr(en)), "ss_snapshot")
        return ids, pos, en

    def snapshot_message(self, decimate: int = 1, throughput: float = 0.0) -> dict:
        """The reference steering server's snapshot message (service.py:380-389)
        built from :meth:`snapshot` -- same keys and layout, ready for its
        ``encode_message``."""
        ids, pos, en = self.snapshot(decimate)
        return {"type": "snapshot", "t": self.t, "n": self.n,
                "positions": [[int(i), *map(float, p)] for i, p in zip(ids, pos)],
                "energies": [float(en[0]), float(en[1]), float(en[2])], "throughput": throughput}

    def step_async(self, count: int) -> None:
        """Enqueue ``count`` steps without synchronising (benchmarks)."""
        self._upload_lent()
        self._push_params()
        _lib.check(_lib.lib().ss_step_async(self._h, int(count)), "ss_step_async")
        self._mark_stepped()

    def synchronize(self) -> None:
        res = _lib.StepResult()
        rc = _lib.lib().ss_sync(self._h, C.byref(res))
        if rc == _lib.SS_EDIVERGED:
            raise self._divergence_error(int(res.diverged_mass), int(res.diverged_step))
        _lib.check(rc, "ss_sync")

    @property
    def stream_ptr(self) -> int:
        return int(_lib.lib().ss_stream(self._h) or 0)

    @property
    def launch_count(self) -> int:
        return int(_lib.lib().ss_launch_count(self._h))

    @property
    def state(self) -> EngineState:
        prev = self.x_prev
        return EngineState(positions=self.x.copy(), velocities=self.v.copy(),
                           prev_positions=None if prev is None else prev.copy(),
                           t=self.t, n=self.n, integrator=self.integrator, mode=self.mode)

    def energies(self, x=None, v=None, t=None):
        """(epe, gpe, ke, total) (engine.py:390-398).  At the engine's own
        state the sums are reduced on the device (the reduction simulate()
        samples with; no state download); a supplied state is reduced on the
        host with the reference's formulas."""
        if x is None and v is None and t is None:
            _, _, en = self.snapshot(ids=np.zeros(0, dtype=np.int64))
            return tuple(float(e) for e in en)
        x = self.x if x is None else x
        v = self.v if v is None else v
        t = self.t if t is None else t
        epe, gpe, ke = energy_breakdown(x, v, self.m, self._si, self._sj, self._sk,
                                        self._rest_lengths(t), self.gravity, self.gpe_datum)
        return epe, gpe, ke, epe + gpe + ke

    # ------------------------------------------------------------ commands
    # Setters and the thread-safe command channel (engine.py:402-466).  The
    # engine reads every parameter fresh at the next step boundary.

    def set_external_force(self, mass_id: int, f) -> None:
        self.f_ext[mass_id] = np.asarray(f, dtype=np.float64)

    def set_damping(self, value: float) -> None:
        if not (0.0 <= value < 1.0):
            raise ValueError("damping must be in [0, 1)")
        self.damping = float(value)

    def set_gravity(self, g) -> None:
        self.gravity = np.asarray(g, dtype=np.float64)

    def set_actuation(self, label: str, amplitude=None, frequency=None, phase=None) -> None:
        """Change a group's signal; ``None`` keeps a parameter, |amplitude| < 1."""
        group = self._groups.get(label)
        if group is None:
            raise ValueError(f"unknown actuation group {label!r}")
        if amplitude is not None and not abs(amplitude) < 1.0:
            raise ValueError("|amplitude| must be < 1")
        group.update({key: float(val) for key, val in
                      (("amplitude", amplitude), ("frequency", frequency), ("phase", phase)) if val is not None})

    def post_command(self, command: dict) -> None:
        """Queue a command (any thread); applied at the next step boundary."""
        self._commands.put(dict(command))

    def _queued(self, wait: float):
        """Commands waiting in the channel; the first may be waited for."""
        try:
            yield self._commands.get(timeout=wait) if wait > 0.0 else self._commands.get_nowait()
            while True:
                yield self._commands.get_nowait()
        except queue.Empty:
            return

    def drain_commands(self, wait: float = 0.0) -> None:
        """Apply every queued command; a failing one is reported in
        ``command_errors`` and the rest still apply."""
        for cmd in self._queued(wait):
            error = _try_command(self, cmd)
            if error:
                self.command_errors.append(error)

    def apply_command(self, cmd: dict) -> None:
        handler = _COMMANDS.get(cmd.get("op"))
        if handler is None:
            raise ValueError(f"unknown command op {cmd.get('op')!r}")
        handler(self, cmd)


def _try_command(engine: "Engine", cmd: dict) -> str | None:
    """Apply one command; a failure comes back as "op: reason" (the
    reference keeps stepping and reports through ``command_errors``)."""
    try:
        engine.apply_command(cmd)
    except Exception as exc:
        return f"{cmd.get('op', '?')}: {exc}"
    return None


def _floats(values) -> list[float]:
    return [float(c) for c in values]


# op -> handler(engine, command) (engine.py:448-466)
_COMMANDS = {
    "pause": lambda e, c: setattr(e, "paused", True),
    "resume": lambda e, c: setattr(e, "paused", False),
    "stop": lambda e, c: setattr(e, "stopped", True),
    "set-damping": lambda e, c: e.set_damping(float(c["value"])),
    "set-gravity": lambda e, c: e.set_gravity(_floats(c["value"])),
    "set-external-force": lambda e, c: e.set_external_force(int(c["mass"]), _floats(c["value"])),
    "set-actuation": lambda e, c: e.set_actuation(c["group"], c.get("amplitude"), c.get("frequency"),
                                                  c.get("phase")),
}


def plan(scene, precision: str = "f32") -> dict:
    """Host-only statistics of the tiled device layout of ``scene`` (no GPU needed):
    tile count, halo ratio, foreign-reference fraction, streamed record bytes,
    shared memory per CTA, algorithmic bytes per step."""
    arr = scene_arrays(scene)
    keep = {
        "x": np.ascontiguousarray(arr.x, dtype=np.float64),
        "si": np.ascontiguousarray(arr.si, dtype=np.int64),
        "sj": np.ascontiguousarray(arr.sj, dtype=np.int64),
        "k": np.ascontiguousarray(arr.k, dtype=np.float64),
        "l0": np.ascontiguousarray(arr.l0, dtype=np.float64),
        "group": np.ascontiguousarray(arr.group, dtype=np.int32),
    }
    d = _lib.SceneDesc()
    d.n_masses = keep["x"].shape[0]
    d.n_springs = keep["si"].shape[0]
    d.x = _lib.dptr(keep["x"])
    d.si = _lib.i64ptr(keep["si"])
    d.sj = _lib.i64ptr(keep["sj"])
    d.k = _lib.dptr(keep["k"])
    d.l0 = _lib.dptr(keep["l0"])
    d.group = _lib.i32ptr(keep["group"])
    d.n_groups = len(arr.group_params)
    d.precision = _lib.SS_F32 if precision == "f32" else _lib.SS_F64
    inf = _lib.Info()
    _lib.check(_lib.lib().ss_plan(C.byref(d), C.byref(inf)), "ss_plan")
    return {f: getattr(inf, f) for f, _ in _lib.Info._fields_}


def total_force(scene, mass_id: int, t: float = 0.0, **engine_kwargs) -> np.ndarray:
    """Total force on one mass of a scene in its initial state at time t
    (engine.py:469-473), evaluated by a throw-away Euler engine."""
    with Engine(scene, integrator=EULER, mode=SERIAL, **engine_kwargs) as engine:
        engine.t = t
        return engine.total_force(mass_id)


_ENERGY_COLUMNS = ("epe", "gpe", "ke", "total")


@dataclass
class RunResult:
    """Sampled output of :func:`simulate` (engine.py:476-515): sample times,
    traced positions per mass id (T,3), energies (T,4) in the column order
    epe, gpe, ke, total.  Under Verlet each sample pairs x_prev with the
    central-difference v, one step behind the final engine state."""

    times: np.ndarray
    positions: dict[int, np.ndarray]
    energies: np.ndarray
    engine: Engine = field(repr=False)

    def position_series(self, mass_id: int, axis: int | None = None) -> TraceSeries:
        track = self.positions[mass_id]
        return TraceSeries(self.times, track if axis is None else track[:, axis])

    def energy_series(self, term: str) -> TraceSeries:
        column = {name: c for c, name in enumerate(_ENERGY_COLUMNS)}[term]     # KeyError like the reference
        return TraceSeries(self.times, self.energies[:, column])

    def write_csv(self, path) -> None:
        """t, then x/y/z of every traced mass (ascending id), then the four
        energies; every number with 17 significant digits."""
        ids = sorted(self.positions)
        header = ["t", *(f"{i}.{axis}" for i in ids for axis in "xyz"), *_ENERGY_COLUMNS]
        table = np.column_stack([np.asarray(self.times, dtype=np.float64).reshape(-1, 1),
                                 *(np.asarray(self.positions[i], dtype=np.float64).reshape(-1, 3) for i in ids),
                                 np.asarray(self.energies, dtype=np.float64).reshape(-1, 4)])
        with open(path, "w") as fh:
            fh.write(",".join(header) + "\n")
            fh.writelines(",".join(format(float(c), ".17g") for c in row) + "\n" for row in table)


SAMPLE_SEGMENT_ROWS = 4096          # samples per device segment of simulate()
DEVICE_SAMPLING = True              # False: sample on the host after every chunk (reference-style)


class _Samples:
    """Sample rows of a run: times, traced positions, energy tuples."""

    def __init__(self, traces):
        self.times: list[float] = []
        self.tracks = {mass_id: [] for mass_id in traces}
        self.energies: list = []

    def host(self, engine: Engine, step_index: int, x, v) -> None:
        """One sample of a host-side state (the reference's simulate loop)."""
        t = step_index * engine.dt
        self.times.append(t)
        for mass_id, track in self.tracks.items():
            track.append(x[mass_id].copy())
        self.energies.append(engine.energies(x, v, t))

    def device(self, t_s, p_s, e_s) -> None:
        """Rows recorded on the device by Engine.step_sampled."""
        self.times.extend(float(t) for t in t_s)
        for q, track in enumerate(self.tracks.values()):
            track.extend(p_s[:, q].copy())
        self.energies.extend(tuple(e) for e in e_s)

    def result(self, engine: Engine) -> RunResult:
        return RunResult(times=np.asarray(self.times),
                         positions={mass_id: np.asarray(track) for mass_id, track in self.tracks.items()},
                         energies=np.asarray(self.energies).reshape(-1, 4), engine=engine)


def _steps_to_next_sample(n: int, verlet: bool, every: int) -> int:
    """Steps until the next sampling point: Verlet samples step n-1 (paired
    with x_prev), the others step n, whenever it is a multiple of ``every``."""
    lag = ((n - 1) if verlet else n) % every
    return every - lag if lag else every


def simulate(scene, duration: float, traces=(), integrator: str = VERLET,
             mode: str = SERIAL, threads: int | None = None, sample_every: int = 1,
             engine: Engine | None = None, **engine_kwargs) -> RunResult:
    """Run ``ceil(duration/dt - 1e-9)`` steps sampling traced positions and
    energies (engine.py:518-565): the reference's sampling points, Verlet
    one-step sample lag and pause / resume / stop handling.  With an empty
    command queue the steps and samples run on the device in segments
    (Engine.step_sampled); a queued command drops to one step at a time, as
    the reference drains before every step."""
    if engine is None:
        engine = Engine(scene, integrator=integrator, mode=mode, threads=threads, **engine_kwargs)
    total = max(0, math.ceil(duration / engine.dt - 1e-9))
    verlet = engine.integrator == VERLET
    every = max(1, int(sample_every))
    out = _Samples(traces)
    if engine.n == 0 and not verlet:
        out.host(engine, 0, engine.x, engine.v)
    done = 0
    while done < total and not engine.stopped:
        while engine.paused and not engine.stopped:
            engine.drain_commands(wait=0.02)
        if engine.stopped:
            break
        quiet = engine._commands.empty()
        if DEVICE_SAMPLING and quiet:
            seg = min(total - done, SAMPLE_SEGMENT_ROWS * every)
            out.device(*engine.step_sampled(seg, every, list(out.tracks)))
            done += seg
            continue
        chunk = min(_steps_to_next_sample(engine.n, verlet, every), total - done) if quiet else 1
        engine.step(chunk)
        done += chunk
        sampled = engine.n - 1 if verlet else engine.n
        if sampled % every == 0:
            out.host(engine, sampled, engine.x_prev if verlet else engine.x, engine.v)
    return out.result(engine)
