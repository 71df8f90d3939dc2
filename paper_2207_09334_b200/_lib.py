"""ctypes binding of the C ABI declared in ``include/springsim_b200.h``.

The shared library is built in-tree (``paper_2207_09334_b200/libspringsim_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_2207_09334_b200/csrc``.  There is
no CPU fallback: if the library is missing, importing the engine fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

LIB_NAME = "libspringsim_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

SS_OK, SS_EINVAL, SS_ECUDA, SS_EDIVERGED, SS_ENOMEM, SS_EFALLBACK = 0, 1, 2, 3, 4, 5
SS_EULER, SS_VERLET, SS_RK4 = 0, 1, 2
SS_F64, SS_F32 = 0, 1
SS_LAYOUT_AUTO, SS_LAYOUT_CSR, SS_LAYOUT_ELL, SS_LAYOUT_TILE = 0, 1, 2, 3
SS_SINUSOID, SS_CONSTANT_EXPANSION = 0, 1

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class SceneDesc(C.Structure):
    _fields_ = [
        ("n_masses", C.c_int64), ("n_springs", C.c_int64),
        ("x", _dp), ("v", _dp), ("m", _dp), ("f_ext", _dp), ("fixed", _u8p),
        ("si", _i64p), ("sj", _i64p), ("k", _dp), ("l0", _dp), ("group", _i32p),
        ("n_groups", C.c_int32), ("group_mode", _i32p), ("group_amplitude", _dp),
        ("group_frequency", _dp), ("group_phase", _dp),
        ("n_planes", C.c_int32), ("planes", _dp),
        ("gravity", C.c_double * 3), ("dt", C.c_double), ("damping", C.c_double),
        ("integrator", C.c_int32), ("precision", C.c_int32), ("layout", C.c_int32),
        ("device", C.c_int32),
    ]


class StepResult(C.Structure):
    _fields_ = [("steps_done", C.c_int64), ("n", C.c_int64), ("t", C.c_double),
                ("diverged_mass", C.c_int64), ("diverged_step", C.c_int64)]


class Info(C.Structure):
    _fields_ = [("n_masses", C.c_int64), ("n_springs", C.c_int64),
                ("precision", C.c_int32), ("layout", C.c_int32), ("integrator", C.c_int32),
                ("device", C.c_int32), ("device_bytes", C.c_int64),
                ("algorithmic_bytes_per_step", C.c_double),
                ("ell_width_own", C.c_int32), ("ell_width_ref", C.c_int32),
                ("canonical_order", C.c_int32), ("smem_per_block", C.c_int32),
                ("tile_count", C.c_int64), ("tile_blob_bytes", C.c_int64),
                ("tile_halo_ratio", C.c_double), ("tile_foreign_frac", C.c_double),
                ("tile_kernel", C.c_int32), ("kernel_smem", C.c_int32)]


# Every symbol include/springsim_b200.h declares, with its ctypes signature.
SIGNATURES = {
    "ss_abi_version": (C.c_int, []),
    "ss_last_error": (C.c_char_p, []),
    "ss_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ss_pinned_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "ss_pinned_free": (C.c_int, [C.c_void_p]),
    "ss_create": (C.c_int, [C.POINTER(SceneDesc), C.POINTER(C.c_void_p)]),
    "ss_destroy": (C.c_int, [C.c_void_p]),
    "ss_step": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(StepResult)]),
    "ss_step_async": (C.c_int, [C.c_void_p, C.c_int64]),
    "ss_sync": (C.c_int, [C.c_void_p, C.POINTER(StepResult)]),
    "ss_stream": (C.c_void_p, [C.c_void_p]),
    "ss_forces": (C.c_int, [C.c_void_p, _dp, _dp, C.c_double, _dp, _i64p]),
    "ss_get_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, C.POINTER(C.c_int)]),
    "ss_set_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "ss_clear_prev": (C.c_int, [C.c_void_p]),
    "ss_get_positions": (C.c_int, [C.c_void_p, _dp]),
    "ss_get_time": (C.c_int, [C.c_void_p, _dp, _i64p]),
    "ss_set_time": (C.c_int, [C.c_void_p, C.c_double, C.c_int64]),
    "ss_set_f_ext": (C.c_int, [C.c_void_p, _dp]),
    "ss_set_damping": (C.c_int, [C.c_void_p, C.c_double]),
    "ss_set_gravity": (C.c_int, [C.c_void_p, _dp]),
    "ss_set_group": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_double,
                               C.c_double]),
    "ss_degenerate_count": (C.c_int, [C.c_void_p, _i64p]),
    "ss_get_info": (C.c_int, [C.c_void_p, C.POINTER(Info)]),
    "ss_launch_count": (C.c_int64, [C.c_void_p]),
    "ss_energy_setup": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _i64p, _dp, _dp,
                                  C.POINTER(C.c_int32), C.c_double]),
    "ss_snapshot": (C.c_int, [C.c_void_p, _i64p, C.c_int64, C.c_double, _dp, _dp]),
    "ss_step_sampled": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, _i64p, C.c_int64, C.c_int64,
                                  _dp, _dp, _dp, _i64p, C.POINTER(StepResult)]),
    "ss_plan": (C.c_int, [C.POINTER(SceneDesc), C.POINTER(Info)]),
    "ss_halo_setup": (C.c_int, [C.c_void_p, C.c_int64, _i64p, C.c_int64, _i64p,
                                C.c_int64, _i64p, C.c_int64, _i64p]),
    "ss_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "ss_halo_nccl": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ss_halo_p2p_export": (C.c_int, [C.c_void_p, C.c_char_p]),
    "ss_halo_recv_slots": (C.c_int, [C.c_void_p, C.c_int, _i32p]),
    "ss_halo_p2p_attach": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, _i32p, C.c_int64]),
    "ss_halo_p2p_link": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "ss_step_group": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.POINTER(StepResult),
                              C.POINTER(C.c_int32)]),
    "ss_lattice_box": (C.c_int, [_dp, _dp, C.c_double, C.c_double, C.c_double,
                                 C.c_int64, C.c_int64, _i64p, _i64p, _i64p,
                                 _dp, _i64p, _i64p, _dp, _dp, _i64p]),
    "ss_check_f64_fastpath": (C.c_int, [C.c_int32, _dp, _dp, C.c_int64, _dp, _i32p]),
    "ss_pending_wait": (C.c_int, [C.c_void_p, C.c_int64]),
    "ss_set_gpe_datum": (C.c_int, [C.c_void_p, C.c_double]),
    "ss_doc_render_masses": (C.c_int, [C.c_int64, _dp, _dp, _dp, _dp, _u8p, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_int64)]),
    "ss_doc_render_springs": (C.c_int, [C.c_int64, _i64p, _i64p, _dp, _dp, _i32p, C.POINTER(C.c_char_p),
                                        C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "ss_doc_render": (C.c_int, [C.c_int64, _dp, _dp, _dp, _dp, _u8p, C.c_int64, _i64p, _i64p, _dp, _dp, _i32p,
                                C.POINTER(C.c_char_p), C.c_int32, C.c_char_p, C.c_char_p, C.c_char_p,
                                C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "ss_doc_free_text": (None, [C.c_void_p]),
    "ss_doc_repr": (C.c_int, [C.c_int64, _dp, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "ss_doc_parse": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "ss_doc_info": (C.c_int, [C.c_void_p, _i64p, _i64p, _i32p, _i32p]),
    "ss_doc_key": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_char_p), _i64p, _i64p]),
    "ss_doc_label": (C.c_char_p, [C.c_void_p, C.c_int32]),
    "ss_doc_masses": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _u8p]),
    "ss_doc_springs": (C.c_int, [C.c_void_p, _i64p, _i64p, _dp, _dp, _i32p]),
    "ss_doc_free": (None, [C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


class LibraryMissing(ImportError):
    pass


def lib():
    """The loaded library (loads on first use; raises if it was never built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()' or "
                    "make -C paper_2207_09334_b200/csrc). There is no CPU fallback.")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            if handle.ss_abi_version() != 2:
                raise LibraryMissing("libspringsim_b200.so ABI version mismatch; rebuild it")
            _lib = handle
        return _lib


def last_error() -> str:
    return lib().ss_last_error().decode(errors="replace")


class CudaError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc == SS_OK:
        return
    msg = last_error()
    if rc == SS_EINVAL:
        raise ValueError(msg)
    if rc == SS_ECUDA:
        raise CudaError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"{what}: status {rc}: {msg}")


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def i32ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_i32p)


def u8ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_u8p)


def device_count() -> int:
    c = C.c_int(0)
    rc = lib().ss_device_count(C.byref(c))
    return c.value if rc == SS_OK else 0


# ------------------------------------------------------------ page-locked host arrays
# numpy arrays over cudaHostAlloc'd memory: ss_set_state / ss_get_state move
# them in one DMA (~53 GB/s on the B200 hosts) instead of staging pageable
# memory through pinned chunks (~30 GB/s, bound by host memory traffic).
# Freed blocks go back to a small pool, so steady-state readbacks allocate
# nothing.

_pin_lock = threading.Lock()
_pin_pool: dict = {}                     # nbytes -> [address, ...]
_pin_pooled = 0
PIN_POOL_BYTES = 2 << 30                 # pooled (idle) page-locked bytes kept at most


class _PinnedBlock:
    __slots__ = ("addr", "nbytes")

    def __init__(self, addr: int, nbytes: int):
        self.addr, self.nbytes = addr, nbytes

    def __del__(self):
        global _pin_pooled
        try:
            with _pin_lock:
                if _pin_pooled + self.nbytes <= PIN_POOL_BYTES:
                    _pin_pool.setdefault(self.nbytes, []).append(self.addr)
                    _pin_pooled += self.nbytes
                    return
            lib().ss_pinned_free(C.c_void_p(self.addr))
        except Exception:                # interpreter shutdown
            pass


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised C-contiguous array in page-locked host memory."""
    global _pin_pooled
    dtype = np.dtype(dtype)
    nbytes = max(1, int(np.prod(shape)) * dtype.itemsize)
    addr = None
    with _pin_lock:
        free = _pin_pool.get(nbytes)
        if free:
            addr = free.pop()
            _pin_pooled -= nbytes
    if addr is None:
        p = C.c_void_p()
        check(lib().ss_pinned_alloc(nbytes, C.byref(p)), "ss_pinned_alloc")
        addr = p.value
    buf = (C.c_char * nbytes).from_address(addr)
    buf._ss_block = _PinnedBlock(addr, nbytes)          # lives as long as any view of buf
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def pinned_copy(a) -> np.ndarray:
    """``a`` copied into page-locked host memory."""
    a = np.asarray(a)
    out = pinned_empty(a.shape, a.dtype)
    np.copyto(out, a)
    return out
