"""ctypes binding of libb200lobpcg.so (include/b200lobpcg.h).

This is the only place Python touches the native library.  There is no CPU
fallback: if the library or a CUDA device is missing, every call raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import os

_HERE = Path(__file__).resolve().parent
# B2L_LIB_PATH: an A/B build of the same sources (tools/build_variant.py); diagnostic only
LIB_PATH = Path(os.environ.get("B2L_LIB_PATH") or _HERE / "lib" / "libb200lobpcg.so")

_lock = threading.Lock()
_lib = None

c_dp = C.POINTER(C.c_double)
c_ip = C.POINTER(C.c_int)


class b2l_block(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("ld", C.c_int), ("cols", C.c_int)]


class b2l_iter_state(C.Structure):
    """Mirror of b2l_iter_state (include/b200lobpcg.h), field for field."""

    _fields_ = [
        ("n", C.c_int), ("m", C.c_int), ("ldx", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("scale", C.c_double),
        ("tmode", C.c_int), ("tinv", C.c_double), ("tvec", C.c_void_p), ("bdiag", C.c_void_p),
        ("tol", C.c_double), ("relative_tol", C.c_int), ("max_iter", C.c_int),
        ("drift_limit", C.c_double), ("pivot_floor", C.c_double),
        ("x", C.c_void_p), ("ax", C.c_void_p), ("p", C.c_void_p), ("ap", C.c_void_p),
        ("x2", C.c_void_p), ("ax2", C.c_void_p), ("p2", C.c_void_p), ("ap2", C.c_void_p),
        ("w_cur", C.c_void_p), ("w_next", C.c_void_p), ("aw", C.c_void_p),
        ("red_dev", C.c_void_p), ("g2_dev", C.c_void_p),
        ("coef_dev", C.c_void_p), ("lam_dev", C.c_void_p), ("pcols_dev", C.c_void_p),
        ("h_red", C.c_void_p), ("h_g2", C.c_void_p), ("h_stage", C.c_void_p),
        ("h_istage", C.c_void_p),
        ("lam", C.c_void_p), ("active", C.c_void_p), ("lock_iteration", C.c_void_p),
        ("it", C.c_int), ("have_p", C.c_int), ("kst", C.c_int),
        ("stream", C.c_void_p),
        ("norms", C.c_void_p), ("newly", C.c_void_p), ("lam_next", C.c_void_p),
        ("drift", C.c_double),
        ("fallbacks", C.c_int), ("k_next", C.c_int), ("kp", C.c_int),
        ("red_on_host", C.c_int),
        ("repaired", C.c_int),
        ("slab", C.c_void_p),
    ]


ITER_OK, ITER_DRIFT, ITER_DONE = 0, 1, 2

# name -> (restype, argtypes); every exported symbol of include/b200lobpcg.h
SIGNATURES = {
    "b2l_last_error": (C.c_char_p, []),
    "b2l_abi_version": (C.c_int, []),
    "b2l_device_info": (C.c_int, [c_ip, c_ip, c_ip]),
    "b2l_stencil7": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p]),
    "b2l_gram": (C.c_int, [C.c_int, C.POINTER(b2l_block), C.c_int, C.POINTER(b2l_block),
                           C.c_int, C.c_uint, C.c_void_p, C.c_char_p, C.c_void_p,
                           C.c_void_p]),
    "b2l_residual": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p,
                               C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                               C.c_void_p, C.c_void_p]),
    "b2l_update": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                             C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                             C.c_void_p]),
    "b2l_stencil7_gram": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int, C.c_int, C.c_double,
                                    C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_void_p]),
    "b2l_lobpcg_step": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                  C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                  C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_int, C.c_double, C.c_void_p,
                                  C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                  C.c_int, C.c_void_p, C.c_void_p]),
    "b2l_seeded_fill": (C.c_int, [C.c_void_p, C.c_int, C.c_longlong, C.c_int, C.c_longlong,
                                  C.c_ulonglong, C.c_ulonglong, C.c_ulonglong, C.c_ulonglong,
                                  C.c_double, C.c_double, C.c_void_p]),
    "b2l_pcg_init": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double,
                               C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2l_pcg_update": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2l_pcg_dot": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2l_pcg_direction": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                    C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2l_fast_iteration": (C.c_int, [C.POINTER(b2l_iter_state)]),
    "b2l_nccl_load": (C.c_int, [C.c_char_p]),
    "b2l_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_int]),
    "b2l_slab_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_void_p)]),
    "b2l_slab_destroy": (C.c_int, [C.c_void_p]),
    "b2l_slab_info": (C.c_int, [C.c_void_p, c_ip, c_ip, c_ip]),
    "b2l_slab_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
    "b2l_slab_stencil7": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                    C.c_void_p]),
    "b2l_slab_stencil7_gram": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_double, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p]),
    "b2l_stencil7_gram_split": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_double,
                                          C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p]),
    "b2l_iter_state_size": (C.c_int, []),
    "b2l_iter_profile": (C.c_int, [C.POINTER(C.c_double), C.c_int]),
    "b2l_launch_count": (C.c_longlong, []),
    "b2l_set_lapack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2l_set_blas": (C.c_int, [C.c_void_p]),
    "b2l_set_rr_reference": (C.c_int, [C.c_int]),
    "b2l_set_rr_align": (C.c_int, [C.c_double]),
    "b2l_set_lapack_mrrr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2l_rayleigh_ritz_begin": (C.c_int, [C.c_int, C.c_int, C.c_int, c_dp, C.c_int, c_ip, C.c_int,
                                          c_ip, C.c_double, C.POINTER(C.c_int)]),
    "b2l_rayleigh_ritz_finish": (C.c_int, [c_dp, c_dp, c_dp, c_dp, c_ip, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int)]),
    "b2l_rayleigh_ritz": (C.c_int, [C.c_int, C.c_int, C.c_int, c_dp, C.c_int, c_dp, c_dp,
                                    c_ip, C.c_int, c_ip, C.c_double, c_dp, c_dp, c_ip, c_ip,
                                    c_ip]),
}

EDEGENERATE = -1003

ABI_VERSION = 1


class NativeError(RuntimeError):
    """A libb200lobpcg call failed (CUDA error or bad arguments)."""


def load():
    """Load (once) and return the native library; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_0705_2626_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.b2l_abi_version() != ABI_VERSION:
            raise ImportError("libb200lobpcg ABI version mismatch; rebuild")
        if lib.b2l_iter_state_size() != C.sizeof(b2l_iter_state):
            raise ImportError("b2l_iter_state layout mismatch between _lib.py and the library")
        _register_lapack(lib)
        _lib = lib
        return lib


def _register_lapack(lib) -> None:
    """Hand the host Rayleigh-Ritz (b2l_rayleigh_ritz) scipy's LAPACK -- the
    routines scipy.linalg.cholesky / solve_triangular / eigh run for the
    reference -- as plain function pointers from scipy.linalg.cython_lapack."""
    from scipy.linalg import cython_lapack

    get = C.pythonapi.PyCapsule_GetPointer
    get.restype = C.c_void_p
    get.argtypes = [C.py_object, C.c_char_p]
    getname = C.pythonapi.PyCapsule_GetName
    getname.restype = C.c_char_p
    getname.argtypes = [C.py_object]
    caps = cython_lapack.__pyx_capi__
    ptrs = []
    for name in ("dpotrf", "dtrtrs", "dtrtri", "dsyevr"):
        cap = caps[name]
        ptrs.append(get(cap, getname(cap)))
    from scipy.linalg import cython_blas

    bcap = cython_blas.__pyx_capi__["dgemm"]
    lib.b2l_set_blas(get(bcap, getname(bcap)))
    rc = lib.b2l_set_lapack(*ptrs)
    if rc != 0:
        raise ImportError("b2l_set_lapack failed: " + lib.b2l_last_error().decode())
    lib.b2l_set_lapack_mrrr(*[get(caps[n], getname(caps[n])) for n in ("dsytrd", "dstemr",
                                                                      "dormtr")])


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().b2l_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


_device_checked = set()


def ensure_device(dev_index: int) -> None:
    """Fail loudly unless device dev_index is a B200 (sm_100)."""
    if dev_index in _device_checked:
        return
    lib = load()
    sm, ma, mi = C.c_int(), C.c_int(), C.c_int()
    check(lib.b2l_device_info(C.byref(sm), C.byref(ma), C.byref(mi)), "b2l_device_info")
    _device_checked.add(dev_index)
