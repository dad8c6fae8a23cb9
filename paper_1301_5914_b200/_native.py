"""ctypes binding of libhobi.so (include/hobi.h).  No fallback: if the library
or a CUDA device is missing, every entry point raises."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhobi.so")

HOBI_OK = 0
HOBI_ERR_VALUE = 1
HOBI_ERR_DEGENERATE_ARC = 2
HOBI_ERR_SINGULARITY = 3
HOBI_ERR_NONCONVERGENCE = 4
HOBI_ERR_CUDA = 5
HOBI_ERR_NCCL = 6
HOBI_ERR_STATE = 7

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_ctxp = C.c_void_p
APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, _dp, _dp, C.c_int64)

# name -> (restype, argtypes); every symbol include/hobi.h declares
SIGNATURES = {
    "hobi_last_error": (C.c_char_p, []),
    "hobi_abi_version": (C.c_int, []),
    "hobi_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "hobi_device_sms": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "hobi_create": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _i64p, C.c_int64, C.c_double, C.c_double,
                              C.c_double, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, C.c_int,
                              C.POINTER(_ctxp)]),
    "hobi_create_from_caches": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _i64p, C.c_int64, C.c_double,
                                          C.c_double, C.c_double, _dp, _dp, _dp, _dp, C.c_int, _dp,
                                          _dp, _dp, _dp, C.c_int, _i64p, _i64p, _i64p, _i64p,
                                          C.POINTER(_ctxp)]),
    "hobi_create_lobi": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _i64p, C.c_int64, C.c_double,
                                   C.c_double, C.c_double, C.POINTER(_ctxp)]),
    "hobi_destroy": (C.c_int, [_ctxp]),
    "hobi_size": (C.c_int, [_ctxp, _i64p, _i64p]),
    "hobi_matvec": (C.c_int, [_ctxp, _dp, _dp]),
    "hobi_matvec_device": (C.c_int, [_ctxp, C.c_void_p, C.c_void_p]),
    "hobi_matvec_rows": (C.c_int, [_ctxp, _dp, C.c_int64, C.c_int64, _dp, _dp]),
    "hobi_rhs": (C.c_int, [_ctxp, _dp, _dp, C.c_int64, _dp]),
    "hobi_energy": (C.c_int, [_ctxp, _dp, _dp, C.c_int64, _dp, _dp, _dp]),
    "hobi_gmres": (C.c_int, [_ctxp, _dp, C.c_double, C.c_int, C.c_int, _dp, C.POINTER(C.c_int), _dp, _dp,
                             C.POINTER(C.c_int)]),
    "hobi_solve": (C.c_int, [_ctxp, _dp, _dp, C.c_int64, C.c_double, C.c_int, C.c_int, _dp, _dp, _dp,
                             C.POINTER(C.c_int), _dp, C.POINTER(C.c_int)]),
    "hobi_gmres_host_operator": (C.c_int, [C.c_int, C.c_int64, APPLY_FN, C.c_void_p, _dp, C.c_double,
                                           C.c_int, C.c_int, _dp, C.POINTER(C.c_int), _dp, _dp,
                                           C.POINTER(C.c_int)]),
    "hobi_comm_p2p_disable": (C.c_int, [_ctxp]),
    "hobi_comm_info": (C.c_int, [_ctxp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "hobi_create_default": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _i64p, C.c_int64, C.c_double, C.c_double,
                                      C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
    "hobi_msms_parse": (C.c_int, [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, _dp, C.c_int64, _i64p, C.c_int64,
                                  _i64p, _i64p]),
    "hobi_group_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p)]),
    "hobi_group_destroy": (C.c_int, [C.c_void_p]),
    "hobi_group_matvec": (C.c_int, [C.c_void_p, _dp, _dp]),
    "hobi_group_gmres": (C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, _dp, C.POINTER(C.c_int),
                                   _dp, _dp, C.POINTER(C.c_int)]),
    "hobi_group_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _i64p, _i64p,
                                  C.POINTER(C.c_int)]),
    "hobi_group_bench": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]),
    "hobi_export_caches": (C.c_int, [_ctxp, _dp, _dp, _dp, _dp, _dp, _dp, _i64p, _i64p, _i64p, _i64p]),
    "hobi_export_nodes": (C.c_int, [_ctxp, _dp, _dp]),
    "hobi_kernel_values": (C.c_int, [C.c_int, _dp, _dp, _dp, C.c_int64, C.c_double, C.c_double,
                                     C.c_double, _dp]),
    "hobi_source_terms": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _dp, _dp, C.c_int64, _dp, _dp]),
    "hobi_geometry_fit_arcs": (C.c_int, [C.c_int, _dp, _dp, _dp, _dp, C.c_int64, _dp, C.POINTER(C.c_int)]),
    "hobi_geometry_arc_normals": (C.c_int, [C.c_int, _dp, _dp, _dp, C.c_int64, _dp, C.POINTER(C.c_int)]),
    "hobi_geometry_nodes": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _dp, _dp, _i64p, C.POINTER(C.c_int)]),
    "hobi_geometry_frames": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _dp, C.c_int, _dp, _dp, _dp, _dp, _dp]),
    "hobi_comm_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "hobi_comm_init": (C.c_int, [_ctxp, C.POINTER(C.c_ubyte), C.c_int, C.c_int]),
    "hobi_emulate_ranks": (C.c_int, [_ctxp, C.c_int]),
    "hobi_comm_p2p_handle": (C.c_int, [_ctxp, C.POINTER(C.c_ubyte)]),
    "hobi_comm_p2p_open": (C.c_int, [_ctxp, C.POINTER(C.c_ubyte), C.c_int, C.c_int]),
    "hobi_comm_init_p2p": (C.c_int, [_ctxp, C.c_int, C.c_int]),
    "hobi_matvec_p2p_phase": (C.c_int, [_ctxp, _dp, _dp, C.c_int]),
    "hobi_kirkwood_traces": (C.c_int, [C.c_int, _dp, C.c_int64, _dp, _dp, C.c_int64, _dp, _dp, C.c_int, _dp,
                                       _dp]),
    "hobi_kirkwood_energy_terms": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _dp, _dp, C.c_int, _dp]),
    "hobi_hypot_check": (C.c_int, [C.c_int, _dp, _dp, C.c_int64, _dp]),
    "hobi_timing_reset": (C.c_int, [_ctxp]),
    "hobi_timing": (C.c_int, [_ctxp, _dp, _i64p, _i64p]),
    "hobi_pairs_per_matvec": (C.c_int, [_ctxp, _dp]),
    "hobi_sweep_layout": (C.c_int, [_ctxp, C.POINTER(C.c_int), _i64p]),
    "hobi_sweep_variant": (C.c_int, [_ctxp, C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    "hobi_bench_rows": (C.c_int, [_ctxp, _dp, C.c_int64, C.c_int64, C.c_int, C.c_int, _dp]),
    "hobi_bench": (C.c_int, [_ctxp, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]),
    "hobi_probe_fp64_tflops": (C.c_int, [C.c_int, C.c_double, _dp]),
}

_lib = None


class NativeError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(message)
        self.status = status


def load():
    """Load libhobi.so, building it first when it is missing or older than its
    sources (build._stale).  Concurrent first loads (every torchrun rank) are
    serialised by an exclusive lock on a file next to the library, so exactly
    one process builds and the others load its result."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build

    if _build.sources_present() and _build._stale():
        import fcntl

        try:
            with open(os.path.join(_HERE, ".build.lock"), "w") as lock:
                fcntl.flock(lock, fcntl.LOCK_EX)
                if _build._stale():
                    _build.build()
        except Exception as exc:  # noqa: BLE001
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"libhobi.so is missing and could not be built: {exc}") from exc
            import warnings

            warnings.warn(f"libhobi.so is older than its sources and the rebuild failed ({exc}); "
                          "loading the existing library", RuntimeWarning, stacklevel=2)
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().hobi_last_error().decode()


def check(status: int):
    if status != HOBI_OK:
        raise NativeError(status, last_error())


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def device_count() -> int:
    n = C.c_int(0)
    st = load().hobi_device_count(C.byref(n))
    return n.value if st == HOBI_OK else 0


def require_device():
    if device_count() < 1:
        raise RuntimeError(
            "paper_1301_5914_b200 needs a CUDA device (B200/sm_100a); there is no CPU fallback")
