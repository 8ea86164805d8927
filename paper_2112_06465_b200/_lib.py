"""ctypes binding of libzk.so (include/zk.h) and the per-process device context.

There is deliberately no CPU fallback: if the shared library or a CUDA
device is missing, the first call that needs the device raises
:class:`DeviceUnavailableError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    BreakdownError,
    DimensionError,
    FormatError,
    ParameterError,
    SingularPreconditionerError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libzk.so")

ZK_OK = 0
ZK_ERR_DIMENSION = 1
ZK_ERR_FORMAT = 2
ZK_ERR_PARAMETER = 3
ZK_ERR_SINGULAR = 4
ZK_ERR_BREAKDOWN = 5
ZK_ERR_CUDA = 6
ZK_ERR_NOMEM = 7
ZK_ERR_NODEVICE = 8

MODE_BLOCKED = 0
MODE_SEQUENTIAL = 1


class DeviceUnavailableError(RuntimeError):
    """libzk.so or a CUDA device is missing; the hot path has no CPU fallback."""


class DeviceError(RuntimeError):
    """A CUDA/driver failure inside libzk."""


class SolveReportC(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("final_relative_residual", ctypes.c_double),
        ("history_len", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
    ]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int
_sz = ctypes.c_size_t

# name -> argtypes (all return zk_status = int unless noted)
SIGNATURES = {
    "zk_context_create": [_i, ctypes.POINTER(_vp)],
    "zk_context_destroy": [_vp],
    "zk_set_arith": [_vp, _i, _i64],
    "zk_malloc": [_vp, _sz, ctypes.POINTER(_vp)],
    "zk_free": [_vp, _vp],
    "zk_host_alloc": [_sz, ctypes.POINTER(_vp)],
    "zk_host_free": [_vp],
    "zk_memcpy_h2d": [_vp, _vp, _vp, _sz],
    "zk_memcpy_d2h": [_vp, _vp, _vp, _sz],
    "zk_memcpy_d2d": [_vp, _vp, _vp, _sz],
    "zk_memset": [_vp, _vp, _i, _sz],
    "zk_synchronize": [_vp],
    "zk_launch_count": [_vp, ctypes.POINTER(_i64)],
    "zk_stream": [_vp, ctypes.POINTER(_vp)],
    "zk_host_register": [_vp, _sz],
    "zk_host_unregister": [_vp],
    "zk_event_record": [_vp, _i],
    "zk_event_elapsed": [_vp, _i, _i, ctypes.POINTER(_d)],
    "zk_profile_enable": [_vp, _i],
    "zk_profile_read": [_vp, ctypes.POINTER(_d), ctypes.POINTER(_i64)],
    "zk_zscal": [_vp, _i64, _d, _d, _vp],
    "zk_zaxpy": [_vp, _i64, _d, _d, _vp, _vp],
    "zk_zaxmy": [_vp, _i64, _vp, _vp],
    "zk_zassign": [_vp, _i64, _vp, _vp],
    "zk_jacobi_apply": [_vp, _i64, _vp, _vp, _vp],
    "zk_zdotc": [_vp, _i64, _vp, _vp, _i, _i64, _i, ctypes.POINTER(_d)],
    "zk_znorm2": [_vp, _i64, _vp, _i64, _i, ctypes.POINTER(_d)],
    "zk_zdotc_dev": [_vp, _i64, _vp, _vp, _i, _i64, _i, _vp],
    "zk_znorm2_dev": [_vp, _i64, _vp, _i64, _i, _vp],
    "zk_csr_create": [_vp, _i64, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)],
    "zk_csr_create_device": [_vp, _i64, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)],
    "zk_csr_destroy": [_vp],
    "zk_csr_bytes": [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "zk_spmv": [_vp, _vp, _vp, _vp],
    "zk_jacobi_build": [_vp, _vp, _vp, ctypes.POINTER(_i64)],
    "zk_spmv_dotc": [_vp, _vp, _vp, _vp, _vp, _i, ctypes.POINTER(_d)],
    "zk_bicgstab": [_vp, _vp, _vp, _vp, _vp, _d, _i64, _vp, ctypes.POINTER(_d), ctypes.POINTER(SolveReportC)],
    "zk_bicgstab_l": [_vp, _vp, _vp, _vp, _vp, _d, _i64, _i, _vp, ctypes.POINTER(_d), ctypes.POINTER(SolveReportC),
                      ctypes.POINTER(ctypes.c_int32)],
    "zk_tfqmr": [_vp, _vp, _vp, _vp, _vp, _d, _i64, _vp, ctypes.POINTER(_d), ctypes.POINTER(SolveReportC)],
    "zk_dshard_create": [_vp, _vp, _i64, _i64, _i, _i64, _i, _i64, ctypes.POINTER(_vp)],
    "zk_dshard_destroy": [_vp],
    "zk_dshard_vector": [_vp, _i, ctypes.POINTER(ctypes.POINTER(_d)), ctypes.POINTER(_i64)],
    "zk_dshard_reset": [_vp, _d, _i64, _i],
    "zk_dshard_phase": [_vp, _i],
    "zk_dshard_finish": [_vp, _i, _vp],
    "zk_dshard_pack": [_vp, _i, _vp, _i64, _vp],
    "zk_dshard_status": [_vp, ctypes.POINTER(SolveReportC), ctypes.POINTER(ctypes.c_int32)],
    "zk_dshard_history": [_vp, _vp, _i64],
}
STRING_FUNCS = ("zk_last_error", "zk_version")

_lib = None
_ctx = None
_lock = threading.Lock()


def load_library():
    """Load libzk.so (building it in-tree with nvcc if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        try:
            from . import _build
            _build.build()
        except Exception as exc:  # noqa: BLE001
            raise DeviceUnavailableError(f"libzk.so is missing and could not be built: {exc}") from exc
    # ZK_LIB_PATH: load an alternative build (kernel-variant experiments only)
    lib = ctypes.CDLL(os.environ.get("ZK_LIB_PATH", LIB_PATH))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    for name in STRING_FUNCS:
        fn = getattr(lib, name)
        fn.argtypes = []
        fn.restype = ctypes.c_char_p
    _lib = lib
    return lib


_EXC = {
    ZK_ERR_DIMENSION: DimensionError,
    ZK_ERR_FORMAT: FormatError,
    ZK_ERR_PARAMETER: ParameterError,
    ZK_ERR_SINGULAR: SingularPreconditionerError,
    ZK_ERR_NODEVICE: DeviceUnavailableError,
}


def check(status: int) -> None:
    if status == ZK_OK:
        return
    msg = _lib.zk_last_error().decode(errors="replace")
    if status == ZK_ERR_BREAKDOWN:
        raise BreakdownError(msg)
    exc = _EXC.get(status, DeviceError)
    raise exc(msg)


def _env_arith():
    mode = os.environ.get("ZK_ARITH", "fma").lower()
    elide = int(os.environ.get("ZK_ELIDE_BYTES", "262144"))
    return (0 if mode == "plain" else 1), elide


def context():
    """The process-wide device context (device = LOCAL_RANK or 0)."""
    global _ctx
    if _ctx is not None:
        return _ctx
    with _lock:
        if _ctx is None:
            lib = load_library()
            dev = int(os.environ.get("ZK_DEVICE", os.environ.get("LOCAL_RANK", "0")))
            h = ctypes.c_void_p()
            check(lib.zk_context_create(dev, ctypes.byref(h)))
            fma, elide = _env_arith()
            check(lib.zk_set_arith(h, fma, elide))
            _ctx = h
    return _ctx


def lib():
    return load_library()


def set_arithmetic(use_fma: bool = True, elide_bytes: int = 262144) -> None:
    """Select the numpy fingerprint being reproduced (see include/zk.h)."""
    check(load_library().zk_set_arith(context(), int(bool(use_fma)), int(elide_bytes)))


def launch_count() -> int:
    c = ctypes.c_int64()
    check(load_library().zk_launch_count(context(), ctypes.byref(c)))
    return c.value


PHASES = ("setup", "p_first", "pivot_first", "pivot_first_dot", "s_update", "x_alpha", "true_res_s", "spmv_t",
          "tt_ts", "xr_update", "true_res", "res_pass", "p_next", "spmv_pivot", "pivot_dot", "spmv2")


def event_record(slot: int) -> None:
    check(load_library().zk_event_record(context(), int(slot)))


def event_elapsed_ms(start: int, stop: int) -> float:
    ms = ctypes.c_double()
    check(load_library().zk_event_elapsed(context(), int(start), int(stop), ctypes.byref(ms)))
    return ms.value


def profile_enable(on: bool) -> None:
    check(load_library().zk_profile_enable(context(), int(bool(on))))


def profile_read() -> dict:
    ms = (ctypes.c_double * len(PHASES))()
    cnt = (ctypes.c_int64 * len(PHASES))()
    check(load_library().zk_profile_read(context(), ms, cnt))
    return {name: (ms[i], cnt[i]) for i, name in enumerate(PHASES)}


def host_register(arr) -> None:
    check(load_library().zk_host_register(arr.ctypes.data, arr.nbytes))


def host_unregister(arr) -> None:
    check(load_library().zk_host_unregister(arr.ctypes.data))


def synchronize() -> None:
    check(load_library().zk_synchronize(context()))


class DeviceBuffer:
    """Device allocation from the context's caching allocator."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        check(load_library().zk_malloc(context(), max(self.nbytes, 1), ctypes.byref(p)))
        self.ptr = p.value

    def __del__(self):
        try:
            if self.ptr and _lib is not None and _ctx is not None:
                _lib.zk_free(_ctx, self.ptr)
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass
        self.ptr = None
