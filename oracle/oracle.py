"""ctypes front end of the C oracle (``zk_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` leg as the checker.  The product package
never imports this module.

Each function restates one reference call (file:line under
``/root/reference/pkg/src/zlinalg``) with the reference's exact floating-point
order; see the C header for the arithmetic contract.  The library is built by
``oracle/Makefile`` (``__graft_entry__.build()`` runs it).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libzk_oracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)

STATUS_CONVERGED, STATUS_NOT_CONVERGED, STATUS_BREAKDOWN = 0, 1, 2
BREAKDOWN_NAMES = {
    1: "rho",
    2: "omega",
    3: "shadow pivot <r~, A M^-1 p>",
    4: "omega denominator <t, t>",
}
# BiCGSTAB(l) / TFQMR breakdown codes (krylov.py:298-489): name for the
# reference's BreakdownError text; 5 carries the basis-vector index j
EXT_BREAKDOWN_NAMES = {
    1: "rho",
    2: "omega",
    3: "shadow pivot",
    5: "minimal-residual basis vector {j}",
    6: "sigma = <r~, v>",
    7: "alpha",
    8: "quasi-residual tau",
}


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.zko_set_arith.argtypes = [ctypes.c_int, ctypes.c_int64]
        L.zko_zscal.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_double, _D]
        L.zko_zaxpy.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_double, _D, _D]
        L.zko_zaxmy.argtypes = [ctypes.c_int64, _D, _D]
        L.zko_jacobi_apply.argtypes = [ctypes.c_int64, _D, _D, _D]
        L.zko_zdot.argtypes = [ctypes.c_int64, _D, _D, ctypes.c_int, ctypes.c_int64, ctypes.c_int, _D]
        L.zko_znorm2.argtypes = [ctypes.c_int64, _D, ctypes.c_int64, ctypes.c_int]
        L.zko_znorm2.restype = ctypes.c_double
        L.zko_spmv.argtypes = [ctypes.c_int64, ctypes.c_int64, _I, _I, _D, _D, _D]
        L.zko_bicgstab.argtypes = [ctypes.c_int64, _I, _I, _D, _D, _D, _D, ctypes.c_double,
                                   ctypes.c_int64, _D, _D, _I, ctypes.POINTER(ctypes.c_int)]
        L.zko_bicgstab.restype = ctypes.c_int
        _IP = ctypes.POINTER(ctypes.c_int)
        L.zko_bicgstab_l.argtypes = [ctypes.c_int64, _I, _I, _D, _D, _D, _D, ctypes.c_double, ctypes.c_int64,
                                     ctypes.c_int, _D, _D, _I, _IP, _IP]
        L.zko_bicgstab_l.restype = ctypes.c_int
        L.zko_tfqmr.argtypes = [ctypes.c_int64, _I, _I, _D, _D, _D, _D, ctypes.c_double, ctypes.c_int64, _D, _D,
                                _I, _IP]
        L.zko_tfqmr.restype = ctypes.c_int
        _lib = L
    return _lib


def _c128(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def set_arith(use_fma: bool = True, elide_bytes: int = 262144) -> None:
    lib().zko_set_arith(int(use_fma), int(elide_bytes))


def zscal(alpha, x):
    """vecops.py:124-127 on a copy of x; returns the new array."""
    a = complex(alpha)
    out = _c128(x).copy()
    lib().zko_zscal(out.shape[0], a.real, a.imag, _dp(out))
    return out


def zaxpy(alpha, x, y):
    """vecops.py:130-134 on a copy of y."""
    a = complex(alpha)
    x = _c128(x)
    out = _c128(y).copy()
    lib().zko_zaxpy(out.shape[0], a.real, a.imag, _dp(x), _dp(out))
    return out


def zaxmy(x, y):
    """vecops.py:137-141 on a copy of y."""
    x = _c128(x)
    out = _c128(y).copy()
    lib().zko_zaxmy(out.shape[0], _dp(x), _dp(out))
    return out


def jacobi_apply(v, minv):
    """krylov.py:92-100 (jacobi branch)."""
    v = _c128(v)
    minv = _c128(minv)
    out = np.empty_like(v)
    lib().zko_jacobi_apply(v.shape[0], _dp(v), _dp(minv), _dp(out))
    return out


def zdot(x, y, conjugate=True, block_size=4096, sequential=False) -> complex:
    """vecops.py:165-186."""
    x = _c128(x)
    y = _c128(y)
    out = np.zeros(2)
    lib().zko_zdot(x.shape[0], _dp(x), _dp(y), int(conjugate), int(block_size), int(sequential), _dp(out))
    return complex(out[0], out[1])


def znorm2(x, block_size=4096, sequential=False) -> float:
    """vecops.py:189-200."""
    x = _c128(x)
    return float(lib().zko_znorm2(x.shape[0], _dp(x), int(block_size), int(sequential)))


def spmv(n_rows, n_cols, ia, ja, aa, x):
    """sparse.py:217-232."""
    ia, ja, aa, x = _i64(ia), _i64(ja), _c128(aa), _c128(x)
    y = np.empty(int(n_rows), dtype=np.complex128)
    lib().zko_spmv(int(n_rows), int(n_cols), ia.ctypes.data_as(_I), ja.ctypes.data_as(_I),
                   _dp(aa), _dp(x), _dp(y))
    return y


def bicgstab(n, ia, ja, aa, b, minv=None, x0=None, tol=1e-9, maxit=1000):
    """krylov.py:213-295.  Returns (x, history, iterations, status, breakdown_what)."""
    ia, ja, aa, b = _i64(ia), _i64(ja), _c128(aa), _c128(b)
    minv = _c128(minv) if minv is not None else None
    x0 = _c128(x0) if x0 is not None else None
    x = np.empty(int(n), dtype=np.complex128)
    hist = np.zeros(int(maxit) + 1)
    iters = ctypes.c_int64(0)
    what = ctypes.c_int(0)
    st = lib().zko_bicgstab(int(n), ia.ctypes.data_as(_I), ja.ctypes.data_as(_I), _dp(aa), _dp(b),
                            _dp(minv), _dp(x0), float(tol), int(maxit), _dp(x), _dp(hist),
                            ctypes.byref(iters), ctypes.byref(what))
    k = iters.value
    return x, hist[: k + 1].tolist(), k, st, what.value


def bicgstab_l(n, ia, ja, aa, b, minv=None, x0=None, tol=1e-9, maxit=1000, ell=8):
    """krylov.py:298-410.  Returns (x, history, iterations, status, what, what_j)."""
    ia, ja, aa, b = _i64(ia), _i64(ja), _c128(aa), _c128(b)
    minv = _c128(minv) if minv is not None else None
    x0 = _c128(x0) if x0 is not None else None
    x = np.empty(int(n), dtype=np.complex128)
    hist = np.zeros(int(maxit) + 1)
    iters = ctypes.c_int64(0)
    what, what_j = ctypes.c_int(0), ctypes.c_int(0)
    st = lib().zko_bicgstab_l(int(n), ia.ctypes.data_as(_I), ja.ctypes.data_as(_I), _dp(aa), _dp(b), _dp(minv),
                              _dp(x0), float(tol), int(maxit), int(ell), _dp(x), _dp(hist), ctypes.byref(iters),
                              ctypes.byref(what), ctypes.byref(what_j))
    k = iters.value
    return x, hist[: k + 1].tolist(), k, st, what.value, what_j.value


def tfqmr(n, ia, ja, aa, b, minv=None, x0=None, tol=1e-9, maxit=1000):
    """krylov.py:413-489.  Returns (x, history, iterations, status, what)."""
    ia, ja, aa, b = _i64(ia), _i64(ja), _c128(aa), _c128(b)
    minv = _c128(minv) if minv is not None else None
    x0 = _c128(x0) if x0 is not None else None
    x = np.empty(int(n), dtype=np.complex128)
    hist = np.zeros(int(maxit) + 1)
    iters = ctypes.c_int64(0)
    what = ctypes.c_int(0)
    st = lib().zko_tfqmr(int(n), ia.ctypes.data_as(_I), ja.ctypes.data_as(_I), _dp(aa), _dp(b), _dp(minv),
                         _dp(x0), float(tol), int(maxit), _dp(x), _dp(hist), ctypes.byref(iters), ctypes.byref(what))
    k = iters.value
    return x, hist[: k + 1].tolist(), k, st, what.value


def breakdown_message(what: int, what_j: int, iterations: int, ext: bool = True) -> str:
    """The reference's BreakdownError text (krylov.py:200-206)."""
    name = (EXT_BREAKDOWN_NAMES if ext else BREAKDOWN_NAMES)[what].format(j=what_j)
    return f"{name} numerically zero (|value| < 1e-300) after {iterations} iterations"
