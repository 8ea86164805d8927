"""numpy port of the reference's hot path -- the CPU baseline.

TEST / BENCH INFRASTRUCTURE ONLY: bench.py's ``cpu_baseline`` leg and
``--impl reference`` arm time this module on the GPU box's host cores (the
reference package itself is not present there).  It issues the same numpy
operations, in the same order, as the reference functions it cites, so its
speed is the reference's speed; the product never imports it.

Its bits equal the reference's on the same host (it IS the same numpy
arithmetic); tests/test_port.py pins it against the golden vectors when the
host's numpy has the fingerprint the goldens were made with.
"""
from __future__ import annotations

import math
import time

import numpy as np

BLOCK = 4096
EPS = 1e-300


def spmv(ia, ja, aa, x, n_rows):
    """sparse.py:217-232: gather, complex multiply, reduceat over nonempty rows."""
    y = np.zeros(n_rows, dtype=np.complex128)
    if aa.shape[0]:
        prod = aa * x[ja]
        starts = ia[:-1]
        nonempty = ia[:-1] < ia[1:]
        if nonempty.any():
            y[nonempty] = np.add.reduceat(prod, starts[nonempty])
    return y


def _fold(values):
    """vecops.py:156-162: reduceat per 4096-block, then a Python left fold."""
    parts = np.add.reduceat(values, np.arange(0, values.shape[0], BLOCK))
    total = parts[0].item()
    for p in parts[1:].tolist():
        total = total + p
    return total


def zdot(x, y):
    """vecops.py:165-186 (conjugated, blocked)."""
    if x.shape[0] == 0:
        return 0j
    return complex(_fold(np.conj(x) * y))


def znorm2(x):
    """vecops.py:189-200 (blocked)."""
    if x.shape[0] == 0:
        return 0.0
    return math.sqrt(_fold(x.real * x.real + x.imag * x.imag))


def zaxpy(alpha, x, y):
    """vecops.py:130-134, in place."""
    y += complex(alpha) * x
    return y


def zscal(alpha, x):
    """vecops.py:124-127, in place."""
    x *= complex(alpha)
    return x


def _cdiv(a: complex, b: complex) -> complex:
    """cnum.py:118-134 (Smith, true divisions)."""
    c, d = b.real, b.imag
    if abs(c) >= abs(d):
        r = d / c
        den = c + d * r
        return complex((a.real + a.imag * r) / den, (a.imag - a.real * r) / den)
    r = c / d
    den = c * r + d
    return complex((a.real * r + a.imag) / den, (a.imag * r - a.real) / den)


def _cmul(a: complex, b: complex) -> complex:
    """cnum.py:113-115."""
    return complex(a.real * b.real - a.imag * b.imag, a.real * b.imag + a.imag * b.real)


def _small(z) -> bool:
    return abs(z) < EPS


class Breakdown(Exception):
    pass


def bicgstab(ia, ja, aa, b, minv=None, tol=1e-9, maxit=1000, x0=None):
    """krylov.py:213-295 with _Run (krylov.py:139-206).

    Returns (x, history, converged, setup_seconds, per_iteration_seconds).
    """
    n = b.shape[0]
    t0 = time.perf_counter()
    apply = (lambda v: v * minv) if minv is not None else (lambda v: v.copy())
    x = x0.copy() if x0 is not None else np.zeros(n, dtype=np.complex128)
    b_norm = znorm2(b)
    r0 = b.copy()
    zaxpy(-1.0, spmv(ia, ja, aa, x, n), r0)
    hist = [znorm2(r0) / b_norm if b_norm > 0.0 else 0.0]
    t_setup = time.perf_counter() - t0
    iter_times = []
    if b_norm == 0.0:
        return np.zeros(n, dtype=np.complex128), [0.0], True, t_setup, iter_times
    if hist[0] <= tol:
        return x, hist, True, t_setup, iter_times

    def true_rel(xv):
        r = b.copy()
        zaxpy(-1.0, spmv(ia, ja, aa, xv, n), r)
        return znorm2(r) / b_norm

    r = r0.copy()
    rs = r0.copy()
    rho = alpha = omega = 1 + 0j
    v = np.zeros(n, dtype=np.complex128)
    p = np.zeros(n, dtype=np.complex128)
    while len(hist) - 1 < maxit:
        ti = time.perf_counter()
        rho_next = zdot(rs, r)
        if _small(rho) or _small(omega):
            raise Breakdown("rho" if _small(rho) else "omega")
        beta = _cmul(_cdiv(rho_next, rho), _cdiv(alpha, omega))
        rho = rho_next
        zaxpy(-omega, v, p)
        zscal(beta, p)
        zaxpy(1.0, r, p)
        ph = apply(p)
        v = spmv(ia, ja, aa, ph, n)
        pivot = zdot(rs, v)
        if _small(pivot):
            raise Breakdown("pivot")
        alpha = _cdiv(rho, pivot)
        s = r.copy()
        zaxpy(-alpha, v, s)
        zaxpy(alpha, ph, x)
        if znorm2(s) / b_norm <= tol:
            rel = true_rel(x)
            if rel <= tol:
                hist.append(rel)
                iter_times.append(time.perf_counter() - ti)
                return x, hist, True, t_setup, iter_times
        sh = apply(s)
        t = spmv(ia, ja, aa, sh, n)
        tt = zdot(t, t)
        if _small(tt):
            raise Breakdown("tt")
        omega = _cdiv(zdot(t, s), tt)
        if _small(omega):
            raise Breakdown("omega")
        zaxpy(omega, sh, x)
        r = s
        zaxpy(-omega, t, r)
        rel = true_rel(x)
        hist.append(rel)
        iter_times.append(time.perf_counter() - ti)
        if rel <= tol:
            return x, hist, True, t_setup, iter_times
    return x, hist, False, t_setup, iter_times
