"""Right-preconditioned BiCGStab on the device (drop-in for the hot-path part
of zlinalg krylov.py).

``solve_bicgstab`` hands the whole loop to libzk (``zk_bicgstab``,
csrc/zk_bicgstab.cu): every vector stays in HBM, axpy/scale updates are fused
with the reductions that follow them, the scalar recurrences run on the
device in Python's arithmetic, and the host waits once for the final report.
Results (solution, iteration count, every residual-history entry) are the
reference's bit for bit (krylov.py:213-295).
"""
from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import BreakdownError, DimensionError, ParameterError, SingularPreconditionerError
from .sparse import CsrMatrix
from .vecops import ZVector

__all__ = ["SolverConfig", "Preconditioner", "SolveReport", "build_jacobi", "solve_bicgstab", "solve_bicgstab_l",
           "solve_tfqmr"]

_BREAKDOWN_EPS = 1e-300
_BREAKDOWN_WHAT = {
    1: "rho",
    2: "omega",
    3: "shadow pivot <r~, A M^-1 p>",
    4: "omega denominator <t, t>",
}


@dataclass(frozen=True)
class SolverConfig:
    """Tolerance, iteration cap and optional initial guess (krylov.py:51-72)."""

    tolerance: float = 1e-9
    max_iterations: int = 1000
    initial_guess: ZVector | None = None
    l: int = 8

    def __post_init__(self):
        if not self.tolerance > 0:
            raise ParameterError(f"tolerance must be positive, got {self.tolerance!r}")
        if self.max_iterations < 1:
            raise ParameterError(f"max_iterations must be >= 1, got {self.max_iterations!r}")
        if self.l < 1:
            raise ParameterError(f"polynomial degree l must be >= 1, got {self.l!r}")


class Preconditioner:
    """Right preconditioner: ``identity`` or ``jacobi`` (krylov.py:75-100).

    ``data`` is the stored inverse diagonal (a complex128 array, as in the
    reference).  It lives in a :class:`ZVector`, so the device copy follows
    the same residency rules as any vector: handing ``data`` out marks the
    device copy stale (the caller may edit it in place), and the next solve
    re-uploads it."""

    __slots__ = ("kind", "_minv")

    def __init__(self, kind: str, data=None):
        if kind not in ("identity", "jacobi"):
            raise ParameterError(f"unknown preconditioner kind {kind!r}")
        if kind == "jacobi" and data is None:
            raise ParameterError("jacobi preconditioner needs the inverse diagonal")
        self.kind = kind
        self._minv = None
        if data is not None:
            self.data = data

    @property
    def data(self):
        return None if self._minv is None else self._minv.data

    @data.setter
    def data(self, value):
        self._minv = value if isinstance(value, ZVector) else ZVector(np.asarray(value, dtype=np.complex128))

    @property
    def size(self) -> int:
        return len(self._minv) if self._minv is not None else 0

    @classmethod
    def identity(cls) -> "Preconditioner":
        return cls("identity")

    def _device_minv(self) -> ZVector:
        return self._minv

    def apply(self, v: ZVector) -> ZVector:
        """M^-1 v as a new vector (krylov.py:92-100)."""
        if self.kind == "identity":
            return v.copy()
        if self.size != len(v):
            raise DimensionError(f"preconditioner built for size {self.size}, vector has {len(v)}")
        out = ZVector._device_new(len(v))
        if len(v):
            m = self._device_minv()._dptr()
            _lib.check(_lib.lib().zk_jacobi_apply(_lib.context(), len(v), v._dptr(), m, out._dptr_out()))
        return out._written()

    def __repr__(self):
        return f"Preconditioner({self.kind})"


def build_jacobi(A: CsrMatrix) -> Preconditioner:
    """Inverse main diagonal (krylov.py:106-120), built on the device
    (zk_jacobi_build): the stored diagonal of each row, a check for missing or
    zero entries, and numpy's complex division 1 / d bit for bit.  The
    preconditioner's vector stays on the device until ``data`` is read."""
    n = min(A.n_rows, A.n_cols)
    minv = ZVector._device_new(n)
    if n:
        zero = ctypes.c_int64(-1)
        status = _lib.lib().zk_jacobi_build(_lib.context(), A._device(), minv._dptr_out(), ctypes.byref(zero))
        if status == _lib.ZK_ERR_SINGULAR:
            raise SingularPreconditionerError(
                f"zero diagonal entry at row {int(zero.value)}; Jacobi preconditioner is singular")
        _lib.check(status)
    return Preconditioner("jacobi", minv._written())


@dataclass
class SolveReport:
    """Per-solve bookkeeping (krylov.py:123-136)."""

    iterations: int = 0
    final_relative_residual: float = math.inf
    converged: bool = False
    residual_history: list = field(default_factory=list)
    elapsed_ms: float = 0.0


# BreakdownError names of BiCGSTAB(l) / TFQMR (krylov.py:341-477), by ZK_BD_* code
_EXT_BREAKDOWN_WHAT = {
    1: "rho",
    2: "omega",
    3: "shadow pivot",
    5: "minimal-residual basis vector {j}",
    6: "sigma = <r~, v>",
    7: "alpha",
    8: "quasi-residual tau",
}


def _device_solve(entry, names, A, b, M, cfg, *extra):
    """Shared front end of the device solvers: the reference's argument
    checks (_Run.__init__, krylov.py:147-163), one libzk call that runs the
    whole solve on the device, and the SolveReport / BreakdownError the
    reference returns (krylov.py:188-206)."""
    cfg = cfg or SolverConfig()
    n = A.n
    if len(b) != n:
        raise DimensionError(f"matrix is {n}x{n} but right-hand side has {len(b)} elements")
    M = M if M is not None else Preconditioner.identity()
    if M.kind == "jacobi" and M.size != n:
        raise DimensionError(f"preconditioner built for size {M.size}, matrix is {n}x{n}")
    t0 = time.perf_counter()
    guess = cfg.initial_guess
    if guess is not None and len(guess) != n:
        raise DimensionError(f"initial guess has {len(guess)} elements, need {n}")
    maxit = int(cfg.max_iterations)
    hist = (ctypes.c_double * (maxit + 1))()
    rep = _lib.SolveReportC()
    x = ZVector._device_new(n)
    fn = getattr(_lib.lib(), entry)
    tail = [hist, ctypes.byref(rep)]
    index = ctypes.c_int32(0)
    if entry == "zk_bicgstab_l":
        tail.append(ctypes.byref(index))
    if n:
        bp = b._dptr()
        mp = M._device_minv()._dptr() if M.kind == "jacobi" else None
        gp = guess._dptr() if guess is not None else None
        status = fn(_lib.context(), A._device(), bp, mp, gp, float(cfg.tolerance), maxit, *extra, x._dptr_out(),
                    *tail)
    else:
        status = fn(_lib.context(), A._device(), None, None, None, float(cfg.tolerance), maxit, *extra, None, *tail)
    if status not in (_lib.ZK_OK, _lib.ZK_ERR_BREAKDOWN):
        _lib.check(status)
    x._written()
    history = list(hist[: rep.history_len])
    report = SolveReport(
        iterations=int(rep.iterations),
        final_relative_residual=history[-1],
        converged=bool(rep.converged),
        residual_history=history,
        elapsed_ms=(time.perf_counter() - t0) * 1e3,
    )
    report.kernel_launches = int(rep.kernel_launches)  # extra attribute, not in the reference
    if status == _lib.ZK_ERR_BREAKDOWN:
        what = names.get(int(rep.breakdown), "recurrence").format(j=index.value)
        raise BreakdownError(
            f"{what} numerically zero (|value| < {_BREAKDOWN_EPS:g}) after {report.iterations} iterations",
            report=report)
    return x, report


def solve_bicgstab(A, b, M=None, cfg=None):
    """Right-preconditioned BiCGStab (van der Vorst), device-resident
    (krylov.py:213-295).

    Returns ``(x, SolveReport)``; non-convergence is a normal return.  Raises
    ``BreakdownError`` (with the partial report) when rho, the shadow pivot,
    <t,t> or omega falls below 1e-300 in magnitude.
    """
    return _device_solve("zk_bicgstab", _BREAKDOWN_WHAT, A, b, M, cfg)


def solve_bicgstab_l(A, b, M=None, cfg=None):
    """Right-preconditioned BiCGSTAB(l) (Sleijpen-Fokkema), device-resident
    (krylov.py:298-410): ``cfg.l`` BiCG steps then the degree-l
    minimal-residual update per cycle; ``cfg.max_iterations`` caps cycles.

    The whole solve is one CUDA-graph launch (csrc/zk_krylov.cu): vectors,
    the scalar recurrences and the modified Gram-Schmidt system stay on the
    device.  Returns and raises as :func:`solve_bicgstab`.
    """
    cfg = cfg or SolverConfig()
    if cfg.l > 32:
        raise ParameterError(f"polynomial degree l must be <= 32 on the device, got {cfg.l!r}")
    return _device_solve("zk_bicgstab_l", _EXT_BREAKDOWN_WHAT, A, b, M, cfg, int(cfg.l))


def solve_tfqmr(A, b, M=None, cfg=None):
    """Right-preconditioned transpose-free QMR (Freund), device-resident
    (krylov.py:413-489): two half-steps per iteration, each followed by the
    true residual check.  One CUDA-graph launch per solve.  Returns and
    raises as :func:`solve_bicgstab`.
    """
    return _device_solve("zk_tfqmr", _EXT_BREAKDOWN_WHAT, A, b, M, cfg)
