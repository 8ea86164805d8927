"""BiCGSTAB(l) and TFQMR (SURVEY 8f "next": the paper's other two solvers,
``PAPER.md:662``), on the device kernels of this package.

Both solvers are orchestrated from the host exactly as the reference writes
them -- the same sequence of level-1 calls, SpMVs and preconditioner
applications (krylov.py:298-410 and 413-489), with the scalar recurrences
in ``Cplx`` arithmetic (cnum.py:113-134) -- while every vector operation
runs in libzk on HBM-resident vectors.  Because each library call returns
the reference's bits, the solutions, iteration counts and residual
histories are the reference's bits too (tests/test_krylov_ext_gpu.py checks
them against fixtures made by the live reference).  Unlike
``solve_bicgstab`` these loops read the scalars back every step (one device
sync per dot product): correctness first, a device-resident graph like
BiCGStab's is the next step.
"""
from __future__ import annotations

import math
import time

from .cnum import Cplx
from .errors import BreakdownError, DimensionError
from .krylov import Preconditioner, SolveReport, SolverConfig
from .sparse import CsrMatrix, spmv
from .vecops import ZVector, zaxpy, zdot, znorm2, zscal

__all__ = ["solve_bicgstab_l", "solve_tfqmr"]

_EPS = 1e-300  # krylov.py:48 _BREAKDOWN_EPS
_ONE = Cplx(1.0)
_MINUS_ONE = Cplx(-1.0)


def _tiny(value) -> bool:
    """krylov.py:209-210: abs() below the breakdown threshold."""
    return abs(value) < _EPS


class _Bookkeeping:
    """Shared setup and reporting (the reference's _Run, krylov.py:139-206):
    norms, initial residual, truthful residual checks, the history."""

    def __init__(self, A: CsrMatrix, b: ZVector, M, cfg: SolverConfig):
        n = A.n
        if len(b) != n:
            raise DimensionError(f"matrix is {n}x{n} but right-hand side has {len(b)} elements")
        self.A, self.b, self.cfg = A, b, cfg
        self.M = M if M is not None else Preconditioner.identity()
        if self.M.kind == "jacobi" and self.M.data.shape[0] != n:
            raise DimensionError(f"preconditioner built for size {self.M.data.shape[0]}, matrix is {n}x{n}")
        self.started = time.perf_counter()
        guess = cfg.initial_guess
        self.x0 = guess.copy() if guess is not None else ZVector.zeros(n)
        if guess is not None and len(self.x0) != n:
            raise DimensionError(f"initial guess has {len(self.x0)} elements, need {n}")
        self.b_norm = znorm2(b)
        self.r0 = self.residual_of(self.x0)
        self.r0_norm = znorm2(self.r0)
        self.history = [self.r0_norm / self.b_norm if self.b_norm > 0.0 else 0.0]

    @property
    def iterations(self) -> int:
        return len(self.history) - 1

    def residual_of(self, x: ZVector) -> ZVector:
        r = self.b.copy()
        zaxpy(_MINUS_ONE, spmv(self.A, x), r)
        return r

    def true_rel(self, x: ZVector) -> float:
        return znorm2(self.residual_of(x)) / self.b_norm

    def report(self, converged: bool) -> SolveReport:
        return SolveReport(iterations=self.iterations, final_relative_residual=self.history[-1],
                           converged=converged, residual_history=list(self.history),
                           elapsed_ms=(time.perf_counter() - self.started) * 1e3)

    def shortcut(self):
        """Zero right-hand side or an exact guess (krylov.py:171-181)."""
        if self.b_norm == 0.0:
            rep = self.report(converged=True)
            rep.residual_history, rep.final_relative_residual = [0.0], 0.0
            return ZVector.zeros(len(self.b)), rep
        if self.history[0] <= self.cfg.tolerance:
            return self.x0, self.report(converged=True)
        return None

    def fail(self, what: str) -> BreakdownError:
        return BreakdownError(f"{what} numerically zero (|value| < {_EPS:g}) after {self.iterations} iterations",
                              report=self.report(converged=False))


def solve_bicgstab_l(A, b, M=None, cfg=None):
    """Right-preconditioned BiCGSTAB(l) (Sleijpen-Fokkema), krylov.py:298-410.

    ``cfg.l`` BiCG steps per cycle, then a degree-l minimal-residual update
    (modified Gram-Schmidt on the residual stack, triangular solves); one
    history entry per cycle or early exit.  Updates accumulate in the
    preconditioned variable: the iterate is x0 + M^-1 acc.
    """
    cfg = cfg or SolverConfig()
    ell = cfg.l
    bk = _Bookkeeping(A, b, M, cfg)
    done = bk.shortcut()
    if done is not None:
        return done
    n = len(b)
    Mop = bk.M

    def apply_op(vec):  # A M^-1 vec
        return spmv(A, Mop.apply(vec))

    def iterate(acc):
        x = bk.x0.copy()
        zaxpy(_ONE, Mop.apply(acc), x)
        return x

    acc = ZVector.zeros(n)
    rs = [bk.r0.copy()] + [ZVector.zeros(n) for _ in range(ell)]
    us = [ZVector.zeros(n) for _ in range(ell + 1)]
    shadow = bk.r0.copy()
    rho, alpha, omega = Cplx(1.0), Cplx(0.0), Cplx(1.0)
    while bk.iterations < cfg.max_iterations:
        if _tiny(omega):
            raise bk.fail("omega")
        rho = -omega * rho
        for j in range(ell):  # BiCG steps (krylov.py:339-363)
            rho_new = zdot(shadow, rs[j], conjugate=True)
            if _tiny(rho):
                raise bk.fail("rho")
            beta = alpha * (rho_new / rho)
            rho = rho_new
            for i in range(j + 1):
                zscal(-beta, us[i])
                zaxpy(_ONE, rs[i], us[i])
            us[j + 1] = apply_op(us[j])
            pivot = zdot(shadow, us[j + 1], conjugate=True)
            if _tiny(pivot):
                raise bk.fail("shadow pivot")
            alpha = rho / pivot
            for i in range(j + 1):
                zaxpy(-alpha, us[i + 1], rs[i])
            rs[j + 1] = apply_op(rs[j])
            zaxpy(alpha, us[0], acc)
            if znorm2(rs[0]) / bk.b_norm <= cfg.tolerance:  # early exit, truthful check
                x = iterate(acc)
                rel = bk.true_rel(x)
                if rel <= cfg.tolerance:
                    bk.history.append(rel)
                    return x, bk.report(converged=True)
        # minimal-residual polynomial (krylov.py:365-397)
        tau = [[Cplx(0.0)] * (ell + 1) for _ in range(ell + 1)]
        sigma = [0.0] * (ell + 1)
        gp = [Cplx(0.0)] * (ell + 1)
        for j in range(1, ell + 1):
            for i in range(1, j):
                t_ij = zdot(rs[i], rs[j], conjugate=True) / sigma[i]
                tau[i][j] = t_ij
                zaxpy(-t_ij, rs[i], rs[j])
            sigma[j] = zdot(rs[j], rs[j], conjugate=True).re
            if _tiny(sigma[j]):
                raise bk.fail(f"minimal-residual basis vector {j}")
            gp[j] = zdot(rs[j], rs[0], conjugate=True) / sigma[j]
        g = [Cplx(0.0)] * (ell + 1)
        g[ell] = gp[ell]
        omega = g[ell]
        for j in range(ell - 1, 0, -1):
            acc_s = Cplx(0.0)
            for i in range(j + 1, ell + 1):
                acc_s = acc_s + tau[j][i] * g[i]
            g[j] = gp[j] - acc_s
        gpp = [Cplx(0.0)] * (ell + 1)
        for j in range(1, ell):
            acc_s = Cplx(0.0)
            for i in range(j + 1, ell):
                acc_s = acc_s + tau[j][i] * g[i + 1]
            gpp[j] = g[j + 1] + acc_s
        # polynomial update (krylov.py:399-404)
        zaxpy(g[1], rs[0], acc)
        zaxpy(-gp[ell], rs[ell], rs[0])
        zaxpy(-g[ell], us[ell], us[0])
        for j in range(1, ell):
            zaxpy(-g[j], us[j], us[0])
            zaxpy(gpp[j], rs[j], acc)
            zaxpy(-gp[j], rs[j], rs[0])
        x = iterate(acc)
        rel = bk.true_rel(x)
        bk.history.append(rel)
        if rel <= cfg.tolerance:
            return x, bk.report(converged=True)
    return iterate(acc), bk.report(converged=False)


def solve_tfqmr(A, b, M=None, cfg=None):
    """Right-preconditioned transpose-free QMR (Freund), krylov.py:413-489:
    two half-steps per iteration, each followed by a true-residual check."""
    cfg = cfg or SolverConfig()
    bk = _Bookkeeping(A, b, M, cfg)
    done = bk.shortcut()
    if done is not None:
        return done
    Mop = bk.M
    x = bk.x0
    w = bk.r0.copy()
    y = bk.r0.copy()
    shadow = bk.r0.copy()
    d = ZVector.zeros(len(b))
    z = Mop.apply(y)
    u = spmv(A, z)
    v = u.copy()
    theta, eta, tau = 0.0, Cplx(0.0), bk.r0_norm
    rho = zdot(shadow, bk.r0, conjugate=True)
    while bk.iterations < cfg.max_iterations:
        sigma = zdot(shadow, v, conjugate=True)
        if _tiny(sigma):
            raise bk.fail("sigma = <r~, v>")
        alpha = rho / sigma
        if _tiny(alpha):
            raise bk.fail("alpha")
        rel, converged = math.inf, False
        for half in (0, 1):
            if half:
                zaxpy(-alpha, v, y)
                z = Mop.apply(y)
                u = spmv(A, z)
            zaxpy(-alpha, u, w)
            zscal((theta * theta) * eta / alpha, d)  # d = z + (theta^2 eta / alpha) d
            zaxpy(_ONE, z, d)
            if _tiny(tau):
                raise bk.fail("quasi-residual tau")
            theta = znorm2(w) / tau
            c = 1.0 / math.sqrt(1.0 + theta * theta)
            tau = tau * theta * c
            eta = (c * c) * alpha
            zaxpy(eta, d, x)
            rel = bk.true_rel(x)
            if rel <= cfg.tolerance:
                converged = True
                break
        bk.history.append(rel)
        if converged:
            return x, bk.report(converged=True)
        rho_new = zdot(shadow, w, conjugate=True)
        if _tiny(rho):
            raise bk.fail("rho")
        beta = rho_new / rho
        rho = rho_new
        zscal(beta, y)  # y = w + beta y
        zaxpy(_ONE, w, y)
        u_prev = u
        z = Mop.apply(y)
        u = spmv(A, z)
        zscal(beta, v)  # v = u + beta (u_prev + beta v)
        zaxpy(_ONE, u_prev, v)
        zscal(beta, v)
        zaxpy(_ONE, u, v)
    return x, bk.report(converged=False)
