"""Generate golden input/output vectors by running the LIVE reference.

Run in the dev container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [krylov_ext]

It imports ``zlinalg`` from ``/root/reference/pkg/src`` read-only, feeds it
seeded inputs, and writes compressed ``.npz`` fixtures next to this script.
The fixtures pin (a) the C oracle (``oracle/zk_oracle.c``) and (b) the CUDA
path, both bitwise, on hosts where the reference itself cannot run (the GPU
box has no /root/reference).  Host facts (numpy version and SIMD dispatch)
are recorded in ``meta.json``.
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import zlinalg as Z  # noqa: E402  (reference, read-only)
from paper_2112_06465_b200 import problems  # noqa: E402


def rz(n, rng):
    return rng.random(n) + 1j * rng.random(n)


def rn(n, rng):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def random_sparse(n_rows, n_cols, density, rng, long_rows=()):
    dense = np.zeros((n_rows, n_cols), dtype=np.complex128)
    mask = rng.random((n_rows, n_cols)) < density
    for r in long_rows:
        mask[r % n_rows, :] = rng.random(n_cols) < 0.9
    cnt = int(mask.sum())
    dense[mask] = rng.standard_normal(cnt) + 1j * rng.standard_normal(cnt)
    return dense


def dense_to_csr(dense):
    coo = Z.CooMatrix(*dense.shape)
    for i, j in zip(*np.nonzero(dense)):
        coo.add(int(i), int(j), complex(dense[i, j]))
    return Z.coo_to_csr(coo)


def dominant(n, density, seed):
    rng = np.random.default_rng(seed)
    dense = random_sparse(n, n, density, rng)
    np.fill_diagonal(dense, 0)
    off = np.sum(np.abs(dense), axis=1)
    phase = np.exp(1j * rng.uniform(-0.4, 0.4, n))
    np.fill_diagonal(dense, (off + 2.0) * phase)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return dense_to_csr(dense), b


def vecops_goldens():
    out = {}
    sizes = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 63, 64, 65, 66, 127, 128, 129, 130, 200,
             4095, 4096, 4097, 8191, 8193, 20000, 65537]
    for n in sizes:
        rng = np.random.default_rng(1000 + n)
        x, y, mv = rz(n, rng), rz(n, rng), rn(n, rng)
        if n > 10:  # exercise signed zeros and exact zeros
            x[3] = -0.0 - 0.0j
            y[5] = 0.0
        a = complex(rng.random(), rng.random())
        X, Y = Z.ZVector(x.copy()), Z.ZVector(y.copy())
        rec = dict(x=x, y=y, minv=mv, alpha=np.array([a]))
        for conj in (True, False):
            tag = "c" if conj else "u"
            rec[f"dot_{tag}_4096"] = np.array([complex(Z.zdot(X, Y, conj))])
            rec[f"dot_{tag}_64"] = np.array([complex(Z.zdot(X, Y, conj, Z.ReductionPlan(64)))])
            rec[f"dot_{tag}_65536"] = np.array([complex(Z.zdot(X, Y, conj, Z.ReductionPlan(65536)))])
            if n <= 20000:
                rec[f"dot_{tag}_seq"] = np.array(
                    [complex(Z.zdot(X, Y, conj, Z.ReductionPlan(mode=Z.SEQUENTIAL)))])
        rec["norm_4096"] = np.array([Z.znorm2(X)])
        rec["norm_64"] = np.array([Z.znorm2(X, Z.ReductionPlan(64))])
        rec["norm_65536"] = np.array([Z.znorm2(X, Z.ReductionPlan(65536))])
        if n <= 20000:
            rec["norm_seq"] = np.array([Z.znorm2(X, Z.ReductionPlan(mode=Z.SEQUENTIAL))])
        if n > 4097:  # elementwise kernels are size-independent; keep fixtures small
            for k, v in rec.items():
                if k != "minv":
                    out[f"n{n}__{k}"] = v
            continue
        rec["axpy"] = Z.zaxpy(a, X, Z.ZVector(y.copy())).data
        rec["scal"] = Z.zscal(a, Z.ZVector(x.copy())).data
        rec["axmy"] = Z.zaxmy(X, Z.ZVector(y.copy())).data
        rec["jacobi"] = Z.Preconditioner("jacobi", mv).apply(X).data
        for k, v in rec.items():
            out[f"n{n}__{k}"] = v
    return out


def spmv_goldens():
    out = {}
    cases = []
    rng = np.random.default_rng(1234)
    for i in range(30):  # test_sparse.py:135-146 shapes: rectangular, [1,120)
        nr, nc = int(rng.integers(1, 120)), int(rng.integers(1, 120))
        cases.append((f"rand{i}", random_sparse(nr, nc, float(rng.uniform(0.01, 0.2)), rng)))
    # long rows: pairwise tree with splits (row length > 65)
    cases.append(("long", random_sparse(40, 700, 0.05, rng, long_rows=(0, 7, 13, 39))))
    # empty rows and an empty matrix row block
    d = random_sparse(50, 50, 0.1, rng)
    d[10:20, :] = 0
    cases.append(("emptyrows", d))
    mats = [(name, dense_to_csr(dd)) for name, dd in cases]
    # around the numpy temporary-elision threshold (nnz*16 >= 256 KiB)
    for tag, cells in (("fd_below", 23), ("fd_above", 27)):
        n, ia, ja, aa, _ = problems.helmholtz_fd(3, cells, frequency=1.3, damping=0.2)
        mats.append((tag, Z.CsrMatrix(n, n, aa, ja, ia)))
    for name, A in mats:
        x = rn(A.n_cols, rng)
        y = Z.spmv(A, Z.ZVector(x)).data
        out[f"{name}__shape"] = np.array([A.n_rows, A.n_cols])
        out[f"{name}__ia"] = A.ia
        out[f"{name}__ja"] = A.ja
        out[f"{name}__aa"] = A.aa
        out[f"{name}__x"] = x
        out[f"{name}__y"] = y
    return out


def solver_cases():
    cases = []
    # the reference CPU path shape at reduced size (load_problem_config-style)
    for cells, freq in ((9, 1.0), (13, 1.5), (17, 2.0)):
        p = Z.HelmholtzProblem(dim=3, cells_per_axis=cells, frequency=freq, source=1 + 0j)
        A, b = Z.assemble(p)
        cases.append((f"fd{cells}", A, b.data, "jacobi", 1e-8, 1000, None))
    # complex-damped indefinite systems (multi-block dots, SpMV above elision)
    for cells, freq, eps in ((21, 21 / 12.0, 0.3), (29, 29 / 12.0, 0.3)):
        n, ia, ja, aa, b = problems.helmholtz_fd(3, cells, frequency=freq, damping=eps)
        cases.append((f"damped{cells}", Z.CsrMatrix(n, n, aa, ja, ia), b, "jacobi", 1e-8, 2000, None))
    n, ia, ja, aa, b = problems.helmholtz_27pt(14, k2=100.0, damping=0.05)
    cases.append(("s27_14", Z.CsrMatrix(n, n, aa, ja, ia), b, "jacobi", 1e-8, 2000, None))
    # random dominant systems, acceptance criterion 4 seeds (test_acceptance.py:115-131)
    for n, seed in ((10, 300), (50, 310), (200, 320), (200, 321)):
        A, b = dominant(n, 0.1, seed)
        cases.append((f"dom{n}_{seed}", A, b, "jacobi", 1e-9, 1000, None))
    A, b = dominant(40, 0.15, 33)
    cases.append(("dom40_identity", A, b, "identity", 1e-9, 1000, None))
    A, b = dominant(80, 0.1, 5)
    cases.append(("dom80_maxit3", A, b, "jacobi", 1e-30, 3, None))
    A, b = dominant(30, 0.2, 14)
    g = np.random.default_rng(99)
    cases.append(("dom30_guess", A, b, "jacobi", 1e-9, 1000, g.standard_normal(30) + 1j * g.standard_normal(30)))
    # identity system, 1 iteration (test_krylov.py:43-54)
    A = Z.CsrMatrix.identity(5)
    cases.append(("ident5", A, np.array([1 + 2j, -3, 0.25j, 4, -1 - 1j]), "identity", 1e-9, 1000, None))
    # zero rhs
    A, _ = dominant(10, 0.3, 2)
    cases.append(("zero_rhs", A, np.zeros(10, dtype=np.complex128), "identity", 1e-9, 1000, None))
    # breakdown: rotation (test_krylov.py:35-40)
    coo = Z.CooMatrix(2, 2)
    coo.add(0, 1, -1)
    coo.add(1, 0, 1)
    cases.append(("rotation", Z.coo_to_csr(coo), np.array([1, 0], dtype=np.complex128), "identity", 1e-9, 1000, None))
    # the BASELINE C1 configuration itself (reference CPU path)
    n, ia, ja, aa, b = problems.config_problem("C1")
    cases.append(("C1", Z.CsrMatrix(n, n, aa, ja, ia), b, "jacobi", 1e-8, 1000, None))
    return cases


def solver_goldens():
    out = {}
    for name, A, b, prec, tol, maxit, guess in solver_cases():
        M = Z.build_jacobi(A) if prec == "jacobi" else Z.Preconditioner.identity()
        cfg = Z.SolverConfig(tolerance=tol, max_iterations=maxit,
                             initial_guess=Z.ZVector(guess.copy()) if guess is not None else None)
        status, what = "converged", ""
        try:
            x, rep = Z.solve_bicgstab(A, Z.ZVector(np.asarray(b, dtype=np.complex128).copy()), M, cfg)
            if not rep.converged:
                status = "not_converged"
            xd = x.data
        except Z.BreakdownError as e:
            rep, status, what, xd = e.report, "breakdown", str(e), np.zeros(0, dtype=np.complex128)
        out[f"{name}__ia"] = A.ia
        out[f"{name}__ja"] = A.ja
        out[f"{name}__aa"] = A.aa
        out[f"{name}__b"] = np.asarray(b, dtype=np.complex128)
        out[f"{name}__minv"] = M.data if prec == "jacobi" else np.zeros(0, dtype=np.complex128)
        out[f"{name}__guess"] = guess if guess is not None else np.zeros(0, dtype=np.complex128)
        out[f"{name}__params"] = np.array([tol, maxit])
        out[f"{name}__x"] = xd
        out[f"{name}__hist"] = np.array(rep.residual_history)
        out[f"{name}__status"] = np.array([status])
        out[f"{name}__what"] = np.array([what])
        print(f"  {name}: n={A.n_rows} nnz={A.nnz} {status} it={rep.iterations} "
              f"rel={rep.final_relative_residual:.3e}")
    return out


def krylov_ext_goldens():
    """BiCGSTAB(l) (l = 2, 8) and TFQMR (krylov.py:298-489) on a subset of the
    BiCGStab cases, for tests/test_krylov_ext_gpu.py."""
    keep = {"fd9", "fd13", "damped21", "s27_14", "dom50_310", "dom200_320", "dom40_identity", "dom80_maxit3",
            "dom30_guess", "ident5", "zero_rhs", "rotation"}
    out = {}
    for name, A, b, prec, tol, maxit, guess in solver_cases():
        if name not in keep:
            continue
        M = Z.build_jacobi(A) if prec == "jacobi" else Z.Preconditioner.identity()
        for solver, ell in (("bicgstabl", 2), ("bicgstabl", 8), ("tfqmr", 8)):
            tag = f"{name}_{solver}{ell if solver == 'bicgstabl' else ''}"
            cfg = Z.SolverConfig(tolerance=tol, max_iterations=maxit, l=ell,
                                 initial_guess=Z.ZVector(guess.copy()) if guess is not None else None)
            fn = Z.solve_bicgstab_l if solver == "bicgstabl" else Z.solve_tfqmr
            status, what = "converged", ""
            try:
                x, rep = fn(A, Z.ZVector(np.asarray(b, dtype=np.complex128).copy()), M, cfg)
                if not rep.converged:
                    status = "not_converged"
                xd = x.data
            except Z.BreakdownError as e:
                rep, status, what, xd = e.report, "breakdown", str(e), np.zeros(0, dtype=np.complex128)
            out[f"{tag}__ia"], out[f"{tag}__ja"], out[f"{tag}__aa"] = A.ia, A.ja, A.aa
            out[f"{tag}__b"] = np.asarray(b, dtype=np.complex128)
            out[f"{tag}__minv"] = M.data if prec == "jacobi" else np.zeros(0, dtype=np.complex128)
            out[f"{tag}__guess"] = guess if guess is not None else np.zeros(0, dtype=np.complex128)
            out[f"{tag}__params"] = np.array([tol, maxit, ell])
            out[f"{tag}__solver"] = np.array([solver])
            out[f"{tag}__x"] = xd
            out[f"{tag}__hist"] = np.array(rep.residual_history)
            out[f"{tag}__status"] = np.array([status])
            out[f"{tag}__what"] = np.array([what])
            print(f"  {tag}: n={A.n_rows} {status} it={rep.iterations} rel={rep.final_relative_residual:.3e}")
    return out


def problem_goldens():
    out = {}
    for dim, cells, freq in ((1, 12, 0.7), (2, 11, 1.1), (3, 9, 1.0), (3, 13, 1.5)):
        p = Z.HelmholtzProblem(dim=dim, cells_per_axis=cells, frequency=freq, source=1 + 0j)
        A, b = Z.assemble(p)
        tag = f"fd{dim}_{cells}"
        out[f"{tag}__params"] = np.array([dim, cells, freq])
        out[f"{tag}__ia"], out[f"{tag}__ja"], out[f"{tag}__aa"], out[f"{tag}__b"] = A.ia, A.ja, A.aa, b.data
    return out


def main():
    if sys.argv[1:] == ["krylov_ext"]:  # add the BiCGSTAB(l)/TFQMR fixtures only
        np.savez_compressed(os.path.join(HERE, "krylov_ext.npz"), **krylov_ext_goldens())
        return
    from numpy._core._multiarray_umath import __cpu_dispatch__, __cpu_baseline__
    meta = dict(numpy=np.__version__, python=sys.version.split()[0], cpu_baseline=list(__cpu_baseline__),
                cpu_dispatch=list(__cpu_dispatch__), reference=REF, generator=os.path.basename(__file__))
    print("vecops ...")
    np.savez_compressed(os.path.join(HERE, "vecops.npz"), **vecops_goldens())
    print("spmv ...")
    np.savez_compressed(os.path.join(HERE, "spmv.npz"), **spmv_goldens())
    print("problems ...")
    np.savez_compressed(os.path.join(HERE, "problems.npz"), **problem_goldens())
    print("solvers ...")
    np.savez_compressed(os.path.join(HERE, "bicgstab.npz"), **solver_goldens())
    np.savez_compressed(os.path.join(HERE, "krylov_ext.npz"), **krylov_ext_goldens())
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
