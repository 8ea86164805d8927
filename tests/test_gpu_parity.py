"""Bitwise parity of the CUDA path with the reference (golden vectors made
by the live reference) and with the C oracle (larger seeded inputs).

Everything here calls the product through its public API, which goes
through the C ABI of libzk.so.  Comparisons are on raw bytes: SpMV, level-1
and BiCGStab results must be the reference's bits, not merely close.
"""
import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from oracle import oracle as O
from paper_2112_06465_b200 import problems
from helpers import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _arith():
    Z.set_arithmetic(True, 262144)
    O.set_arith(True, 262144)


# ---- level 1 vs golden ---------------------------------------------------------

def test_vecops_golden(vecops_golden):
    for case, g in vecops_golden.items():
        X, Y = Z.ZVector(g["x"].copy()), Z.ZVector(g["y"].copy())
        for conj, tag in ((True, "c"), (False, "u")):
            for bs in (64, 4096, 65536):
                got = complex(Z.zdot(X, Y, conj, Z.ReductionPlan(bs)))
                assert bits([got]) == bits(g[f"dot_{tag}_{bs}"]), (case, tag, bs)
            if f"dot_{tag}_seq" in g:
                got = complex(Z.zdot(X, Y, conj, Z.ReductionPlan(mode=Z.SEQUENTIAL)))
                assert bits([got]) == bits(g[f"dot_{tag}_seq"]), (case, tag)
        for bs in (64, 4096, 65536):
            assert np.float64(Z.znorm2(X, Z.ReductionPlan(bs))).tobytes() == g[f"norm_{bs}"].tobytes(), (case, bs)
        if "norm_seq" in g:
            assert np.float64(Z.znorm2(X, Z.ReductionPlan(mode=Z.SEQUENTIAL))).tobytes() == g["norm_seq"].tobytes()
        if "axpy" in g:
            a = complex(g["alpha"][0])
            assert bits(Z.zaxpy(a, X, Z.ZVector(g["y"].copy())).data) == bits(g["axpy"]), case
            assert bits(Z.zscal(a, Z.ZVector(g["x"].copy())).data) == bits(g["scal"]), case
            assert bits(Z.zaxmy(X, Z.ZVector(g["y"].copy())).data) == bits(g["axmy"]), case
            M = Z.Preconditioner("jacobi", g["minv"])
            assert bits(M.apply(X).data) == bits(g["jacobi"]), case


@pytest.mark.parametrize("n", [1_000_000, 3 * 4096 + 17, 10_000_019])
def test_zdot_znorm2_vs_oracle_large(n):
    rng = np.random.default_rng(n)
    x = rng.random(n) + 1j * rng.random(n)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    X, Y = Z.ZVector(x), Z.ZVector(y)
    for conj in (True, False):
        assert bits([complex(Z.zdot(X, Y, conj))]) == bits([O.zdot(x, y, conj)])
    assert Z.znorm2(Y) == O.znorm2(y)
    assert Z.znorm2(X, Z.ReductionPlan(65536)) == O.znorm2(x, 65536)


def test_reductions_signalling_nan_inputs():
    """The streaming fold marks empty partial slots with a signalling NaN
    (zk_blas1.cu kSlotEmpty); inputs holding that exact pattern must still
    give quiet-NaN results, never a hang (arithmetic quiets sNaN)."""
    snan = np.frombuffer(np.uint64(0x7FF47FF47FF47FF4).tobytes(), dtype=np.float64)[0]
    for n, bs in ((64 * 5 + 1, 64), (4096 * 3 + 1, 4096), (1, 64)):
        x = np.ones(n, dtype=np.complex128)
        x.real[::bs] = snan
        x.imag[-1] = snan
        X = Z.ZVector(x)
        plan = Z.ReductionPlan(bs)
        assert np.isnan(complex(Z.zdot(X, X, True, plan)).real)
        assert np.isnan(Z.znorm2(X, plan))
        y = np.ones(n, dtype=np.complex128)  # and the slots are clean again afterwards
        Y = Z.ZVector(y)
        assert complex(Z.zdot(Y, Y, True, plan)) == O.zdot(y, y, True, bs)
        assert Z.znorm2(Y, plan) == O.znorm2(y, bs)


# ---- SpMV ------------------------------------------------------------------------

def test_spmv_golden(spmv_golden):
    for case, g in spmv_golden.items():
        nr, nc = (int(v) for v in g["shape"])
        A = Z.CsrMatrix(nr, nc, g["aa"], g["ja"], g["ia"])
        y = Z.spmv(A, Z.ZVector(g["x"]))
        assert bits(y.data) == bits(g["y"]), case


@pytest.mark.parametrize("kind", ["fd7_damped", "fd7_undamped", "s27", "ragged"])
def test_spmv_vs_oracle_large(kind):
    rng = np.random.default_rng(7)
    if kind == "fd7_damped":
        n, ia, ja, aa, _ = problems.helmholtz_fd(3, 65, frequency=5.0, damping=0.3)
    elif kind == "fd7_undamped":
        n, ia, ja, aa, _ = problems.helmholtz_fd(3, 41, frequency=2.0)
    elif kind == "s27":
        n, ia, ja, aa, _ = problems.helmholtz_27pt(40)
    else:  # ragged rows incl. empty, short (<5) and long (> 65) rows, random values
        n = 20000
        lens = rng.integers(0, 12, n)
        lens[rng.integers(0, n, 40)] = rng.integers(66, 400, 40)
        lens[:50] = 0
        ia = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=ia[1:])
        ja = np.concatenate([np.sort(rng.choice(n, size=int(k), replace=False)) for k in lens]).astype(np.int64)
        aa = rng.standard_normal(ia[-1]) + 1j * rng.standard_normal(ia[-1])
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = Z.spmv(A, Z.ZVector(x)).data
    assert bits(y) == bits(O.spmv(n, n, ia, ja, aa, x))


# ---- BiCGStab --------------------------------------------------------------------

def _solve_golden(g):
    n = g["b"].shape[0]
    A = Z.CsrMatrix(n, n, g["aa"], g["ja"], g["ia"])
    M = Z.Preconditioner("jacobi", g["minv"]) if g["minv"].size else Z.Preconditioner.identity()
    tol, maxit = float(g["params"][0]), int(g["params"][1])
    guess = Z.ZVector(g["guess"].copy()) if g["guess"].size else None
    cfg = Z.SolverConfig(tolerance=tol, max_iterations=maxit, initial_guess=guess)
    return Z.solve_bicgstab(A, Z.ZVector(g["b"].copy()), M, cfg)


def test_bicgstab_golden(bicgstab_golden):
    for case, g in bicgstab_golden.items():
        status = str(g["status"][0])
        if status == "breakdown":
            with pytest.raises(Z.BreakdownError) as info:
                _solve_golden(g)
            assert str(info.value) == str(g["what"][0]), case
            assert np.array(info.value.report.residual_history).tobytes() == g["hist"].tobytes(), case
            continue
        x, rep = _solve_golden(g)
        assert np.array(rep.residual_history).tobytes() == g["hist"].tobytes(), case
        assert rep.converged == (status == "converged"), case
        assert rep.iterations == len(g["hist"]) - 1, case
        assert bits(x.data) == bits(g["x"]), case


@pytest.mark.parametrize("shape", [("fd", 49, 49 / 12.0, 0.3), ("s27", 30, 0, 0), ("fd", 65, 3.0, 0.0),
                                   ("fe", 24, 0, 0)])
def test_bicgstab_vs_oracle_multiblock(shape):
    """Larger systems (many 4096-row blocks, partial tail block) vs the C oracle."""
    kind, m, freq, eps = shape
    if kind == "fd":
        n, ia, ja, aa, b = problems.helmholtz_fd(3, m, frequency=freq, damping=eps)
    elif kind == "fe":  # BASELINE C3 shape (P1-FE cylinder), irregular rows
        n, ia, ja, aa, b = problems.cylinder_p1fe(m)
    else:
        n, ia, ja, aa, b = problems.helmholtz_27pt(m, k2=100.0, damping=0.05)
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    M = Z.build_jacobi(A)
    x, rep = Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-8, max_iterations=3000))
    xo, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, M.data, None, 1e-8, 3000)
    assert rep.iterations == it
    assert np.array(rep.residual_history).tobytes() == np.array(hist).tobytes()
    assert bits(x.data) == bits(xo)


def test_c3_spmv_and_capped_solve_vs_oracle():
    """BASELINE C3 itself (996k rows, 14.7M nnz): SpMV and a capped solve, bitwise."""
    n, ia, ja, aa, b = problems.config_problem("C3")
    A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
    rng = np.random.default_rng(5)
    xv = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert bits(Z.spmv(A, Z.ZVector(xv)).data) == bits(O.spmv(n, n, ia, ja, aa, xv))
    M = Z.build_jacobi(A)
    x, rep = Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-8, max_iterations=20))
    xo, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, M.data, None, 1e-8, 20)
    assert rep.iterations == it == 20
    assert np.array(rep.residual_history).tobytes() == np.array(hist).tobytes()
    assert bits(x.data) == bits(xo)


@pytest.mark.parametrize("kind", ["fd", "s27", "fe"])
def test_spmv_dot_fused_vs_oracle(kind):
    """zk_spmv_dotc: y = A x and <w, y> in one pass == spmv then zdot, bitwise."""
    from paper_2112_06465_b200.sparse import spmv_dot
    if kind == "fd":
        n, ia, ja, aa, b = problems.helmholtz_fd(3, 49, frequency=4.0, damping=0.3)
    elif kind == "s27":
        n, ia, ja, aa, b = problems.helmholtz_27pt(30)
    else:
        n, ia, ja, aa, b = problems.cylinder_p1fe(24)
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    rng = np.random.default_rng(11)
    xv = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    wv = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y, d = spmv_dot(A, Z.ZVector(xv), Z.ZVector(wv))
    yo = O.spmv(n, n, ia, ja, aa, xv)
    assert bits(y.data) == bits(yo)
    assert complex(d) == O.zdot(wv, yo)
    y2, d2 = spmv_dot(A, Z.ZVector(xv), Z.ZVector(wv), conjugate=False)
    assert complex(d2) == O.zdot(wv, yo, conjugate=False)


def test_solver_host_loop_matches_graph(monkeypatch, bicgstab_golden):
    """The CUDA-graph WHILE loop and the host-driven loop are the same kernels."""
    monkeypatch.setenv("ZK_SOLVER_LOOP", "host")
    g = bicgstab_golden["damped21"]
    x, rep = _solve_golden(g)
    assert np.array(rep.residual_history).tobytes() == g["hist"].tobytes()
    assert bits(x.data) == bits(g["x"])


def test_solver_reuse_and_determinism(bicgstab_golden):
    g = bicgstab_golden["fd13"]
    r1 = _solve_golden(g)
    r2 = _solve_golden(g)
    assert r1[1].residual_history == r2[1].residual_history
    assert bits(r1[0].data) == bits(r2[0].data)


def _wide_dominant(n, lo, hi, seed):
    """Diagonally dominant matrix with lo..hi entries per row (wide SELL
    slices: few ring stages, so stages are reused within and across blocks)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, n)
    ia = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=ia[1:])
    rows, cols, vals = [], [], []
    for i, k in enumerate(lens):
        c = np.sort(rng.choice(np.setdiff1d(np.arange(max(0, i - 200), min(n, i + 200)), [i]), k - 1, replace=False))
        c = np.sort(np.append(c, i))
        v = rng.standard_normal(k) + 1j * rng.standard_normal(k)
        v[c == i] = (np.abs(v).sum() + 2.0) * np.exp(1j * rng.uniform(-0.4, 0.4))
        cols.append(c)
        vals.append(v)
    ja = np.concatenate(cols).astype(np.int64)
    aa = np.concatenate(vals)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return ia, ja, aa, b


@pytest.mark.parametrize("n,lo,hi", [(200, 30, 45), (9000, 40, 65), (13000, 60, 65)])
def test_wide_rows_stage_reuse(n, lo, hi):
    """Regression: ring stages shared by several consumer warps raced (the
    mbarrier parity wait cannot tell use u from use u+2)."""
    ia, ja, aa, b = _wide_dominant(n, lo, hi, seed=n)
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for _ in range(3):
        assert bits(Z.spmv(A, Z.ZVector(x)).data) == bits(O.spmv(n, n, ia, ja, aa, x))
    M = Z.build_jacobi(A)
    xo, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, M.data, None, 1e-10, 500)
    for _ in range(3):
        xs, rep = Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-10, max_iterations=500))
        assert rep.residual_history == hist
        assert bits(xs.data) == bits(xo)


@pytest.mark.parametrize("swap", [False, True])
def test_long_rows_warp_path_vs_oracle(swap):
    """Rows longer than 65 entries (side CSR, one warp per row): lengths
    around the leaf / chunk / split boundaries and up to 60k entries, mixed
    with short and empty rows in the same slices, both elision orders."""
    rng = np.random.default_rng(2024)
    n_rows, n_cols = 300, 70000
    lens = rng.integers(0, 12, n_rows)
    special = [66, 67, 129, 130, 200, 897, 898, 1793, 5000, 20001, 60000]
    for k, L in enumerate(special):
        lens[7 + 23 * k] = L
    ia = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ja = np.concatenate([np.sort(rng.choice(n_cols, L, replace=False)) for L in lens]).astype(np.int64)
    aa = rng.standard_normal(ia[-1]) + 1j * rng.standard_normal(ia[-1])
    x = rng.standard_normal(n_cols) + 1j * rng.standard_normal(n_cols)
    elide = 16 if swap else 1 << 62  # force numpy's elided (swapped) product order or not
    Z.set_arithmetic(True, elide)
    O.set_arith(True, elide)
    try:
        A = Z.CsrMatrix(n_rows, n_cols, aa, ja, ia)
        assert bits(Z.spmv(A, Z.ZVector(x)).data) == bits(O.spmv(n_rows, n_cols, ia, ja, aa, x))
    finally:
        Z.set_arithmetic(True, 262144)
        O.set_arith(True, 262144)


def test_solver_graph_follows_arithmetic_changes():
    """The captured solver graph carries the fingerprint in its kernel
    parameters (FMA formula, numpy's elision swap): changing it with
    set_arithmetic between solves must rebuild the graph, not replay stale
    parameters."""
    n, ia, ja, aa, b = problems.helmholtz_fd(3, 41, frequency=41 / 12.0, damping=0.3)  # 64000 rows, nnz > 16384
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    M = Z.build_jacobi(A)
    minv = M.data
    cfg = Z.SolverConfig(tolerance=1e-8, max_iterations=40)
    try:
        for fma, elide in ((True, 262144), (True, 1 << 62), (False, 262144), (True, 262144)):
            Z.set_arithmetic(fma, elide)
            O.set_arith(fma, elide)
            x, rep = Z.solve_bicgstab(A, Z.ZVector(b), Z.Preconditioner("jacobi", minv), cfg)
            xo, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, minv, None, 1e-8, 40)
            assert np.array(rep.residual_history).tobytes() == np.array(hist).tobytes(), (fma, elide)
            assert bits(x.data) == bits(xo), (fma, elide)
    finally:
        Z.set_arithmetic(True, 262144)
        O.set_arith(True, 262144)


@pytest.mark.parametrize("fma,elide", [(True, 262144), (True, 1 << 62), (True, 16), (False, 262144)])
def test_narrow_path_vs_oracle(monkeypatch, fma, elide):
    """Matrices at most 8 / 16 entries wide take the narrow kernels (per-warp
    TMA double buffer; ZK_NARROW=0 the ring): ragged rows with empty rows,
    whole empty slices, a partial last slice, both elision orders and both
    product formulas -- every width class and the ring the oracle's bits, in
    SpMV and in BiCGStab solves (whose SpMV phases, the two-vector one
    included, use the same kernels)."""
    rng = np.random.default_rng(88)
    n = 70001  # partial last slice; > 16 warps x 2 CTAs x 148 SMs of slices
    Z.set_arithmetic(fma, elide)
    O.set_arith(fma, elide)
    try:
        for wmax in (8, 16):
            lens = rng.integers(0, wmax + 1, n)
            lens[64:128] = 0  # two empty slices
            lens[1000:1040] = wmax
            ia = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            ja = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int64)
            aa = rng.standard_normal(ia[-1]) + 1j * rng.standard_normal(ia[-1])
            x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            want = bits(O.spmv(n, n, ia, ja, aa, x))
            for mode in ("16", "8", "0"):
                monkeypatch.setenv("ZK_NARROW", mode)
                A = Z.CsrMatrix(n, n, aa, ja, ia)
                assert bits(Z.spmv(A, Z.ZVector(x)).data) == want, (wmax, mode)
        monkeypatch.delenv("ZK_NARROW")
        # a width-16 system through the solver (two-vector SpMV phase)
        ia, ja, aa, b = _wide_dominant(3000, 9, 16, seed=5)
        A = Z.CsrMatrix(3000, 3000, aa, ja, ia)
        M = Z.build_jacobi(A)
        xs, rep = Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-10, max_iterations=200))
        xo, hist, it, st, _ = O.bicgstab(3000, ia, ja, aa, b, M.data, None, 1e-10, 200)
        assert rep.residual_history == hist and bits(xs.data) == bits(xo)
        # a diagonally dominant narrow system for the solver
        m, ia2, ja2, aa2, b = problems.helmholtz_fd(3, 33, frequency=33 / 12.0, damping=0.3)
        A = Z.CsrMatrix(m, m, aa2, ja2, ia2)
        M = Z.build_jacobi(A)
        xs, rep = Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-8, max_iterations=60))
        xo, hist, it, st, _ = O.bicgstab(m, ia2, ja2, aa2, b, M.data, None, 1e-8, 60)
        assert rep.residual_history == hist and bits(xs.data) == bits(xo)
    finally:
        Z.set_arithmetic(True, 262144)
        O.set_arith(True, 262144)


@pytest.mark.parametrize("seed", range(12))
def test_narrow_path_random_shapes(seed):
    """Random small/odd shapes through the narrow kernels (n from 1 to a few
    slices past a multiple of 32, rectangular, widths 0..16 with empty
    slices), SpMV bitwise against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 2, 31, 32, 33, 63, 65, 257, 1000, 4097, 5003, 40961]))
    ncols = int(max(1, n + rng.integers(-min(n - 1, 5), 40)))
    wmax = int(rng.choice([1, 3, 7, 8, 9, 12, 16]))
    lens = rng.integers(0, wmax + 1, n)
    if n > 64:
        lens[32:64] = 0  # an empty slice in the middle
    lens = np.minimum(lens, ncols)
    ia = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ja = (np.concatenate([np.sort(rng.choice(ncols, int(L), replace=False)) for L in lens])
          if ia[-1] else np.zeros(0)).astype(np.int64)
    aa = rng.standard_normal(ia[-1]) + 1j * rng.standard_normal(ia[-1])
    x = rng.standard_normal(ncols) + 1j * rng.standard_normal(ncols)
    A = Z.CsrMatrix(n, ncols, aa, ja, ia)
    assert bits(Z.spmv(A, Z.ZVector(x)).data) == bits(O.spmv(n, ncols, ia, ja, aa, x)), (n, ncols, wmax)
