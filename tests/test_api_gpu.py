"""The reference test-suite's hot-path behaviour, run against this package.

Each test restates a check from /root/reference/pkg/tests (cited) so the
drop-in is held to the same contract: level-1 kernels (test_vecops.py),
SpMV (test_sparse.py), BiCGStab (test_krylov.py) and acceptance criteria 3,
4, 5 and 9 (test_acceptance.py), all executed on the GPU through libzk.
"""
import math

import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from helpers import GOLDEN_5X5_DENSE, bits, dense_to_csr, random_dominant_system, random_sparse_dense

pytestmark = pytest.mark.gpu

SEQ = Z.ReductionPlan(mode=Z.SEQUENTIAL)


def rand_zv(n, seed=0):
    rng = np.random.default_rng(seed)
    return Z.ZVector(rng.random(n) + 1j * rng.random(n))


# ---- test_vecops.py ------------------------------------------------------------

def test_zassign_copies():  # test_vecops.py:105-112
    src = Z.ZVector.from_values([1 + 2j, 3 + 4j])
    dst = Z.ZVector.zeros(2)
    assert Z.zassign(dst, src) is dst
    assert np.array_equal(dst.data, src.data)
    src.data[0] = 9
    assert dst.data[0] == 1 + 2j


def test_zscal_examples():  # test_vecops.py:121-131
    x = Z.ZVector.from_values([1 + 1j, -2j])
    Z.zscal(Z.Cplx(1, 0), x)
    assert np.array_equal(x.data, np.array([1 + 1j, -2j]))
    x = Z.ZVector.from_values([3 + 4j])
    Z.zscal(Z.Cplx(2, -1), x)
    assert x.data[0] == 10 + 5j


def test_zaxpy_examples():  # test_vecops.py:134-153
    y = Z.ZVector.from_values([5 + 5j, 1j])
    before = y.data.copy()
    Z.zaxpy(Z.Cplx(0, 0), rand_zv(2), y)
    assert np.array_equal(y.data, before)
    x0, y0 = rand_zv(500, 5), rand_zv(500, 6)
    a = Z.Cplx(0.7, -0.4)
    y = y0.copy()
    Z.zaxpy(a, x0, y)
    Z.zaxpy(-a, x0, y)
    scale = np.maximum(np.abs(y0.data), np.abs(complex(a) * x0.data))
    assert np.all(np.abs(y.data - y0.data) <= 4 * np.spacing(scale))


def test_zaxmy_examples():  # test_vecops.py:156-169
    x = Z.ZVector.from_values([2 + 3j])
    y = Z.ZVector.from_values([4 - 5j])
    Z.zaxmy(x, y)
    assert y.data[0] == 23 + 2j


@pytest.mark.parametrize("kernel", ["zassign", "zaxpy", "zaxmy", "zdot"])
def test_length_mismatch_raises_before_any_write(kernel):  # test_vecops.py:172-187
    x, y = rand_zv(4, 1), rand_zv(3, 2)
    x0, y0 = x.data.copy(), y.data.copy()
    with pytest.raises(Z.DimensionError):
        {"zassign": lambda: Z.zassign(y, x), "zaxpy": lambda: Z.zaxpy(Z.Cplx(1, 1), x, y),
         "zaxmy": lambda: Z.zaxmy(x, y), "zdot": lambda: Z.zdot(x, y)}[kernel]()
    assert np.array_equal(x.data, x0) and np.array_equal(y.data, y0)


def test_pure_variants_leave_operands_alone():  # test_vecops.py:190-198
    x, y = rand_zv(8, 3), rand_zv(8, 4)
    x0, y0 = x.data.copy(), y.data.copy()
    Z.zscal_copy(2 + 1j, x)
    Z.zaxpy_copy(1 - 1j, x, y)
    Z.zaxmy_copy(x, y)
    assert np.array_equal(x.data, x0) and np.array_equal(y.data, y0)


def test_zdot_examples():  # test_vecops.py:201-209
    assert Z.zdot(rand_zv(6, 7), Z.ZVector.zeros(6)) == Z.Cplx(0, 0)
    x = Z.ZVector.from_values([1j])
    assert Z.zdot(x, x, conjugate=True) == Z.Cplx(1, 0)
    x = Z.ZVector.from_values([1 + 1j, 2 + 0j])
    y = Z.ZVector.from_values([1 - 1j, 3j])
    assert Z.zdot(x, y, conjugate=False) == Z.Cplx(2, 6)


def test_empty_vectors_are_legal_everywhere():  # test_vecops.py:212-220
    e = Z.ZVector.zeros(0)
    assert Z.zdot(e, e) == Z.Cplx(0, 0) and Z.zdot(e, e, plan=SEQ) == Z.Cplx(0, 0)
    assert Z.znorm2(e) == 0.0 and Z.znorm2(e, SEQ) == 0.0
    assert len(Z.zscal(2 + 1j, Z.ZVector.zeros(0))) == 0
    assert len(Z.zaxpy(1j, e, Z.ZVector.zeros(0))) == 0
    assert len(Z.zaxmy(e, Z.ZVector.zeros(0))) == 0


@pytest.mark.parametrize("n", [1, 2, 63, 64, 4095, 4096, 4097, 20000])
@pytest.mark.parametrize("conjugate", [True, False])
def test_zdot_sequential_matches_python_loop_bitwise(n, conjugate):  # test_vecops.py:223-230
    x, y = rand_zv(n, n), rand_zv(n, n + 1)
    acc = 0j
    for px, py in zip(x.data.tolist(), y.data.tolist()):
        acc += (px.conjugate() if conjugate else px) * py
    assert complex(Z.zdot(x, y, conjugate=conjugate, plan=SEQ)) == acc


@pytest.mark.parametrize("n", [1, 65, 4096, 100_000, 1_000_000])
def test_zdot_blocked_close_to_fsum(n):  # test_vecops.py:233-243
    x, y = rand_zv(n, 100 + n % 97), rand_zv(n, 200 + n % 89)
    got = complex(Z.zdot(x, y, True))
    prod = np.conj(x.data) * y.data
    want = complex(math.fsum(prod.real), math.fsum(prod.imag))
    assert abs(got - want) <= 1e-12 * max(abs(want), 1e-30)


def test_zdot_linearity():  # test_vecops.py:261-277
    rng = np.random.default_rng(21)
    for _ in range(10):
        n = int(rng.integers(1, 300))
        x, y, z = (Z.ZVector(rng.standard_normal(n) + 1j * rng.standard_normal(n)) for _ in range(3))
        a = complex(rng.standard_normal(), rng.standard_normal())
        lhs = complex(Z.zdot(x, Z.ZVector(a * y.data + z.data), conjugate=False))
        rhs = a * complex(Z.zdot(x, y, conjugate=False)) + complex(Z.zdot(x, z, conjugate=False))
        assert lhs == pytest.approx(rhs, rel=1e-10, abs=1e-12)


def test_znorm2_examples_and_consistency():  # test_vecops.py:280-299
    assert Z.znorm2(Z.ZVector.zeros(5)) == 0.0
    assert Z.znorm2(Z.ZVector.from_values([3 + 4j])) == 5.0
    for n in (1, 100, 4097, 50_000):
        x = rand_zv(n, 300 + n % 71)
        d = Z.zdot(x, x, conjugate=True)
        nrm = Z.znorm2(x)
        assert nrm * nrm == pytest.approx(d.re, rel=1e-12)
        assert abs(d.im) <= 1e-13 * nrm * nrm
    x = rand_zv(777, 31)
    acc = 0.0
    for z in x.data.tolist():
        acc += z.real * z.real + z.imag * z.imag
    assert Z.znorm2(x, SEQ) == math.sqrt(acc)


def test_zvector_wraps_without_copy_and_syncs_back():  # test_vecops.py:324-328
    data = np.ones(4, dtype=np.complex128)
    v = Z.ZVector(data)
    v.data[0] = 7j
    assert data[0] == 7j
    Z.zscal(2, v)              # device write ...
    assert v.data is data      # ... lands in the caller's array on read
    assert data[0] == 14j and data[1] == 2


def test_host_mutation_between_kernels_is_seen():
    v = Z.ZVector(np.arange(5, dtype=np.complex128))
    Z.zscal(2, v)
    v.data[1] = 100
    Z.zscal(1j, v)
    assert v.data[1] == 100j and v.data[2] == 4j


# ---- test_sparse.py ------------------------------------------------------------

def test_spmv_golden_row_sums():  # test_sparse.py:111-115
    y = Z.spmv(dense_to_csr(GOLDEN_5X5_DENSE), Z.ZVector.from_values([1] * 5))
    assert [complex(c) for c in y] == [17, 9, 8, 5, 16]


def test_spmv_empty_row_yields_zero():  # test_sparse.py:118-126
    d = np.zeros((3, 3), dtype=np.complex128)
    d[0, 0], d[2, 1] = 2, 1j
    y = Z.spmv(dense_to_csr(d), Z.ZVector.from_values([1, 1, 1]))
    assert complex(y[1]) == 0j and complex(y[0]) == 2 and complex(y[2]) == 1j


def test_spmv_dimension_mismatch():  # test_sparse.py:129-132
    with pytest.raises(Z.DimensionError):
        Z.spmv(dense_to_csr(GOLDEN_5X5_DENSE), Z.ZVector.zeros(4))


def test_spmv_matches_dense_oracle_rectangular():  # test_sparse.py:135-146, criterion 3
    rng = np.random.default_rng(1234)
    for _ in range(40):
        nr, nc = int(rng.integers(1, 120)), int(rng.integers(1, 120))
        dense = random_sparse_dense(nr, nc, float(rng.uniform(0.01, 0.2)), rng)
        x = Z.ZVector(rng.standard_normal(nc) + 1j * rng.standard_normal(nc))
        want = dense @ x.data
        got = Z.spmv(dense_to_csr(dense), x).data
        assert np.all(np.abs(got - want) <= 1e-12 * np.maximum(np.abs(want), 1e-30))


def test_spmv_row_independence():  # test_sparse.py:157-165
    rng = np.random.default_rng(6)
    dense = random_sparse_dense(60, 60, 0.15, rng)
    x = Z.ZVector(rng.standard_normal(60) + 1j * rng.standard_normal(60))
    perm = rng.permutation(60)
    a = Z.spmv(dense_to_csr(dense), x).data
    b = Z.spmv(dense_to_csr(dense[perm]), x).data
    assert bits(b) == bits(a[perm])


def test_zero_row_matrix():
    A = Z.CsrMatrix(0, 3, [], [], [0])
    assert len(Z.spmv(A, Z.ZVector.zeros(3))) == 0


# ---- test_krylov.py (BiCGStab) -----------------------------------------------

def _relres(A, x, b):
    return Z.znorm2(Z.ZVector(b.data - Z.spmv(A, x).data)) / Z.znorm2(b)


def test_identity_system_one_iteration():  # test_krylov.py:43-54
    A = Z.CsrMatrix.identity(5)
    b = Z.ZVector.from_values([1 + 2j, -3, 0.25j, 4, -1 - 1j])
    x, rep = Z.solve_bicgstab(A, b)
    assert rep.converged and rep.iterations == 1
    assert np.array_equal(x.data, b.data)
    assert rep.residual_history[0] == 1.0
    assert len(rep.residual_history) == rep.iterations + 1
    assert rep.residual_history[-1] == rep.final_relative_residual and rep.elapsed_ms >= 0


def test_jacobi_diagonal_one_iteration():  # test_krylov.py:57-69
    A = dense_to_csr(np.diag(np.full(6, 2 + 0j)))
    rng = np.random.default_rng(1)
    b = Z.ZVector(rng.standard_normal(6) + 1j * rng.standard_normal(6))
    x, rep = Z.solve_bicgstab(A, b, Z.build_jacobi(A))
    assert rep.converged and rep.iterations == 1
    assert np.allclose(x.data, b.data / 2, rtol=1e-12)


def test_dense_lu_oracle_50():  # test_krylov.py:72-79
    A, dense, b = random_dominant_system(50, 0.15, seed=42)
    x, rep = Z.solve_bicgstab(A, b, Z.build_jacobi(A), Z.SolverConfig())
    want = np.linalg.solve(dense, b.data)
    assert rep.converged and np.max(np.abs(x.data - want)) / np.max(np.abs(want)) <= 1e-6


def test_residual_truthful_and_history():  # test_krylov.py:128-144
    A, _, b = random_dominant_system(80, 0.1, seed=3)
    x, rep = Z.solve_bicgstab(A, b, Z.build_jacobi(A))
    assert rep.converged
    assert abs(_relres(A, x, b) - rep.final_relative_residual) <= 1e-10 * rep.final_relative_residual
    assert all(math.isfinite(r) and r >= 0 for r in rep.residual_history)


def test_identity_preconditioner_is_neutral():  # test_krylov.py:157-163
    A, _, b = random_dominant_system(40, 0.15, seed=33)
    x1, r1 = Z.solve_bicgstab(A, b, None)
    x2, r2 = Z.solve_bicgstab(A, b, Z.Preconditioner.identity())
    assert r1.residual_history == r2.residual_history and np.array_equal(x1.data, x2.data)


def test_scaling_equivariance():  # test_krylov.py:166-180
    A, dense, b = random_dominant_system(50, 0.15, seed=17)
    c = 0.7 - 0.3j
    Ac, bc = dense_to_csr(c * dense), Z.ZVector(c * b.data)
    x1, r1 = Z.solve_bicgstab(A, b, Z.build_jacobi(A))
    x2, r2 = Z.solve_bicgstab(Ac, bc, Z.build_jacobi(Ac))
    assert np.max(np.abs(x1.data - x2.data)) <= 1e-8 * np.max(np.abs(x1.data))
    assert len(r1.residual_history) == len(r2.residual_history)


def test_non_convergence_is_normal_return():  # test_krylov.py:183-190
    A, _, b = random_dominant_system(80, 0.1, seed=5)
    x, rep = Z.solve_bicgstab(A, b, Z.build_jacobi(A), Z.SolverConfig(tolerance=1e-30, max_iterations=3))
    assert not rep.converged and rep.iterations == 3 and len(rep.residual_history) == 4


def test_breakdown_raises_with_partial_report():  # test_krylov.py:193-202
    A = dense_to_csr(np.array([[0, -1], [1, 0]], dtype=np.complex128))
    with pytest.raises(Z.BreakdownError) as info:
        Z.solve_bicgstab(A, Z.ZVector.from_values([1, 0]), Z.Preconditioner.identity())
    rep = info.value.report
    assert rep is not None and not rep.converged and rep.residual_history[0] == 1.0


def test_zero_rhs_trivial():  # test_krylov.py:205-212
    A, _, _ = random_dominant_system(10, 0.3, seed=2)
    x, rep = Z.solve_bicgstab(A, Z.ZVector.zeros(10))
    assert rep.converged and rep.iterations == 0 and np.all(x.data == 0) and rep.final_relative_residual == 0.0


def test_zero_rhs_with_guess_returns_zero():
    A, _, _ = random_dominant_system(10, 0.3, seed=2)
    g = Z.ZVector(np.ones(10, dtype=np.complex128))
    x, rep = Z.solve_bicgstab(A, Z.ZVector.zeros(10), None, Z.SolverConfig(initial_guess=g))
    assert rep.iterations == 0 and np.all(x.data == 0)


def test_exact_guess_short_circuits_and_guess_untouched():  # test_krylov.py:215-237
    A, dense, b = random_dominant_system(20, 0.2, seed=13)
    exact = Z.ZVector(np.linalg.solve(dense, b.data))
    x, rep = Z.solve_bicgstab(A, b, None, Z.SolverConfig(initial_guess=exact))
    assert rep.converged and rep.iterations <= 1 and _relres(A, x, b) <= 1e-12
    A, dense, b = random_dominant_system(30, 0.2, seed=14)
    rng = np.random.default_rng(99)
    guess = Z.ZVector(rng.standard_normal(30) + 1j * rng.standard_normal(30))
    g0 = guess.data.copy()
    x, rep = Z.solve_bicgstab(A, b, Z.build_jacobi(A), Z.SolverConfig(initial_guess=guess))
    assert rep.converged and np.array_equal(guess.data, g0)


def test_dimension_checks():  # test_krylov.py:284-293
    A = Z.CsrMatrix.identity(3)
    with pytest.raises(Z.DimensionError):
        Z.solve_bicgstab(A, Z.ZVector.zeros(4))
    with pytest.raises(Z.DimensionError):
        Z.solve_bicgstab(Z.CsrMatrix(2, 3, [], [], [0, 0, 0]), Z.ZVector.zeros(2))
    with pytest.raises(Z.DimensionError):
        Z.solve_bicgstab(A, Z.ZVector.zeros(3), Z.Preconditioner("jacobi", np.ones(5, dtype=np.complex128)))


def test_build_jacobi_inverse_diagonal():  # test_krylov.py:240-250
    A = dense_to_csr(np.diag([2, 1j]))
    out = Z.build_jacobi(A).apply(Z.ZVector.from_values([1, 1]))
    assert out.data[0] == 0.5 and out.data[1] == -1j


def test_empty_system():
    x, rep = Z.solve_bicgstab(Z.CsrMatrix(0, 0, [], [], [0]), Z.ZVector.zeros(0))
    assert rep.converged and rep.iterations == 0 and len(x) == 0


# ---- acceptance criteria 4, 5 and 9 (test_acceptance.py:115-151, 234-254) ------

def _criterion_4():
    runs = []
    seeds = iter(range(300, 400))
    for n in (10, 50, 200):
        for _ in range(10):
            seed = next(seeds)
            A, dense, b = random_dominant_system(n, 0.1, seed=seed)
            want = np.linalg.solve(dense, b.data)
            x, rep = Z.solve_bicgstab(A, b, Z.build_jacobi(A), Z.SolverConfig(tolerance=1e-9))
            assert rep.converged
            assert np.max(np.abs(x.data - want)) / np.max(np.abs(want)) <= 1e-6
            runs.append((A, b, x, rep))
    return runs


def test_acceptance_4_5_9():
    first = _criterion_4()
    for A, b, x, rep in first:
        r = b.copy()
        r.data -= Z.spmv(A, x).data
        rec = Z.znorm2(r) / Z.znorm2(b)
        assert abs(rec - rep.final_relative_residual) <= 1e-10 * rep.final_relative_residual
    second = _criterion_4()
    for (_, _, xa, ra), (_, _, xb, rb) in zip(first, second):
        assert ra.residual_history == rb.residual_history and bits(xa.data) == bits(xb.data)


def test_build_jacobi_device_errors_and_values():  # krylov.py:106-120, test_krylov.py:240-250
    A = Z.CsrMatrix(2, 2, [1.0, 1.0], [0, 0], [0, 1, 2])
    with pytest.raises(Z.SingularPreconditionerError, match="row 1"):
        Z.build_jacobi(A)
    M = Z.build_jacobi(Z.CsrMatrix(2, 2, [2.0, 1j], [0, 1], [0, 1, 2]))
    assert M.data[0] == 0.5 and M.data[1] == -1j
    with pytest.raises(Z.SingularPreconditionerError, match="row 0"):  # explicit zero on the diagonal
        Z.build_jacobi(Z.CsrMatrix(2, 2, [0j, 1.0], [0, 1], [0, 1, 2]))


def test_build_jacobi_device_is_numpy_division_bitwise():
    """1 / d on the device == np.divide(1.0, d) (numpy's Smith variant), over
    magnitudes 1e-26..1e26, pure real / pure imaginary entries and signed
    zeros in the other part; rectangular shapes use min(n_rows, n_cols)."""
    rng = np.random.default_rng(7)
    n = 50000
    d = rng.standard_normal(n) * np.exp(rng.uniform(-60, 60, n)) + 1j * (
        rng.standard_normal(n) * np.exp(rng.uniform(-60, 60, n)))
    d[:500] = d[:500].real + 0j
    d[500:1000] = 1j * d[500:1000].imag
    d[1000:1500] = d[1000:1500].real - 0j
    A = Z.CsrMatrix(n, n, d, np.arange(n), np.arange(n + 1))
    assert bits(Z.build_jacobi(A).data) == bits(np.divide(1.0, d))
    # a dense-ish matrix with the diagonal among other entries, 3 x 5
    dense = rng.standard_normal((3, 5)) + 1j * rng.standard_normal((3, 5))
    from helpers import dense_to_csr
    A = dense_to_csr(dense)
    assert bits(Z.build_jacobi(A).data) == bits(np.divide(1.0, np.diag(dense)))


def test_build_jacobi_long_rows():
    """Diagonal entries inside rows longer than 65 (side CSR)."""
    n = 300
    rows, cols = [], []
    for i in range(n):
        cs = sorted(set([i] + list(range(0, n, 3)))) if i % 7 == 0 else [i]
        rows += [i] * len(cs)
        cols += cs
    rng = np.random.default_rng(3)
    vals = rng.standard_normal(len(cols)) + 1j * rng.standard_normal(len(cols))
    ia = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))])
    A = Z.CsrMatrix(n, n, vals, np.array(cols), ia)
    assert bits(Z.build_jacobi(A).data) == bits(np.divide(1.0, A.diagonal()))
