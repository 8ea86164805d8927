"""Bitwise parity at the BASELINE headline sizes (C4: 8M rows / 214M nnz,
C5: 16.8M rows / 117M nnz) -- the sizes where int32 column offsets, the
numpy elision swap (nnz >= 16384) and thousands of 4096-row reduction blocks
folded in order all matter at once.

Per configuration: one full-size SpMV (sparse.py:217-232) and a capped
Jacobi-BiCGStab solve (krylov.py:213-295, max_iterations=3) through the
public API, compared on raw bytes with the C oracle on the same inputs
(residual history, iteration count, solution).  The oracle is single-threaded
C: ~5 s per C4 iteration on the box's host, so the cap keeps each case under
a minute.
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


@pytest.fixture(scope="module", params=["C4", "C5"])
def headline(request):
    name = request.param
    n, ia, ja, aa, b = problems.config_problem(name)
    A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
    yield name, n, ia, ja, aa, b, A
    del A


def test_headline_spmv_bitwise(headline):
    name, n, ia, ja, aa, b, A = headline
    rng = np.random.default_rng(42)
    xv = rng.random(n) + 1j * rng.random(n)  # random_zvector's distribution (bench.py:137-139)
    y = Z.spmv(A, Z.ZVector(xv)).data
    assert bits(y) == bits(O.spmv(n, n, ia, ja, aa, xv)), name


def test_headline_capped_solve_bitwise(headline):
    name, n, ia, ja, aa, b, A = headline
    tol = problems.CONFIGS[name]["tol"]
    M = Z.build_jacobi(A)
    x, rep = Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=tol, max_iterations=3))
    xo, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, M.data, None, tol, 3)
    assert rep.iterations == it == 3, name
    assert not rep.converged and st == O.STATUS_NOT_CONVERGED, name
    assert np.array(rep.residual_history).tobytes() == np.array(hist).tobytes(), name
    assert bits(x.data) == bits(xo), name
