"""BiCGSTAB(l) and TFQMR on the device kernels vs fixtures made by the live
reference (tests/golden/make_golden.py krylov_ext): solution, iteration
count, every residual-history entry and breakdown reports, bit for bit."""
import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from conftest import golden_cases, load_golden
from helpers import bits

pytestmark = pytest.mark.gpu

CASES = golden_cases(load_golden("krylov_ext"))


@pytest.fixture(scope="module", autouse=True)
def _arith():
    Z.set_arithmetic(True, 262144)


@pytest.mark.parametrize("tag", sorted(CASES))
def test_solver_matches_reference(tag):
    g = CASES[tag]
    n = len(g["ia"]) - 1
    A = Z.CsrMatrix(n, n, g["aa"], g["ja"], g["ia"])
    M = Z.Preconditioner("jacobi", g["minv"]) if len(g["minv"]) else None
    tol, maxit, ell = g["params"]
    guess = Z.ZVector(g["guess"].copy()) if len(g["guess"]) else None
    cfg = Z.SolverConfig(tolerance=float(tol), max_iterations=int(maxit), l=int(ell), initial_guess=guess)
    fn = Z.solve_bicgstab_l if str(g["solver"][0]) == "bicgstabl" else Z.solve_tfqmr
    status = str(g["status"][0])
    if status == "breakdown":
        with pytest.raises(Z.BreakdownError) as e:
            fn(A, Z.ZVector(g["b"].copy()), M, cfg)
        assert str(e.value) == str(g["what"][0])
        assert np.array(e.value.report.residual_history).tobytes() == g["hist"].tobytes()
        return
    x, rep = fn(A, Z.ZVector(g["b"].copy()), M, cfg)
    assert rep.converged == (status == "converged")
    assert rep.iterations == len(g["hist"]) - 1
    assert np.array(rep.residual_history).tobytes() == g["hist"].tobytes()
    assert bits(x.data) == bits(g["x"])
