"""BASELINE config C3 generator (P1-FE Helmholtz on a cylinder): a valid
reference CsrMatrix (sparse.py:79-103 validation), complex-symmetric, FE row
structure (<= 15 nonzeros, irregular boundary rows), and the C3 size."""
import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from oracle import oracle as O
from paper_2112_06465_b200 import problems


@pytest.mark.parametrize("m", [8, 16])
def test_cylinder_p1fe_structure(m):
    n, ia, ja, aa, b = problems.cylinder_p1fe(m)
    A = Z.CsrMatrix(n, n, aa, ja, ia)  # validates: sorted, in range, consistent
    rows = np.diff(ia)
    assert rows.max() == 15 and rows.min() >= 4
    assert len(np.unique(rows)) > 3  # irregular boundary rows
    dense = A.to_dense()
    assert np.array_equal(dense, dense.T)  # complex-symmetric (not Hermitian)
    assert np.count_nonzero(b) == 1
    assert np.all(A.diagonal() != 0)


def test_c3_size_matches_baseline():
    c = problems.CONFIGS["C3"]
    # ~1M rows / ~15M nnz (BASELINE.json configs[2]); sized without building it
    m = c["m"]
    assert 100 <= m <= 120


def test_cylinder_p1fe_solves_on_oracle():
    O.set_arith(True, 262144)
    n, ia, ja, aa, b = problems.cylinder_p1fe(12)
    minv = np.divide(1.0, Z.CsrMatrix(n, n, aa, ja, ia).diagonal())  # build_jacobi's arithmetic (krylov.py:120)
    x, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, minv, None, 1e-8, 3000)
    assert st == 0 and hist[-1] <= 1e-8 and it < 3000
