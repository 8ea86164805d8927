"""Test fixtures shared by the parity suites (same shapes and seeds as the
reference's pkg/tests/helpers.py, rebuilt on this package's API)."""
import numpy as np

import paper_2112_06465_b200 as Z

# The worked 5x5 CSR example of the paper.
GOLDEN_5X5_DENSE = np.array([
    [3, 14, 0, 0, 0],
    [0, 8, 1, 0, 0],
    [2, 0, 6, 0, 0],
    [0, 4, 0, 2, -1],
    [0, 0, 9, 0, 7],
], dtype=np.complex128)


def dense_to_csr(dense) -> "Z.CsrMatrix":
    dense = np.asarray(dense, dtype=np.complex128)
    rows, cols = np.nonzero(dense)
    ia = np.zeros(dense.shape[0] + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=dense.shape[0]), out=ia[1:])
    return Z.CsrMatrix(dense.shape[0], dense.shape[1], dense[rows, cols], cols, ia)


def random_sparse_dense(n_rows, n_cols, density, rng):
    dense = np.zeros((n_rows, n_cols), dtype=np.complex128)
    mask = rng.random((n_rows, n_cols)) < density
    k = int(mask.sum())
    dense[mask] = rng.standard_normal(k) + 1j * rng.standard_normal(k)
    return dense


def random_dominant_system(n, density, seed):
    """Strictly diagonally dominant complex system: (A, dense, b)."""
    rng = np.random.default_rng(seed)
    dense = random_sparse_dense(n, n, density, rng)
    np.fill_diagonal(dense, 0)
    off = np.sum(np.abs(dense), axis=1)
    np.fill_diagonal(dense, (off + 2.0) * np.exp(1j * rng.uniform(-0.4, 0.4, n)))
    b = Z.ZVector(rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return dense_to_csr(dense), dense, b


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128)).tobytes()
