"""Pin the C oracle against golden vectors produced by the live reference.

CPU-only.  Every comparison is bitwise (``tobytes`` equality, so signed
zeros count): the oracle is trusted as the GPU checker only because it
reproduces the reference's own outputs bit for bit.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2112_06465_b200 import problems


def same_bits(a, b):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.complex128))
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def same_float(a, b):
    return np.float64(a).tobytes() == np.float64(b).tobytes()


@pytest.fixture(scope="module", autouse=True)
def _arith():
    O.set_arith(True, 262144)


def test_oracle_vecops_bitwise(vecops_golden):
    checked = 0
    for case, g in vecops_golden.items():
        x, y = g["x"], g["y"]
        for conj, tag in ((True, "c"), (False, "u")):
            for bs in (64, 4096, 65536):
                got = O.zdot(x, y, conj, bs)
                assert same_bits([got], g[f"dot_{tag}_{bs}"]), (case, tag, bs)
                checked += 1
            if f"dot_{tag}_seq" in g:
                assert same_bits([O.zdot(x, y, conj, sequential=True)], g[f"dot_{tag}_seq"]), (case, tag)
        for bs in (64, 4096, 65536):
            assert same_float(O.znorm2(x, bs), g[f"norm_{bs}"][0]), (case, bs)
        if "norm_seq" in g:
            assert same_float(O.znorm2(x, sequential=True), g["norm_seq"][0]), case
        if "axpy" in g:
            a = complex(g["alpha"][0])
            assert same_bits(O.zaxpy(a, x, y), g["axpy"]), case
            assert same_bits(O.zscal(a, x), g["scal"]), case
            assert same_bits(O.zaxmy(x, y), g["axmy"]), case
            assert same_bits(O.jacobi_apply(x, g["minv"]), g["jacobi"]), case
    assert checked > 100


def test_oracle_spmv_bitwise(spmv_golden):
    for case, g in spmv_golden.items():
        nr, nc = (int(v) for v in g["shape"])
        y = O.spmv(nr, nc, g["ia"], g["ja"], g["aa"], g["x"])
        assert same_bits(y, g["y"]), case


def test_elision_threshold_matters(spmv_golden):
    """Above nnz*16 >= 256 KiB numpy computes F1(x[ja], aa); pin that the
    swap is real by showing the unswapped product misses the golden."""
    g = spmv_golden["fd_above"]
    n = int(g["shape"][0])
    O.set_arith(True, 1 << 62)  # never swap
    try:
        y = O.spmv(n, n, g["ia"], g["ja"], g["aa"], g["x"])
    finally:
        O.set_arith(True, 262144)
    assert not same_bits(y, g["y"])


def test_oracle_bicgstab_bitwise(bicgstab_golden):
    for case, g in bicgstab_golden.items():
        n = g["b"].shape[0]
        tol, maxit = float(g["params"][0]), int(g["params"][1])
        minv = g["minv"] if g["minv"].size else None
        guess = g["guess"] if g["guess"].size else None
        x, hist, it, st, what = O.bicgstab(n, g["ia"], g["ja"], g["aa"], g["b"], minv, guess, tol, maxit)
        want_hist = g["hist"]
        assert np.asarray(hist).tobytes() == want_hist.tobytes(), case
        status = str(g["status"][0])
        if status == "breakdown":
            assert st == O.STATUS_BREAKDOWN
            assert str(g["what"][0]).startswith(O.BREAKDOWN_NAMES[what] + " numerically zero"), case
        else:
            assert st == (O.STATUS_CONVERGED if status == "converged" else O.STATUS_NOT_CONVERGED), case
            assert same_bits(x, g["x"]), case


def test_fd_generator_matches_reference_assemble(problems_golden):
    for case, g in problems_golden.items():
        dim, cells, freq = g["params"]
        n, ia, ja, aa, b = problems.helmholtz_fd(int(dim), int(cells), frequency=float(freq))
        assert np.array_equal(ia, g["ia"]) and np.array_equal(ja, g["ja"]), case
        assert same_bits(aa, g["aa"]) and same_bits(b, g["b"]), case


def test_27pt_generator_structure():
    n, ia, ja, aa, b = problems.helmholtz_27pt(6)
    counts = np.diff(ia)
    assert n == 216 and counts.max() == 27 and counts.min() == 8
    # nnz of a 27-point stencil on m^3: (3m-2)^3
    assert ia[-1] == (3 * 6 - 2) ** 3
    rows = np.repeat(np.arange(n), counts)
    within = np.diff(ja)[np.diff(rows) == 0]
    assert np.all(within > 0)
    assert np.all(aa[ja == rows] == aa[0])


def test_oracle_krylov_ext_bitwise():
    """BiCGSTAB(l) / TFQMR restatements vs fixtures from the live reference
    (krylov.py:298-489): history, status, breakdown text and solution."""
    from conftest import golden_cases, load_golden
    for case, g in golden_cases(load_golden("krylov_ext")).items():
        n = g["b"].shape[0]
        tol, maxit, ell = g["params"]
        minv = g["minv"] if g["minv"].size else None
        guess = g["guess"] if g["guess"].size else None
        if str(g["solver"][0]) == "bicgstabl":
            x, hist, it, st, what, wj = O.bicgstab_l(n, g["ia"], g["ja"], g["aa"], g["b"], minv, guess, float(tol),
                                                     int(maxit), int(ell))
        else:
            x, hist, it, st, what = O.tfqmr(n, g["ia"], g["ja"], g["aa"], g["b"], minv, guess, float(tol), int(maxit))
            wj = 0
        assert np.asarray(hist).tobytes() == g["hist"].tobytes(), case
        status = str(g["status"][0])
        if status == "breakdown":
            assert st == O.STATUS_BREAKDOWN, case
            assert O.breakdown_message(what, wj, it) == str(g["what"][0]), case
        else:
            assert st == (O.STATUS_CONVERGED if status == "converged" else O.STATUS_NOT_CONVERGED), case
            assert same_bits(x, g["x"]), case
