"""Bench CLI on the device (benchtool.py): records with GPU columns, the
reference's exit codes for solves (0 converged, 2 not converged, 4
breakdown), Matrix Market and problem-config inputs."""
import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from paper_2112_06465_b200 import benchtool as B

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("op", B.KERNEL_OPS)
def test_bench_kernel_records(op):
    r = B.bench_kernel(op, 1_000_000, repetitions=5)
    assert r.repetitions == 5 and r.mean_time_ms > 0 and r.gflops > 0
    assert r.gbs > 50 and 0 < r.roofline_frac < 1.5 and r.n_gpus == 1
    assert r.ref_cpu_ms == B.REFERENCE_CPU_KERNELS[op][1_000_000][0]


def test_bench_spmv_and_cli(tmp_path, capsys):
    n, ia, ja, aa, b = Z.problems.helmholtz_fd(3, 17, frequency=1.0)
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    p = tmp_path / "a.mtx"
    Z.write_matrix_market(A, p)
    r = B.bench_spmv(p, repetitions=5)
    assert r.size == A.nnz and r.gbs > 0
    assert B.main(["spmv", "--matrix", str(p), "--reps", "3", "--format", "csv-gpu"]) == 0
    rec = Z.read_report_csv(capsys.readouterr().out)[0]
    assert rec.op_name == "spmv" and rec.gbs > 0


def test_cli_solve_exit_codes(tmp_path):
    cfg = tmp_path / "p.cfg"
    cfg.write_text("dim=3\ncells=9\nfrequency=1.5\n")
    for method in ("bicgstab", "bicgstab_l", "tfqmr"):
        assert B.main(["solve", "--method", method, "--problem", str(cfg), "--format", "csv"]) == 0
    assert B.main(["solve", "--method", "bicgstab", "--problem", str(cfg), "--maxit", "2", "--tol", "1e-14"]) == 2
    # the zero matrix: the shadow pivot <r~, A r> is 0 at once -> breakdown
    zero = tmp_path / "zero.mtx"
    zero.write_text("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 0\n")
    for method in ("bicgstab", "bicgstab_l", "tfqmr"):
        assert B.main(["solve", "--method", method, "--matrix", str(zero), "--precond", "none"]) == 4


def test_cli_singular_preconditioner_exit_4(tmp_path):
    p = tmp_path / "s.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 1 1\n")
    assert B.main(["solve", "--method", "tfqmr", "--matrix", str(p)]) == 4
