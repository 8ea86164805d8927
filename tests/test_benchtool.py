"""Bench CLI and records (benchtool.py, drop-in for zlinalg bench.py): the
reference's CSV layout and parser, the GPU columns, usage/parse exit codes
(host only here; device timings in test_benchtool_gpu)."""
import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from paper_2112_06465_b200 import benchtool as B


def _recs():
    return [Z.BenchRecord("zdot", 1000, 100, 0.0123, gflops=0.65, gbs=2.6, roofline_frac=0.0004, n_gpus=1),
            Z.BenchRecord("bicgstab", 32768, 1, 15.5, iterations=69, residual=8.5e-9, converged=True),
            Z.BenchRecord("tfqmr", 10, 1, 1.0, iterations=3, residual=0.5, converged=False)]


def test_csv_is_the_reference_layout_and_round_trips():
    text = Z.emit_report(_recs(), "csv")
    assert text.splitlines()[0] == "op,size,reps,time_ms,gflops,iterations,residual,converged"
    assert text.splitlines()[2] == "bicgstab,32768,1,15.5,,69,8.5e-09,true"
    back = Z.read_report_csv(text)
    assert [r.op_name for r in back] == ["zdot", "bicgstab", "tfqmr"] and back[2].converged is False


def test_csv_gpu_columns_round_trip():
    back = Z.read_report_csv(Z.emit_report(_recs(), "csv-gpu"))
    assert back[0].gbs == 2.6 and back[0].roofline_frac == 0.0004 and back[0].n_gpus == 1
    assert back[1].gbs is None


def test_markdown_table():
    md = Z.emit_report(_recs(), "md")
    assert md.startswith("| op | h | time (ms) | Gflops | GB/s | of HBM | iters |")


def test_bad_inputs():
    with pytest.raises(Z.ParseError):
        Z.read_report_csv("a,b\n1,2\n")
    with pytest.raises(Z.ParseError, match="line 2"):
        Z.read_report_csv("op,size,reps,time_ms,gflops,iterations,residual,converged\nx,1\n")
    with pytest.raises(Z.ParameterError):
        Z.emit_report(_recs(), "xml")
    with pytest.raises(Z.ParameterError):
        B.bench_kernel("zfoo", 10)
    with pytest.raises(Z.ParameterError):
        B.bench_solver("bicgstab")


def test_cli_usage_errors_exit_3(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        B.main(["kernel", "--op", "zdot"])
    assert e.value.code == 3
    with pytest.raises(SystemExit) as e:
        B.main(["kernel", "--op", "zdot", "--size", "10", "--threads", "0"])
    assert e.value.code == 3
    assert B.main(["spmv", "--matrix", str(tmp_path / "missing.mtx")]) == 3
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix array real general\n")
    assert B.main(["spmv", "--matrix", str(bad)]) == 3
    assert "unsupported format" in capsys.readouterr().err


def test_reference_cpu_table_matches_paper_numbers():
    assert B.REFERENCE_CPU_KERNELS["zdot"][15_000_000] == (130.00, 0.92)
    assert set(B.REFERENCE_CPU_KERNELS) == set(B.KERNEL_OPS)
