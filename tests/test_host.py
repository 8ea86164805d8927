"""CPU-only checks: the C ABI library loads and exports every symbol the
header declares, host-side validation mirrors the reference, and the product
refuses to run without a device (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from paper_2112_06465_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "zk.h")).read()
    return sorted(set(re.findall(r"^\s*(?:zk_status|const char\*)\s+(zk_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load_library()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES) | set(_lib.STRING_FUNCS)
    assert lib.zk_version().decode().endswith("sm_100a")


def test_profile_phase_table_matches_header():
    """zk_profile_read fills ZK_NPHASES entries in the order include/zk.h lists;
    the Python table must have the same length (a mismatch reads past the
    arrays or drops the narrow-matrix two-vector phase)."""
    text = open(os.path.join(ROOT, "include", "zk.h")).read()
    n = int(re.search(r"#define ZK_NPHASES (\d+)", text).group(1))
    assert len(_lib.PHASES) == n
    assert _lib.PHASES[-1] == "spmv2"


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(Z.DeviceUnavailableError):
        Z.znorm2(Z.ZVector([1 + 1j]))


def test_reduction_plan_validation():
    Z.ReductionPlan(block_size=64)
    Z.ReductionPlan(block_size=65536, mode=Z.SEQUENTIAL)
    for bad in (32, 100, 131072, 0, -4096):
        with pytest.raises(Z.ParameterError):
            Z.ReductionPlan(block_size=bad)
    with pytest.raises(Z.ParameterError):
        Z.ReductionPlan(mode="warp")


def test_solver_config_and_preconditioner_validation():
    for kw in (dict(tolerance=0.0), dict(max_iterations=0), dict(l=0)):
        with pytest.raises(Z.ParameterError):
            Z.SolverConfig(**kw)
    cfg = Z.SolverConfig()
    assert (cfg.tolerance, cfg.max_iterations, cfg.l) == (1e-9, 1000, 8)
    with pytest.raises(Z.ParameterError):
        Z.Preconditioner("ilu")
    with pytest.raises(Z.ParameterError):
        Z.Preconditioner("jacobi")
    with pytest.raises(Z.DimensionError):
        Z.Preconditioner("jacobi", np.ones(3, dtype=np.complex128)).apply(Z.ZVector.zeros(4))


def test_csr_validation():  # sparse.py:79-103 / test_sparse.py:96-108
    with pytest.raises(Z.FormatError):
        Z.CsrMatrix(2, 2, [1.0], [0, 1], [0, 1, 2])
    with pytest.raises(Z.FormatError):
        Z.CsrMatrix(2, 2, [1.0, 2.0], [0, 0], [0, 2, 2])
    with pytest.raises(Z.FormatError):
        Z.CsrMatrix(2, 2, [1.0, 2.0], [1, 0], [0, 2, 2])
    with pytest.raises(Z.FormatError):
        Z.CsrMatrix(2, 2, [1.0], [0], [0, 2, 1])
    with pytest.raises(Z.FormatError):
        Z.CsrMatrix(2, 2, [1.0], [5], [0, 1, 1])
    with pytest.raises(Z.DimensionError):
        Z.CsrMatrix(2, 3, [1.0], [0], [0, 1, 1]).n
    # empty rows between nonempty ones are fine
    Z.CsrMatrix(4, 4, [1.0, 2.0, 3.0], [0, 3, 1], [0, 2, 2, 2, 3])


def test_diagonal_vectorised_matches_loop():
    rng = np.random.default_rng(3)
    d = (rng.random((30, 30)) < 0.2) * (rng.standard_normal((30, 30)) + 1j)
    from helpers import dense_to_csr
    A = dense_to_csr(d)
    assert np.array_equal(A.diagonal(), np.diag(d))


def test_cplx_arithmetic():
    a, b = Z.Cplx(1.5, -2.0), Z.Cplx(0.25, 3.0)
    assert a * b == Z.Cplx(1.5 * 0.25 - (-2.0) * 3.0, 1.5 * 3.0 + (-2.0) * 0.25)
    q = a / b
    assert complex(q) == pytest.approx(complex(a) / complex(b), rel=1e-15)
    assert -a == Z.Cplx(-1.5, 2.0) and abs(Z.Cplx(3, 4)) == 5.0
    assert Z.Cplx.from_bytes(a.to_bytes()) == a
    with pytest.raises(ZeroDivisionError):
        a / Z.Cplx(0, 0)
    assert Z.FLOPS.flops("zdot", 10) == 80 and Z.FLOPS.flops("spmv", 3) == 24


def test_zvector_host_semantics():
    v = Z.ZVector.from_values([1 + 2j, Z.Cplx(3, -4)])
    assert len(v) == 2 and v[1] == Z.Cplx(3, -4)
    v[0] = Z.Cplx(0, 1)
    assert [complex(c) for c in v] == [1j, 3 - 4j]
    with pytest.raises(Z.DimensionError):
        Z.ZVector(np.zeros((2, 2), dtype=np.complex128))
    with pytest.raises(Z.DimensionError):
        Z.zdot(Z.ZVector.zeros(3), Z.ZVector.zeros(4))
    assert Z.zdot(Z.ZVector.zeros(0), Z.ZVector.zeros(0)) == Z.Cplx(0, 0)


def test_vector_binary_roundtrip(tmp_path):
    v = Z.ZVector(np.array([1 + 2j, -0.0 - 0.0j, 3.5j]))
    Z.write_zvector(v, tmp_path / "v.zvec")
    back = Z.read_zvector(tmp_path / "v.zvec")
    assert back.data.tobytes() == v.data.tobytes()
