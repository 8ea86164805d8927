"""The numpy port used as the CPU baseline reproduces the reference: bitwise
against the golden vectors when this host's numpy has the fingerprint the
goldens were generated with (otherwise the values still agree to 1e-10)."""
import numpy as np
import pytest

from oracle import fingerprint, port


@pytest.fixture(scope="module")
def same_fingerprint():
    return fingerprint.complex_multiply_formula() == "fma"


def test_port_bicgstab_matches_golden(bicgstab_golden, same_fingerprint):
    for case in ("fd13", "damped21", "s27_14", "dom50_310", "dom80_maxit3", "dom40_identity"):
        g = bicgstab_golden[case]
        tol, maxit = float(g["params"][0]), int(g["params"][1])
        minv = g["minv"] if g["minv"].size else None
        x, hist, conv, _, _ = port.bicgstab(g["ia"], g["ja"], g["aa"], g["b"], minv, tol, maxit)
        if same_fingerprint:
            assert np.array(hist).tobytes() == g["hist"].tobytes(), case
            assert x.tobytes() == g["x"].tobytes(), case
        else:
            assert len(hist) == len(g["hist"]), case
            assert np.allclose(hist, g["hist"], rtol=1e-6), case


def test_port_kernels_match_golden(vecops_golden, spmv_golden, same_fingerprint):
    if not same_fingerprint:
        pytest.skip("host numpy uses a different complex-multiply formula")
    for case, g in vecops_golden.items():
        assert np.array([port.zdot(g["x"], g["y"])]).tobytes() == g["dot_c_4096"].tobytes(), case
        assert np.float64(port.znorm2(g["x"])).tobytes() == g["norm_4096"].tobytes(), case
    for case, g in spmv_golden.items():
        nr = int(g["shape"][0])
        assert port.spmv(g["ia"], g["ja"], g["aa"], g["x"], nr).tobytes() == g["y"].tobytes(), case


def test_host_facts():
    f = fingerprint.host_facts()
    assert f["os_cpu_count"] >= 1 and f["complex_multiply"] in ("fma", "plain", "unknown")
