"""Host ingestion (matio.py) against fixtures from the live reference
(tests/golden/make_io_golden.py): Matrix Market -> CSR arrays bitwise
(duplicate summation order, symmetric mirroring, value spellings), the
reference's ParseError text for malformed files, writer round trips, binary
CSR round trips and stats()."""
import json
import os

import numpy as np
import pytest

import paper_2112_06465_b200 as Z
from paper_2112_06465_b200 import matio

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
META = json.load(open(os.path.join(IO, "io.json")))
ARR = np.load(os.path.join(IO, "io.npz"))


@pytest.mark.parametrize("name", sorted(META["good"]))
def test_matrix_market_to_csr_matches_reference(name):
    g = META["good"][name]
    A = Z.coo_to_csr(Z.read_matrix_market(os.path.join(IO, g["file"])))
    assert [A.n_rows, A.n_cols] == g["shape"]
    assert np.array_equal(A.ia, ARR[f"{name}__ia"]) and np.array_equal(A.ja, ARR[f"{name}__ja"])
    assert A.aa.tobytes() == ARR[f"{name}__aa"].tobytes()
    st = Z.stats(A)
    assert [st.h, st.nz, st.density, st.bandwidth, st.max_row, st.nz_per_h, st.nz_per_h_stddev] == g["stats"]


@pytest.mark.parametrize("name", sorted(META["bad"]))
def test_matrix_market_errors_match_reference(name):
    g = META["bad"][name]
    path = os.path.join(IO, g["file"])
    if g["error"] is None:
        Z.read_matrix_market(path)
        return
    with pytest.raises(Z.ParseError) as e:
        Z.read_matrix_market(path)
    assert str(e.value) == g["error"]


def test_coo_entries_are_the_reference_tuples():
    m = Z.read_matrix_market(os.path.join(IO, "sym_real.mtx"))
    assert m.nnz == len(m.entries) == 12  # 8 stored, 4 mirrored
    assert m.entries[1] == (1, 0, m.entries[1][2]) and m.entries[2] == (0, 1, m.entries[1][2])
    m.add(4, 4, 1.0)  # still a CooMatrix
    assert Z.coo_to_csr(m).nnz == 12  # (4, 4) was already stored: summed


def test_writer_round_trip_and_reference_text(tmp_path):
    A = Z.coo_to_csr(Z.read_matrix_market(os.path.join(IO, "dup_complex.mtx")))
    p = tmp_path / "w.mtx"
    Z.write_matrix_market(A, p)
    assert p.read_text() == open(os.path.join(IO, "written_ref.mtx")).read()
    B = Z.coo_to_csr(Z.read_matrix_market(p))
    assert np.array_equal(A.ia, B.ia) and np.array_equal(A.ja, B.ja) and A.aa.tobytes() == B.aa.tobytes()


def test_binary_round_trip(tmp_path):
    A = Z.coo_to_csr(Z.read_matrix_market(os.path.join(IO, "big.mtx")))
    p = tmp_path / "a.bin"
    Z.write_csr_binary(A, p)
    B = Z.read_csr_binary(p)
    assert np.array_equal(A.ia, B.ia) and np.array_equal(A.ja, B.ja) and A.aa.tobytes() == B.aa.tobytes()
    with open(p, "r+b") as fh:
        fh.truncate(os.path.getsize(p) - 16)
    with pytest.raises(Z.ParseError, match="truncated arrays"):
        Z.read_csr_binary(p)
    with pytest.raises(Z.DimensionError):
        Z.write_csr_binary(Z.CsrMatrix(2, 3, [], [], [0, 0, 0]), tmp_path / "r.bin")


def test_sparse_module_exports_io():
    from paper_2112_06465_b200 import sparse
    assert sparse.read_matrix_market is matio.read_matrix_market
    assert sparse.stats is matio.stats


HELM = json.load(open(os.path.join(IO, "helmholtz.json")))
HARR = np.load(os.path.join(IO, "helmholtz.npz"))


@pytest.mark.parametrize("name", sorted(HELM["assemble"]))
def test_assemble_constant_fields_bitwise(name):
    from paper_2112_06465_b200 import helmholtz as H
    kw = {k: complex(*v) if isinstance(v, list) else v for k, v in HELM["assemble"][name].items()}
    A, b = H.assemble(H.HelmholtzProblem(**kw))
    assert np.array_equal(A.ia, HARR[f"{name}__ia"]) and np.array_equal(A.ja, HARR[f"{name}__ja"])
    assert A.aa.tobytes() == HARR[f"{name}__aa"].tobytes()
    assert b.data.tobytes() == HARR[f"{name}__b"].tobytes()


@pytest.mark.parametrize("name", sorted(HELM["configs"]))
def test_load_problem_config(name):
    from paper_2112_06465_b200 import helmholtz as H
    g = HELM["configs"][name]
    path = os.path.join(IO, f"cfg_{name}.cfg")
    if "error" in g:
        with pytest.raises(Z.ParseError) as e:
            H.load_problem_config(path)
        assert str(e.value) == g["error"]
    else:
        p = H.load_problem_config(path)
        assert [p.dim, p.cells_per_axis, p.domain_length, p.frequency, p.velocity] == g["ok"]
        assert p.source == 1 + 0j
