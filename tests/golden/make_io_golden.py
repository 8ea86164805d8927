"""Fixtures for the host ingestion path (matio.py) from the LIVE reference:
Matrix Market files (real/complex, general/symmetric, duplicates, comments,
blank lines) with the CSR arrays zlinalg produces from them
(coo_to_csr(read_matrix_market(p))), malformed files with the reference's
ParseError text, binary CSR round trips and stats().  Run in the dev
container (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import zlinalg as R  # noqa: E402

OUT = os.path.join(HERE, "io")


def w(name, text):
    p = os.path.join(OUT, name)
    with open(p, "w") as fh:
        fh.write(text)
    return p


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(5)
    good = {}
    # general complex with duplicates (summation order matters), comments and blank lines
    lines = ["%%MatrixMarket matrix coordinate complex general", "% a comment", "", "7 6 40"]
    for _ in range(40):
        i, j = rng.integers(1, 8), rng.integers(1, 7)
        lines.append(f"{i} {j} {rng.standard_normal():.17g} {rng.standard_normal() * 1e-7:.17g}")
    lines.insert(10, "% interleaved comment")
    good["dup_complex"] = w("dup_complex.mtx", "\n".join(lines) + "\n")
    # real symmetric
    lines = ["%%MatrixMarket matrix coordinate real symmetric", "5 5 8"]
    for i, j in [(1, 1), (2, 1), (3, 2), (3, 3), (5, 1), (4, 4), (5, 5), (5, 2)]:
        lines.append(f"{i} {j} {rng.standard_normal():.17g}")
    good["sym_real"] = w("sym_real.mtx", "\n".join(lines) + "\n")
    # values in exotic spellings float() accepts
    good["spellings"] = w("spellings.mtx", "%%MatrixMarket matrix coordinate complex general\n3 3 4\n"
                          "1 1 1e-300 -0.0\n2 2 +3.25 1E+2\n3 3 .5 -7.\n1 3 0.1 0.30000000000000004\n")
    good["empty"] = w("empty.mtx", "%%MatrixMarket matrix coordinate real general\n4 3 0\n")
    # a larger one for the vectorised path
    n, nz = 300, 3000
    lines = ["%%MatrixMarket matrix coordinate complex general", f"{n} {n} {nz}"]
    for _ in range(nz):
        lines.append(f"{rng.integers(1, n + 1)} {rng.integers(1, n + 1)} {rng.standard_normal():.17g} "
                     f"{rng.standard_normal():.17g}")
    good["big"] = w("big.mtx", "\n".join(lines) + "\n")
    bad = {
        "empty_file": "",
        "bad_banner": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
        "array_fmt": "%%MatrixMarket matrix array real general\n1 1\n1\n",
        "pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
        "hermitian": "%%MatrixMarket matrix coordinate complex hermitian\n1 1 1\n1 1 1 0\n",
        "no_header": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
        "short_header": "%%MatrixMarket matrix coordinate real general\n2 2\n",
        "float_header": "%%MatrixMarket matrix coordinate real general\n2 2 1.5\n1 1 1\n",
        "neg_header": "%%MatrixMarket matrix coordinate real general\n2 -2 1\n1 1 1\n",
        "few_fields": "%%MatrixMarket matrix coordinate complex general\n2 2 2\n1 1 1 0\n2 2 3\n",
        "bad_value": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 x3\n",
        "float_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.0 1 1\n",
        "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n",
        "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
        "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n",
        "trailing_comment": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1 % x\n",
    }
    out = {"good": {}, "bad": {}}
    arrays = {}
    for name, p in good.items():
        A = R.coo_to_csr(R.read_matrix_market(p))
        arrays[f"{name}__ia"], arrays[f"{name}__ja"], arrays[f"{name}__aa"] = A.ia, A.ja, A.aa
        st = R.stats(A)
        out["good"][name] = {"file": os.path.basename(p), "shape": [A.n_rows, A.n_cols],
                             "stats": [st.h, st.nz, st.density, st.bandwidth, st.max_row, st.nz_per_h,
                                       st.nz_per_h_stddev]}
    for name, text in bad.items():
        p = w(f"bad_{name}.mtx", text)
        try:
            R.read_matrix_market(p)
            msg = None
        except R.ParseError as e:
            msg = str(e)
        out["bad"][name] = {"file": os.path.basename(p), "error": msg}
    # written by the reference writer: the text a read-back must reproduce
    A = R.coo_to_csr(R.read_matrix_market(good["dup_complex"]))
    R.write_matrix_market(A, os.path.join(OUT, "written_ref.mtx"))
    np.savez_compressed(os.path.join(OUT, "io.npz"), **arrays)
    with open(os.path.join(OUT, "io.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out["bad"], indent=1))


if __name__ == "__main__":
    main()


def helmholtz_cases():
    """assemble() with nonzero constant Dirichlet data and source, and
    load_problem_config files (valid and malformed)."""
    out, meta = {}, {}
    cases = {"d2": dict(dim=2, cells_per_axis=9, domain_length=2.0, frequency=0.7, velocity=1.5,
                        dirichlet_value=0.5 - 0.25j, source=2 + 1j),
             "d3": dict(dim=3, cells_per_axis=6, frequency=1.1, dirichlet_value=-1.0 + 0j, source=0.5j),
             "d1": dict(dim=1, cells_per_axis=17, domain_length=0.5, dirichlet_value=1e-3 + 7j, source=1 + 0j)}
    for name, kw in cases.items():
        A, b = R.assemble(R.HelmholtzProblem(**kw))
        out[f"{name}__ia"], out[f"{name}__ja"], out[f"{name}__aa"], out[f"{name}__b"] = A.ia, A.ja, A.aa, b.data
        meta[name] = {k: [v.real, v.imag] if isinstance(v, complex) else v for k, v in kw.items()}
    cfgs = {"ok": "# C1-like\ndim = 3\ncells=9  # comment\nfrequency = 1.5\nlength=1.0\n",
            "nokey": "dim=3\n", "badkey": "dim=2\ncells=5\ncolor=3\n", "noeq": "dim 3\n",
            "badval": "dim=3\ncells=five\n", "badparam": "dim=4\ncells=5\n"}
    cfg_meta = {}
    for name, text in cfgs.items():
        p = w(f"cfg_{name}.cfg", text)
        try:
            pr = R.load_problem_config(p)
            cfg_meta[name] = {"ok": [pr.dim, pr.cells_per_axis, pr.domain_length, pr.frequency, pr.velocity]}
        except R.ParseError as e:
            cfg_meta[name] = {"error": str(e)}
    np.savez_compressed(os.path.join(OUT, "helmholtz.npz"), **out)
    with open(os.path.join(OUT, "helmholtz.json"), "w") as fh:
        json.dump({"assemble": meta, "configs": cfg_meta}, fh, indent=1)


if __name__ == "__main__" and "helmholtz" in sys.argv[1:]:
    helmholtz_cases()
