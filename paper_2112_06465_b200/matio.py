"""Matrix ingestion: Matrix Market and binary CSR files, matrix statistics
(drop-in for the host-side I/O of zlinalg sparse.py:160-402).

These feed the device path; they run on the host.  The reference parses a
Matrix Market body line by line into a list of tuples and renders files row
by row; here the body is parsed and checked with vectorised numpy
(``np.loadtxt``, whose float parser is correctly rounded like ``float()``),
and only a file that fails the fast checks is re-read line by line -- so
every ``ParseError`` carries the reference's message and line number.  The
parsed entries stay in arrays (:class:`ArrayCooMatrix`) all the way into
:func:`coo_to_csr`, whose duplicate summation order (stable sort, reduceat)
is the reference's.  Binary CSR files are read with ``np.fromfile``.
"""
from __future__ import annotations

import struct
import warnings
from dataclasses import dataclass

import numpy as np

from .errors import ParseError
from .sparse import CooMatrix, CsrMatrix

__all__ = ["ArrayCooMatrix", "MatrixStats", "stats", "read_matrix_market", "write_matrix_market",
           "read_csr_binary", "write_csr_binary"]

_MM_BANNER = "%%matrixmarket"
_BIN_HEADER = struct.Struct("<QQ")


class ArrayCooMatrix(CooMatrix):
    """A CooMatrix whose (row, col, value) triples live in numpy arrays; the
    ``entries`` list of tuples is built only if someone asks for it."""

    def __init__(self, n_rows, n_cols, rows, cols, vals):
        super().__init__(n_rows, n_cols)
        self._arrays = (np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64),
                        np.asarray(vals, dtype=np.complex128))
        self._materialized = False

    def __getattribute__(self, name):
        if name == "entries" and not object.__getattribute__(self, "_materialized"):
            r, c, v = object.__getattribute__(self, "_arrays")
            object.__setattr__(self, "entries", list(zip(r.tolist(), c.tolist(), v.tolist())))
            object.__setattr__(self, "_materialized", True)
        return object.__getattribute__(self, name)

    @property
    def nnz(self) -> int:
        return int(self._arrays[0].shape[0]) if not self._materialized else len(self.entries)

    def arrays(self):
        if self._materialized:  # entries may have been appended to
            e = self.entries
            return (np.fromiter((t[0] for t in e), np.int64, len(e)), np.fromiter((t[1] for t in e), np.int64, len(e)),
                    np.fromiter((complex(t[2]) for t in e), np.complex128, len(e)))
        return self._arrays


@dataclass(frozen=True)
class MatrixStats:
    """Sketch of a sparse matrix (sparse.py:160-170)."""

    h: int
    nz: int
    density: float  # percent: 100 * nz / (rows * cols)
    bandwidth: int  # max |i - j| over stored entries
    max_row: int
    nz_per_h: float
    nz_per_h_stddev: float  # population standard deviation of row counts


def stats(A: CsrMatrix) -> MatrixStats:
    """Row-density statistics (sparse.py:235-266): density over the full
    h x h grid, population standard deviation of the row counts."""
    counts = np.diff(A.ia)
    nz, h = A.nnz, A.n_rows
    if nz:
        rows = np.repeat(np.arange(A.n_rows), counts)
        bandwidth = int(np.abs(rows - A.ja).max())
        max_row = int(counts.max())
    else:
        bandwidth = 0
        max_row = int(counts.max()) if h else 0
    cells = A.n_rows * A.n_cols
    return MatrixStats(h=h, nz=nz, density=100.0 * nz / cells if cells else 0.0, bandwidth=bandwidth,
                       max_row=max_row, nz_per_h=nz / h if h else 0.0,
                       nz_per_h_stddev=float(np.std(counts)) if h else 0.0)


# ---- Matrix Market coordinate files -----------------------------------------------

def _header(lines):
    """Banner and size line (sparse.py:299-331); returns (field, symmetry,
    n_rows, n_cols, nnz, index of the first body line)."""
    if not lines:
        raise ParseError("empty file", line=1)
    banner = lines[0].strip().lower().split()
    if len(banner) != 5 or banner[0] != _MM_BANNER or banner[1] != "matrix":
        raise ParseError(f"bad banner {lines[0]!r}", line=1)
    fmt, field_kind, symmetry = banner[2], banner[3], banner[4]
    if fmt != "coordinate":
        raise ParseError(f"unsupported format {fmt!r} (only coordinate)", line=1)
    if field_kind not in ("real", "complex"):
        raise ParseError(f"unsupported field {field_kind!r} (only real/complex)", line=1)
    if symmetry not in ("general", "symmetric"):
        raise ParseError(f"unsupported symmetry {symmetry!r} (only general/symmetric)", line=1)
    for k in range(1, len(lines)):
        text = lines[k].strip()
        if not text or text.startswith("%"):
            continue
        parts = text.split()
        if len(parts) != 3:
            raise ParseError(f"size header needs 'rows cols nnz', got {text!r}", line=k + 1)
        try:
            n_rows, n_cols, nnz = (int(p) for p in parts)
        except ValueError:
            raise ParseError(f"non-integer size header {text!r}", line=k + 1) from None
        if n_rows < 0 or n_cols < 0 or nnz < 0:
            raise ParseError(f"negative size header {text!r}", line=k + 1)
        return field_kind, symmetry, n_rows, n_cols, nnz, k + 1
    raise ParseError("missing size header", line=len(lines))


def _body_slow(lines, start, field_kind, n_rows, n_cols, nnz):
    """Line-by-line body scan with the reference's conversions, checks and
    messages (sparse.py:333-357): returns (rows, cols, values) one-based."""
    want = 4 if field_kind == "complex" else 3
    rows, cols, vals = [], [], []
    seen = 0
    for k in range(start, len(lines)):
        text = lines[k].strip()
        if not text or text.startswith("%"):
            continue
        parts = text.split()
        if len(parts) != want:
            raise ParseError(f"expected {want} fields, got {len(parts)}", line=k + 1)
        try:
            i, j = int(parts[0]), int(parts[1])
            re = float(parts[2])
            im = float(parts[3]) if want == 4 else 0.0
        except ValueError:
            raise ParseError(f"malformed entry {text!r}", line=k + 1) from None
        if not (1 <= i <= n_rows and 1 <= j <= n_cols):
            raise ParseError(f"index ({i}, {j}) out of range for {n_rows}x{n_cols}", line=k + 1)
        seen += 1
        if seen > nnz:
            raise ParseError(f"more than the declared {nnz} entries", line=k + 1)
        rows.append(i)
        cols.append(j)
        vals.append(complex(re, im))
    if seen != nnz:
        raise ParseError(f"declared {nnz} entries but found {seen}", line=len(lines))
    return (np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), np.array(vals, dtype=np.complex128))


def _body_fast(body, want, n_rows, n_cols, nnz):
    """Vectorised parse of well-formed body lines (None when anything is off:
    the caller then takes the line-by-line path)."""
    if len(body) != nnz:
        return None
    if nnz == 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy(), np.zeros(0, dtype=np.complex128)
    dt = [("i", "i8"), ("j", "i8"), ("re", "f8")] + ([("im", "f8")] if want == 4 else [])
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rec = np.loadtxt(body, dtype=dt, comments=None, ndmin=1)
    except (ValueError, OverflowError):
        return None
    if rec.shape != (nnz,):
        return None
    rows, cols = rec["i"].astype(np.int64), rec["j"].astype(np.int64)
    if np.any((rows < 1) | (rows > n_rows) | (cols < 1) | (cols > n_cols)):
        return None
    vals = np.empty(nnz, dtype=np.complex128)
    vals.real = rec["re"]
    vals.imag = rec["im"] if want == 4 else 0.0
    return rows, cols, vals


def read_matrix_market(path) -> CooMatrix:
    """Matrix Market coordinate file -> CooMatrix (sparse.py:286-357):
    real or complex, general or symmetric (mirrored, entry then mirror),
    one-based indices; ``ParseError`` with the line number otherwise."""
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.read().splitlines()
    field_kind, symmetry, n_rows, n_cols, nnz, start = _header(lines)
    want = 4 if field_kind == "complex" else 3
    body = [t for t in (ln.strip() for ln in lines[start:]) if t and not t.startswith("%")]
    parsed = _body_fast(body, want, n_rows, n_cols, nnz)
    if parsed is None:
        parsed = _body_slow(lines, start, field_kind, n_rows, n_cols, nnz)
    rows, cols, vals = parsed
    rows = rows - 1
    cols = cols - 1
    if symmetry == "symmetric":  # entry, then its mirror when off-diagonal (sparse.py:354-356)
        off = rows != cols
        reps = 1 + off.astype(np.int64)
        pos = np.cumsum(reps) - reps
        total = int(reps.sum())
        r2 = np.empty(total, np.int64)
        c2 = np.empty(total, np.int64)
        v2 = np.empty(total, np.complex128)
        r2[pos], c2[pos], v2[pos] = rows, cols, vals
        mp = pos[off] + 1
        r2[mp], c2[mp], v2[mp] = cols[off], rows[off], vals[off]
        rows, cols, vals = r2, c2, v2
    return ArrayCooMatrix(n_rows, n_cols, rows, cols, vals)


def write_matrix_market(A: CsrMatrix, path) -> None:
    """CSR -> Matrix Market coordinate complex general, 17 significant
    digits so a read-back reproduces every value (sparse.py:360-372)."""
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(A.ia)) + 1
    with open(path, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate complex general\n")
        fh.write(f"{A.n_rows} {A.n_cols} {A.nnz}\n")
        if A.nnz:
            fh.write("".join(f"{i} {j} {re:.17g} {im:.17g}\n" for i, j, re, im in
                             zip(rows.tolist(), (A.ja + 1).tolist(), A.aa.real.tolist(), A.aa.imag.tolist())))


# ---- binary CSR: u64 n, u64 nz, IA (n+1 u64), JA (nz u64), AA (nz re/im pairs) -------

def write_csr_binary(A: CsrMatrix, path) -> None:
    """Little-endian dump of a square CSR matrix (sparse.py:380-387)."""
    n = A.n  # raises for rectangular
    with open(path, "wb") as fh:
        fh.write(_BIN_HEADER.pack(n, A.nnz))
        fh.write(A.ia.astype("<u8").tobytes())
        fh.write(A.ja.astype("<u8").tobytes())
        fh.write(A.aa.astype("<c16", copy=False).tobytes())


def read_csr_binary(path) -> CsrMatrix:
    """Inverse of :func:`write_csr_binary` (sparse.py:390-402); validated."""
    with open(path, "rb") as fh:
        header = fh.read(_BIN_HEADER.size)
        if len(header) != _BIN_HEADER.size:
            raise ParseError(f"{path}: truncated header")
        n, nnz = _BIN_HEADER.unpack(header)
        ia = np.fromfile(fh, dtype="<u8", count=n + 1)
        ja = np.fromfile(fh, dtype="<u8", count=nnz)
        aa = np.fromfile(fh, dtype="<c16", count=nnz)
    if ia.shape[0] != n + 1 or ja.shape[0] != nnz or aa.shape[0] != nnz:
        raise ParseError(f"{path}: truncated arrays")
    return CsrMatrix(n, n, aa.astype(np.complex128), ja.astype(np.int64), ia.astype(np.int64))
