"""CSR matrices and SpMV (drop-in for the hot-path part of zlinalg sparse.py).

``CsrMatrix`` keeps the reference's constructor, fields and validation
(sparse.py:60-158): zero-based int64 ``ia``/``ja``, complex128 ``aa``,
strictly increasing columns per row, immutable after construction.  The
first kernel that needs it uploads it once into libzk's SELL-32 device layout
(int32 columns; csrc/zk_spmv.cuh) and keeps the handle for the matrix's
lifetime.  ``spmv`` runs on the device and returns a device-resident
``ZVector`` with the reference's bits (sparse.py:217-232).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DimensionError, FormatError
from .vecops import ZVector

__all__ = ["CooMatrix", "CsrMatrix", "coo_to_csr", "spmv", "spmv_dot"]


@dataclass
class CooMatrix:
    """(row, col, value) triples; duplicates are summed by :func:`coo_to_csr`."""

    n_rows: int
    n_cols: int
    entries: list = field(default_factory=list)

    def __post_init__(self):
        if self.n_rows < 0 or self.n_cols < 0:
            raise FormatError(f"negative dimensions ({self.n_rows}, {self.n_cols})")

    def add(self, i: int, j: int, value) -> None:
        if not (0 <= i < self.n_rows and 0 <= j < self.n_cols):
            raise FormatError(f"entry ({i}, {j}) outside {self.n_rows}x{self.n_cols} matrix")
        self.entries.append((i, j, complex(value)))

    @property
    def nnz(self) -> int:
        return len(self.entries)


class CsrMatrix:
    """Compressed sparse row matrix over complex128 values (immutable)."""

    __slots__ = ("n_rows", "n_cols", "aa", "ja", "ia", "_handle", "__weakref__")

    def __init__(self, n_rows, n_cols, aa, ja, ia, validate=True):
        object.__setattr__(self, "_handle", None)
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.aa = np.ascontiguousarray(np.asarray(aa, dtype=np.complex128))
        self.ja = np.ascontiguousarray(np.asarray(ja, dtype=np.int64))
        self.ia = np.ascontiguousarray(np.asarray(ia, dtype=np.int64))
        if validate:
            self._check()

    def _check(self):
        nnz = self.aa.shape[0]
        if self.ja.shape[0] != nnz:
            raise FormatError(f"aa has {nnz} values but ja has {self.ja.shape[0]} indices")
        if self.ia.shape[0] != self.n_rows + 1:
            raise FormatError(f"ia must have n_rows+1 = {self.n_rows + 1} pointers, got {self.ia.shape[0]}")
        if self.n_rows == 0:
            if nnz:
                raise FormatError("nonzeros in a 0-row matrix")
            return
        if self.ia[0] != 0 or self.ia[-1] != nnz:
            raise FormatError(f"row pointers must span [0, {nnz}], got [{self.ia[0]}, {self.ia[-1]}]")
        steps = np.diff(self.ia)
        if np.any(steps < 0):
            raise FormatError("row pointers are not nondecreasing")
        if nnz:
            if self.ja.min() < 0 or self.ja.max() >= self.n_cols:
                raise FormatError("column index out of range")
            if nnz > 1:
                # a step inside a row must be positive; row starts are exempt
                row_start = np.zeros(nnz, dtype=bool)
                row_start[self.ia[:-1][steps > 0]] = True
                if np.any(np.diff(self.ja)[~row_start[1:]] <= 0):
                    raise FormatError("column indices are not strictly increasing within a row")

    # -- shape ----------------------------------------------------------------
    @property
    def n(self) -> int:
        if self.n_rows != self.n_cols:
            raise DimensionError(f"matrix is {self.n_rows}x{self.n_cols}, not square")
        return self.n_rows

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @property
    def nnz(self) -> int:
        return self.aa.shape[0]

    def row(self, i: int):
        lo, hi = self.ia[i], self.ia[i + 1]
        return self.ja[lo:hi], self.aa[lo:hi]

    def diagonal(self) -> np.ndarray:
        """Stored main-diagonal entries, 0 where absent (sparse.py:125-134),
        vectorised: columns are strictly increasing, so each row matches at
        most once."""
        n = min(self.n_rows, self.n_cols)
        diag = np.zeros(n, dtype=np.complex128)
        if self.nnz:
            rows = np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.ia))
            hit = (rows == self.ja) & (rows < n)
            diag[rows[hit]] = self.aa[hit]
        return diag

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.n_rows, self.n_cols), dtype=np.complex128)
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.ia))
        dense[rows, self.ja] = self.aa
        return dense

    @classmethod
    def identity(cls, n: int) -> "CsrMatrix":
        return cls(n, n, np.ones(n, dtype=np.complex128), np.arange(n), np.arange(n + 1))

    def __repr__(self):
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"

    # -- device twin ----------------------------------------------------------
    def _device(self):
        """libzk handle of the SELL-32 copy (uploaded on first use)."""
        h = self._handle
        if h is None:
            out = ctypes.c_void_p()
            lib = _lib.lib()
            _lib.check(lib.zk_csr_create(_lib.context(), self.n_rows, self.n_cols, self.nnz,
                                         self.ia.ctypes.data, self.ja.ctypes.data if self.nnz else None,
                                         self.aa.ctypes.data if self.nnz else None, ctypes.byref(out)))
            h = _Handle(out.value)
            object.__setattr__(self, "_handle", h)
        return h.ptr

    def release_device(self) -> None:
        """Drop the device copy (the next kernel re-uploads)."""
        object.__setattr__(self, "_handle", None)

    def device_bytes(self):
        """(bytes of the device layout, padded element count)."""
        b, p = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().zk_csr_bytes(self._device(), ctypes.byref(b), ctypes.byref(p)))
        return b.value, p.value


class _Handle:
    __slots__ = ("ptr",)

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr and _lib._lib is not None:
                _lib._lib.zk_csr_destroy(self.ptr)
        except Exception:  # noqa: BLE001
            pass
        self.ptr = None


def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """Sort by (row, col) and sum duplicates (host ingestion, sparse.py:174-214)."""
    n_rows, n_cols = m.n_rows, m.n_cols
    if hasattr(m, "arrays"):  # array-backed (matio.ArrayCooMatrix): no tuple list
        rows, cols, vals = m.arrays()
    else:
        rows = np.fromiter((e[0] for e in m.entries), dtype=np.int64, count=len(m.entries))
        cols = np.fromiter((e[1] for e in m.entries), dtype=np.int64, count=len(m.entries))
        vals = np.fromiter((complex(e[2]) for e in m.entries), dtype=np.complex128, count=len(m.entries))
    if rows.shape[0] == 0:
        return CsrMatrix(n_rows, n_cols, np.zeros(0, np.complex128), np.zeros(0, np.int64),
                         np.zeros(n_rows + 1, np.int64))
    bad = (rows < 0) | (rows >= n_rows) | (cols < 0) | (cols >= n_cols)
    if bad.any():
        k = int(np.flatnonzero(bad)[0])
        raise FormatError(f"entry ({rows[k]}, {cols[k]}) outside {n_rows}x{n_cols} matrix")
    key = rows * np.int64(n_cols) + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    first = np.flatnonzero(np.concatenate(([True], key[1:] != key[:-1])))
    summed = np.add.reduceat(vals, first)
    ukey = key[first]
    counts = np.bincount(ukey // n_cols, minlength=n_rows)
    ia = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=ia[1:])
    return CsrMatrix(n_rows, n_cols, summed, ukey % n_cols, ia)


def spmv_dot(A: CsrMatrix, x: ZVector, w: ZVector, conjugate: bool = True):
    """``(y, <w, y>)`` with ``y = A x``, fused in one pass over the matrix:
    bitwise ``spmv(A, x)`` then ``zdot(w, y, conjugate)`` (DEFAULT_PLAN)."""
    from .cnum import Cplx
    if len(x) != A.n_cols:
        raise DimensionError(f"matrix has {A.n_cols} columns, vector has {len(x)} elements")
    if len(w) != A.n_rows:
        raise DimensionError(f"vector lengths differ: {len(w)} vs {A.n_rows}")
    if A.n_rows == 0:
        return ZVector(np.zeros(0, dtype=np.complex128)), Cplx(0.0, 0.0)
    y = ZVector._device_new(A.n_rows)
    out = (ctypes.c_double * 2)()
    _lib.check(_lib.lib().zk_spmv_dotc(_lib.context(), A._device(), x._dptr(), y._dptr_out(), w._dptr(),
                                       int(bool(conjugate)), out))
    return y._written(), Cplx(out[0], out[1])


def spmv(A: CsrMatrix, x: ZVector) -> ZVector:
    """y = A x on the device; bitwise the reference's numpy result."""
    if len(x) != A.n_cols:
        raise DimensionError(f"matrix has {A.n_cols} columns, vector has {len(x)} elements")
    if A.n_rows == 0:
        return ZVector(np.zeros(0, dtype=np.complex128))
    y = ZVector._device_new(A.n_rows)
    xp = x._dptr()
    _lib.check(_lib.lib().zk_spmv(_lib.context(), A._device(), xp, y._dptr_out()))
    return y._written()


def __getattr__(name):  # the reference exports its I/O from sparse (sparse.py:160-402)
    if name in ("MatrixStats", "stats", "read_matrix_market", "write_matrix_market", "read_csr_binary",
                "write_csr_binary"):
        from . import matio
        return getattr(matio, name)
    raise AttributeError(name)
