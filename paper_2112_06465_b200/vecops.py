"""Level-1 complex kernels on device-resident vectors (drop-in for
zlinalg vecops.py).

``ZVector`` keeps the reference's contract -- it wraps a caller's complex128
array without copying and exposes it as ``.data`` (vecops.py:45-86) -- but
adds a device twin.  Whichever side was written last is authoritative:

* kernels run on the device copy (uploaded lazily from ``.data``) and mark
  the host copy stale;
* reading ``.data`` downloads into the *same* host array object (so aliases
  of it see the result) and, because the caller may then mutate it, marks the
  device copy stale.

Every kernel call goes through libzk.so (include/zk.h); a missing library or
device raises instead of falling back to numpy.
"""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cnum import Cplx
from .errors import DimensionError, ParameterError

__all__ = [
    "ZVector", "ReductionPlan", "SEQUENTIAL", "BLOCKED", "DEFAULT_PLAN",
    "zassign", "zscal", "zaxpy", "zaxmy", "zdot", "znorm2",
    "zscal_copy", "zaxpy_copy", "zaxmy_copy", "write_zvector", "read_zvector",
]

SEQUENTIAL = "sequential"
BLOCKED = "blocked"
_HDR = struct.Struct("<Q")


class ZVector:
    """Dense complex128 vector with lazily synchronised host and device copies."""

    __slots__ = ("_host", "_dev", "_n", "_host_ok", "_dev_ok", "__weakref__")

    def __init__(self, data):
        arr = np.asarray(data, dtype=np.complex128)
        if arr.ndim != 1:
            raise DimensionError(f"ZVector needs 1-D data, got shape {arr.shape}")
        self._host = np.ascontiguousarray(arr)
        self._n = int(self._host.shape[0])
        self._dev = None
        self._host_ok = True
        self._dev_ok = False

    # -- construction helpers ------------------------------------------------
    @classmethod
    def _device_new(cls, n: int) -> "ZVector":
        """Uninitialised device-resident vector (host array allocated on demand)."""
        v = cls.__new__(cls)
        v._host = None
        v._n = int(n)
        v._dev = _lib.DeviceBuffer(16 * v._n) if v._n else None
        v._host_ok = False
        v._dev_ok = True
        return v

    @classmethod
    def zeros(cls, n: int) -> "ZVector":
        return cls(np.zeros(int(n), dtype=np.complex128))

    @classmethod
    def from_values(cls, values) -> "ZVector":
        return cls(np.array([complex(v) for v in values], dtype=np.complex128))

    def copy(self) -> "ZVector":
        """Fresh vector with the same contents; stays on the device when the
        device copy is current (neither side of the source is invalidated)."""
        if self._dev_ok and self._n:
            out = ZVector._device_new(self._n)
            _lib.check(_lib.lib().zk_memcpy_d2d(_lib.context(), out._dev.ptr, self._dev.ptr, 16 * self._n))
            return out
        return ZVector(self._host_view().copy())

    # -- residency ------------------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        """The host array (the reference's ``.data``).  Callers may write
        through it (test_vecops.py:262-266, test_acceptance.py:146-148), so
        handing it out marks the device copy stale; the library's own
        read-only accesses go through ``_host_view`` instead."""
        if not self._host_ok:
            if self._host is None:
                self._host = np.empty(self._n, dtype=np.complex128)
            if self._n:
                _lib.check(_lib.lib().zk_memcpy_d2h(_lib.context(), self._host.ctypes.data, self._dev.ptr,
                                                    16 * self._n))
            self._host_ok = True
        self._dev_ok = False  # the caller may write through the array
        return self._host

    @data.setter
    def data(self, value):
        arr = np.ascontiguousarray(np.asarray(value, dtype=np.complex128))
        if arr.ndim != 1:
            raise DimensionError(f"ZVector needs 1-D data, got shape {arr.shape}")
        self._host = arr
        self._n = int(arr.shape[0])
        self._dev = None
        self._host_ok = True
        self._dev_ok = False

    def _host_view(self) -> np.ndarray:
        """Current contents on the host for reading (device copy stays valid)."""
        if not self._host_ok:
            self.data  # noqa: B018  (downloads)
            self._dev_ok = self._dev is not None
        return self._host

    def _dptr(self):
        """Device pointer of current contents (uploads if the host is newer)."""
        if self._n == 0:
            return None
        if not self._dev_ok:
            if self._dev is None or self._dev.nbytes < 16 * self._n:
                self._dev = _lib.DeviceBuffer(16 * self._n)
            _lib.check(_lib.lib().zk_memcpy_h2d(_lib.context(), self._dev.ptr, self._host.ctypes.data, 16 * self._n))
            self._dev_ok = True
        return self._dev.ptr

    def _dptr_out(self):
        """Device pointer for a kernel that overwrites the whole vector."""
        if self._n == 0:
            return None
        if self._dev is None:
            self._dev = _lib.DeviceBuffer(16 * self._n)
        return self._dev.ptr

    def _written(self) -> "ZVector":
        self._dev_ok = True
        self._host_ok = False
        return self

    # -- sequence protocol ---------------------------------------------------
    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i: int) -> Cplx:
        z = self._host_view()[int(i)]
        return Cplx(z.real, z.imag)

    def __setitem__(self, i: int, value) -> None:
        self.data[int(i)] = complex(value)

    def __iter__(self):
        for z in self._host_view().copy():
            yield Cplx(z.real, z.imag)

    def __repr__(self) -> str:
        return f"ZVector(len={self._n})"


@dataclass(frozen=True)
class ReductionPlan:
    """Reduction grouping: ``block_size`` elements per partial sum, partials
    folded in ascending block order (``blocked``), or one left-to-right loop
    (``sequential``)."""

    block_size: int = 4096
    mode: str = BLOCKED

    def __post_init__(self):
        bs = self.block_size
        if not (isinstance(bs, int) and 64 <= bs <= 65536 and bs & (bs - 1) == 0):
            raise ParameterError(f"block_size must be a power of two in [64, 65536], got {bs!r}")
        if self.mode not in (SEQUENTIAL, BLOCKED):
            raise ParameterError(f"mode must be {SEQUENTIAL!r} or {BLOCKED!r}, got {self.mode!r}")

    @property
    def _mode_code(self) -> int:
        return _lib.MODE_SEQUENTIAL if self.mode == SEQUENTIAL else _lib.MODE_BLOCKED


DEFAULT_PLAN = ReductionPlan()


def _same_length(a: ZVector, b: ZVector) -> None:
    if len(a) != len(b):
        raise DimensionError(f"vector lengths differ: {len(a)} vs {len(b)}")


def _call(name, *args):
    _lib.check(getattr(_lib.lib(), name)(_lib.context(), *args))


def zassign(dst: ZVector, src: ZVector) -> ZVector:
    """dst[i] = src[i] (vecops.py:117-121)."""
    _same_length(dst, src)
    if len(dst) and dst is not src:
        sp = src._dptr()
        _call("zk_zassign", len(dst), dst._dptr_out(), sp)
        dst._written()
    return dst


def zscal(alpha, x: ZVector) -> ZVector:
    """x[i] = x[i] * alpha in place (vecops.py:124-127)."""
    a = complex(alpha)
    if len(x):
        _call("zk_zscal", len(x), a.real, a.imag, x._dptr())
        x._written()
    return x


def zaxpy(alpha, x: ZVector, y: ZVector) -> ZVector:
    """y[i] = y[i] + alpha * x[i] in place (vecops.py:130-134)."""
    _same_length(x, y)
    a = complex(alpha)
    if len(y):
        xp = x._dptr()
        _call("zk_zaxpy", len(y), a.real, a.imag, xp, y._dptr())
        y._written()
    return y


def zaxmy(x: ZVector, y: ZVector) -> ZVector:
    """y[i] = y[i] * x[i] in place (vecops.py:137-141)."""
    _same_length(x, y)
    if len(y):
        xp = x._dptr()
        _call("zk_zaxmy", len(y), xp, y._dptr())
        y._written()
    return y


def zscal_copy(alpha, x: ZVector) -> ZVector:
    return zscal(alpha, x.copy())


def zaxpy_copy(alpha, x: ZVector, y: ZVector) -> ZVector:
    return zaxpy(alpha, x, y.copy())


def zaxmy_copy(x: ZVector, y: ZVector) -> ZVector:
    return zaxmy(x, y.copy())


def zdot(x: ZVector, y: ZVector, conjugate: bool = True, plan: ReductionPlan = DEFAULT_PLAN) -> Cplx:
    """sum_i cbar(x[i]) * y[i] with the reference's exact grouping
    (vecops.py:165-186): per-block numpy pairwise sums, left fold."""
    _same_length(x, y)
    n = len(x)
    if n == 0:
        return Cplx(0.0, 0.0)
    out = (ctypes.c_double * 2)()
    xp, yp = x._dptr(), y._dptr()
    _call("zk_zdotc", n, xp, yp, int(bool(conjugate)), plan.block_size, plan._mode_code, out)
    return Cplx(out[0], out[1])


def znorm2(x: ZVector, plan: ReductionPlan = DEFAULT_PLAN) -> float:
    """sqrt(sum_i |x[i]|^2) (vecops.py:189-200)."""
    n = len(x)
    if n == 0:
        return 0.0
    out = (ctypes.c_double * 1)()
    _call("zk_znorm2", n, x._dptr(), plan.block_size, plan._mode_code, out)
    return float(out[0])


def write_zvector(v: ZVector, path) -> None:
    """u64 little-endian length, then the (re, im) pairs (vecops.py:203-207)."""
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(len(v)))
        fh.write(v.data.astype("<c16", copy=False).tobytes())


def read_zvector(path) -> ZVector:
    with open(path, "rb") as fh:
        head = fh.read(_HDR.size)
        if len(head) != _HDR.size:
            raise ParameterError(f"{path}: truncated vector header")
        (n,) = _HDR.unpack(head)
        body = fh.read(16 * n)
    if len(body) != 16 * n:
        raise ParameterError(f"{path}: expected {n} elements, file is short")
    return ZVector(np.frombuffer(body, dtype="<c16").astype(np.complex128))
