"""Row-sharded BiCGStab over several GPUs.

The reference solves on one CPU core; it has no distributed path.  Sharding
here changes nothing in the arithmetic: every rank runs the loop of
``krylov.solve_bicgstab`` (krylov.py:213-295) on its own rows, and every
reduction is completed in the *unsharded* order, so the solution, the
iteration count and every residual-history entry are bit-for-bit those of
the 1-GPU solve and of the reference.

* **Partition** (:func:`partition_rows`): contiguous row ranges whose
  boundaries are multiples of the 4096-element reduction block
  (``vecops.DEFAULT_PLAN``), balanced by nonzeros.  Every block partial is
  then computed whole on one rank.
* **Shard** (:func:`localize`): the rank's rows with columns renumbered --
  own rows ``[0, n)``, then the external ("halo") columns in ascending
  global order.  Entry order inside a row is untouched, so each row's
  products and sums are the unsharded ones.
* **Halo plan** (:func:`halo_plan`): for every peer, the contiguous slice of
  my halo it owns (receive) and the local indices of my rows it needs
  (send); built once with one object all-gather.
* **Exchange**: before each SpMV phase the gathered vector's halo is
  refreshed (pack kernel + point-to-point); after each reduction phase every
  rank's block partials are all-gathered and ``zk_dshard_finish`` folds them
  left to right in global block order (vecops.py:159-161) and runs the
  scalar recurrences -- the same bits on every rank.

The device work is libzk's (``zk_dshard_*``, include/zk.h); the transport is
``torch.distributed``: NCCL on device buffers (the GPUs of one node over
NVLink/NVSwitch, ops ordered on libzk's stream), or host staging over gloo
(tests: several ranks sharing one GPU).
"""
from __future__ import annotations

import ctypes
import time
import weakref

import numpy as np

from . import _lib
from .errors import BreakdownError, DimensionError, ParameterError
from .krylov import Preconditioner, SolveReport, SolverConfig, _BREAKDOWN_EPS, _BREAKDOWN_WHAT
from .sparse import CsrMatrix

__all__ = ["BLOCK", "partition_rows", "localize", "halo_plan", "HaloPlan", "ShardedBiCGStab",
           "solve_bicgstab_sharded"]

BLOCK = 4096  # vecops.DEFAULT_PLAN.block_size: rank boundaries must be multiples

# zk.h constants
DVEC_X, DVEC_PHAT, DVEC_SHAT, DVEC_B, DVEC_MINV, DVEC_PARTIALS, DVEC_GATHERED = range(7)
(PH_SETUP, PH_P_FIRST, PH_PIVOT, PH_S_UPDATE, PH_X_ALPHA, PH_TRUE_RES_S, PH_SPMV_T, PH_XR_UPDATE,
 PH_TRUE_RES, PH_P_NEXT) = range(10)


# ---- host-side planning (pure numpy; covered by the gloo tests on CPU) -------

def partition_rows(ia: np.ndarray, nranks: int) -> np.ndarray:
    """Row boundaries ``b[0]=0 < b[1] < ... < b[nranks]=n``: multiples of
    4096 (except ``n``), each rank at least one block, nonzeros balanced."""
    ia = np.asarray(ia, dtype=np.int64)
    n = ia.shape[0] - 1
    nb = -(-n // BLOCK)
    if nranks < 1 or nb < nranks:
        raise ParameterError(f"{n} rows ({nb} blocks of {BLOCK}) cannot be split over {nranks} ranks")
    ends = np.minimum(np.arange(1, nb + 1, dtype=np.int64) * BLOCK, n)
    cum = ia[ends]  # nonzeros up to the end of each block
    total = int(ia[-1])
    bounds = [0]
    for r in range(1, nranks):
        target = total * r / nranks
        k = int(np.searchsorted(cum, target))  # first block end reaching the target
        k = min(max(k + 1, bounds[-1] // BLOCK + 1), nb - (nranks - r))  # >= 1 block each side
        bounds.append(k * BLOCK)
    bounds.append(n)
    return np.asarray(bounds, dtype=np.int64)


def localize(ja_rows: np.ndarray, r0: int, r1: int):
    """Renumber a shard's global column indices: own rows -> ``[0, n)``,
    external columns -> ``n + position`` in the sorted halo.  Returns
    ``(ja_local, halo_cols)``."""
    ja_rows = np.asarray(ja_rows, dtype=np.int64)
    n = r1 - r0
    own = (ja_rows >= r0) & (ja_rows < r1)
    halo = np.unique(ja_rows[~own])
    ja_local = np.where(own, ja_rows - r0, n + np.searchsorted(halo, ja_rows))
    return ja_local.astype(np.int64), halo


class HaloPlan:
    """recv[q] = (offset, count): my halo slice owned by rank q;
    send[q] = local row indices rank q needs from me."""

    def __init__(self, rank: int, bounds: np.ndarray, halo: np.ndarray, all_halos):
        self.rank = rank
        self.bounds = np.asarray(bounds, dtype=np.int64)
        r0, r1 = self.bounds[rank], self.bounds[rank + 1]
        self.recv = {}
        self.send = {}
        for q in range(len(self.bounds) - 1):
            if q == rank:
                continue
            lo, hi = np.searchsorted(halo, [self.bounds[q], self.bounds[q + 1]])
            if hi > lo:
                self.recv[q] = (int(lo), int(hi - lo))
            theirs = np.asarray(all_halos[q], dtype=np.int64)
            a, b = np.searchsorted(theirs, [r0, r1])
            if b > a:
                self.send[q] = theirs[a:b] - r0

    @property
    def halo_size(self) -> int:
        return sum(c for _, c in self.recv.values())


def halo_plan(rank: int, bounds: np.ndarray, halo: np.ndarray, group=None) -> HaloPlan:
    """Exchange halo column lists (one all-gather of objects) and build the plan."""
    import torch.distributed as dist
    world = len(bounds) - 1
    if world == 1:
        return HaloPlan(rank, bounds, halo, [halo])
    all_halos = [None] * world
    dist.all_gather_object(all_halos, halo, group=group)
    return HaloPlan(rank, bounds, halo, all_halos)


# ---- transports ----------------------------------------------------------------

class _CudaArray:
    """Zero-copy torch view of a libzk device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _dev_tensor(ptr: int, count: int):
    import torch
    return torch.as_tensor(_CudaArray(ptr, count), device=f"cuda:{torch.cuda.current_device()}")


class NcclTransport:
    """Device-to-device over NCCL (one GPU per rank), ops ordered on libzk's stream."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        sp = ctypes.c_void_p()
        _lib.check(_lib.lib().zk_stream(_lib.context(), ctypes.byref(sp)))
        self.stream = torch.cuda.ExternalStream(sp.value)

    def ordered(self):
        import torch
        return torch.cuda.stream(self.stream)

    def gather_partials(self, shard):
        n = shard.partials_len
        src = _dev_tensor(shard.vec_ptr(DVEC_PARTIALS), n)
        dst = _dev_tensor(shard.vec_ptr(DVEC_GATHERED), n * shard.world)
        self.dist.all_gather_into_tensor(dst, src, group=self.group)

    def gather_x(self, shard):
        """The whole solution, all-gathered on the devices (rows padded to the
        largest shard), as a device-resident ZVector."""
        import torch
        from .vecops import ZVector
        nmax = int(np.diff(shard.bounds).max())
        with self.ordered():
            src = torch.zeros(2 * nmax, dtype=torch.float64, device=f"cuda:{torch.cuda.current_device()}")
            src[: 2 * shard.n].copy_(_dev_tensor(shard.vec_ptr(DVEC_X), 2 * shard.n))
            dst = torch.empty(2 * nmax * shard.world, dtype=src.dtype, device=src.device)
            self.dist.all_gather_into_tensor(dst, src, group=self.group)
            n = int(shard.bounds[-1])
            x = ZVector._device_new(n)
            out = _dev_tensor(x._dptr_out(), 2 * n)
            for q in range(shard.world):
                a, b = int(shard.bounds[q]), int(shard.bounds[q + 1])
                out[2 * a: 2 * b].copy_(dst[2 * q * nmax: 2 * q * nmax + 2 * (b - a)])
        self.stream.synchronize()
        return x._written()

    def halo(self, shard, which):
        plan = shard.plan
        if not plan.send and not plan.recv:
            return
        ops = []
        base = shard.vec_ptr(which)
        for q, (off, cnt) in plan.recv.items():
            ops.append(self.dist.P2POp(self.dist.irecv, _dev_tensor(base + 16 * (shard.n + off), 2 * cnt), q,
                                       group=self.group))
        for q, idx in plan.send.items():
            buf = shard.pack(which, q)
            ops.append(self.dist.P2POp(self.dist.isend, _dev_tensor(buf, 2 * len(idx)), q, group=self.group))
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()


class HostTransport:
    """Host-staged exchange over a CPU (gloo) process group: several ranks can
    share one GPU, so the sharded path is testable on a single device."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def ordered(self):
        import contextlib
        return contextlib.nullcontext()

    def gather_x(self, shard):
        from .vecops import ZVector
        x = np.empty(shard.n, dtype=np.complex128)
        _lib.check(_lib.lib().zk_memcpy_d2h(_lib.context(), x.ctypes.data, shard.vec_ptr(DVEC_X), 16 * shard.n))
        parts = [None] * shard.world
        self.dist.all_gather_object(parts, x, group=self.group)
        return ZVector(np.concatenate(parts))

    def gather_partials(self, shard):
        import torch
        n = shard.partials_len
        mine = np.empty(n, dtype=np.float64)
        _lib.check(_lib.lib().zk_memcpy_d2h(_lib.context(), mine.ctypes.data, shard.vec_ptr(DVEC_PARTIALS), 8 * n))
        parts = [torch.empty(n, dtype=torch.float64) for _ in range(shard.world)]
        self.dist.all_gather(parts, torch.from_numpy(mine), group=self.group)
        allp = np.ascontiguousarray(torch.cat(parts).numpy())
        _lib.check(_lib.lib().zk_memcpy_h2d(_lib.context(), shard.vec_ptr(DVEC_GATHERED), allp.ctypes.data,
                                            8 * allp.size))

    def halo(self, shard, which):
        import torch
        plan = shard.plan
        if not plan.send and not plan.recv:
            return
        base = shard.vec_ptr(which)
        works, sends, recvs = [], [], {}
        for q, idx in plan.send.items():
            buf = shard.pack(which, q)
            host = np.empty(2 * len(idx), dtype=np.float64)
            _lib.check(_lib.lib().zk_memcpy_d2h(_lib.context(), host.ctypes.data, buf, 8 * host.size))
            t = torch.from_numpy(host)
            sends.append(t)
            works.append(self.dist.isend(t, q, group=self.group))
        for q, (off, cnt) in plan.recv.items():
            t = torch.empty(2 * cnt, dtype=torch.float64)
            recvs[q] = (off, t)
            works.append(self.dist.irecv(t, q, group=self.group))
        for w in works:
            w.wait()
        for q, (off, t) in recvs.items():
            arr = np.ascontiguousarray(t.numpy())
            _lib.check(_lib.lib().zk_memcpy_h2d(_lib.context(), base + 16 * (shard.n + off), arr.ctypes.data,
                                                8 * arr.size))


# ---- the sharded solver ----------------------------------------------------------

class ShardedBiCGStab:
    """One rank's shard of a row-partitioned system.

    ``ia``/``ja``/``aa``: this rank's rows ``[row0, row1)`` (``ia`` rebased to
    0, ``ja`` global column indices, ascending per row); ``bounds``: every
    rank's row boundaries (:func:`partition_rows`); ``nnz_global``: nonzeros
    of the whole matrix (numpy's elision rule sees the whole SpMV).
    """

    def __init__(self, bounds, rank: int, ia, ja, aa, nnz_global: int, jacobi: bool = True,
                 max_iterations: int = 1000, group=None, transport: str = "nccl", layout=None):
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.world = len(self.bounds) - 1
        self.rank = rank
        self.row0, self.row1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.n = self.row1 - self.row0
        if self.row0 % BLOCK:
            raise ParameterError(f"shard start {self.row0} is not a multiple of {BLOCK}")
        ia = np.asarray(ia, dtype=np.int64)
        if ia.shape[0] != self.n + 1:
            raise DimensionError(f"shard has {self.n} rows but ia has {ia.shape[0]} pointers")
        # host-side shard layout (renumbered columns, halo plan): computed here,
        # or reused from an earlier shard of the same immutable matrix
        if layout is None:
            ja_local, halo = localize(ja, self.row0, self.row1)
            layout = (ja_local, halo, halo_plan(rank, self.bounds, halo, group))
        ja_local, halo, self.plan = layout
        self.layout = layout
        self.n_halo = int(halo.shape[0])
        self.rank_blocks = np.asarray([-(-(int(self.bounds[q + 1] - self.bounds[q])) // BLOCK)
                                       for q in range(self.world)], dtype=np.int64)
        self.maxb = int(self.rank_blocks.max())
        self.jacobi = bool(jacobi)
        self.cap = int(max_iterations)
        # local matrix: n rows, n + n_halo columns.  Renumbering puts halo
        # columns after the own ones, so a row's local indices need not
        # ascend (its entry order -- the summation order -- is the global
        # one); the device upload still range-checks every index.
        self.A = CsrMatrix(self.n, self.n + self.n_halo, aa, ja_local, ia, validate=False)
        lib = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(lib.zk_dshard_create(_lib.context(), self.A._device(), self.n_halo, int(nnz_global),
                                        int(self.jacobi), self.cap, self.world, self.maxb, ctypes.byref(h)))
        self._h = h
        self._ptr = {}
        # device index arrays + staging for the halo sends
        self._send = {}
        for q, idx in self.plan.send.items():
            ib = _lib.DeviceBuffer(8 * len(idx))
            arr = np.ascontiguousarray(idx, dtype=np.int64)
            _lib.check(lib.zk_memcpy_h2d(_lib.context(), ib.ptr, arr.ctypes.data, 8 * len(idx)))
            self._send[q] = (ib, _lib.DeviceBuffer(16 * len(idx)), len(idx))
        self.transport = NcclTransport(group) if transport == "nccl" else HostTransport(group)
        n_part = ctypes.c_int64()
        d = ctypes.POINTER(ctypes.c_double)()
        _lib.check(lib.zk_dshard_vector(self._h, DVEC_PARTIALS, ctypes.byref(d), ctypes.byref(n_part)))
        self.partials_len = int(n_part.value)  # two slots: two reductions per all-gather
        # NCCL: one CUDA graph per iteration (kernels, halo send/recv and
        # all-gathers on libzk's stream), replayed with one host launch;
        # ZK_DIST_GRAPH=0 issues op by op (and capture failures fall back).
        import os
        self.use_graph = transport == "nccl" and os.environ.get("ZK_DIST_GRAPH") != "0"
        self._graph = None

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.zk_dshard_destroy(self._h)
        except Exception:  # noqa: BLE001
            pass

    # -- device plumbing ----------------------------------------------------------
    def vec_ptr(self, which: int) -> int:
        p = self._ptr.get(which)
        if p is None:
            d, n = ctypes.POINTER(ctypes.c_double)(), ctypes.c_int64()
            _lib.check(_lib.lib().zk_dshard_vector(self._h, which, ctypes.byref(d), ctypes.byref(n)))
            p = ctypes.cast(d, ctypes.c_void_p).value
            self._ptr[which] = p
        return p

    def pack(self, which: int, q: int) -> int:
        ib, out, cnt = self._send[q]
        _lib.check(_lib.lib().zk_dshard_pack(self._h, which, ib.ptr, cnt, out.ptr))
        return out.ptr

    def _upload(self, which: int, arr, n: int) -> None:
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.complex128))
        if a.shape[0] != n:
            raise DimensionError(f"shard vector needs {n} entries, got {a.shape[0]}")
        _lib.check(_lib.lib().zk_memcpy_h2d(_lib.context(), self.vec_ptr(which), a.ctypes.data, 16 * n))

    def _phase(self, ph: int) -> None:
        _lib.check(_lib.lib().zk_dshard_phase(self._h, ph))

    def _finish(self, ph: int) -> None:
        _lib.check(_lib.lib().zk_dshard_finish(self._h, ph, self.rank_blocks.ctypes.data))

    def _reduce(self, ph: int) -> None:
        self._phase(ph)
        self.transport.gather_partials(self)
        self._finish(ph)

    def _status(self):
        rep, done = _lib.SolveReportC(), ctypes.c_int32()
        _lib.check(_lib.lib().zk_dshard_status(self._h, ctypes.byref(rep), ctypes.byref(done)))
        return rep, done.value

    def _iteration(self) -> None:
        """One loop iteration (krylov.py:254-294); every call is a device-side
        no-op once the solve stopped.  Four all-gathers and four halo
        exchanges: the s-check path's residual (K6x) is gathered with K4's
        <t,t>, <t,s>, and K5's <r~,r> with K61's residual (two partials slots;
        K4 / K61 run speculatively and their finishes are skipped when the
        preceding finish stopped the solve), then finished in the reference's
        order."""
        T = self.transport
        self._reduce(PH_S_UPDATE)
        self._phase(PH_X_ALPHA)
        T.halo(self, DVEC_X)
        self._phase(PH_TRUE_RES_S)
        T.halo(self, DVEC_SHAT)
        self._phase(PH_SPMV_T)
        T.gather_partials(self)
        self._finish(PH_TRUE_RES_S)
        self._finish(PH_SPMV_T)
        self._phase(PH_XR_UPDATE)
        T.halo(self, DVEC_X)
        self._phase(PH_TRUE_RES)
        T.gather_partials(self)
        self._finish(PH_XR_UPDATE)
        self._finish(PH_TRUE_RES)
        self._phase(PH_P_NEXT)
        T.halo(self, DVEC_PHAT)
        self._reduce(PH_PIVOT)

    def _capture(self):
        """CUDA graph of one iteration -- kernels and NCCL ops on libzk's
        stream -- so the host issues one launch per iteration."""
        import torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.transport.stream):
            self._iteration()
        return g

    # -- the loop -----------------------------------------------------------------
    def solve(self, b_local, minv_local=None, x0_local=None, tolerance: float = 1e-9,
              max_iterations: int = 1000, check_every: int = 8, gather: bool = False):
        """Returns ``(x_local, SolveReport)`` -- or, with ``gather``, the whole
        solution as a ZVector (device all-gather over NCCL) -- and raises
        BreakdownError like the reference.  Identical reports on every rank."""
        if max_iterations > self.cap:
            raise ParameterError(f"max_iterations {max_iterations} above this shard's {self.cap}")
        t0 = time.perf_counter()
        self._upload(DVEC_B, b_local, self.n)
        if self.jacobi:
            self._upload(DVEC_MINV, minv_local, self.n)
        if x0_local is not None:
            self._upload(DVEC_X, x0_local, self.n)
        lib, T = _lib.lib(), self.transport
        _lib.check(lib.zk_dshard_reset(self._h, float(tolerance), int(max_iterations), int(x0_local is not None)))
        with T.ordered():
            T.halo(self, DVEC_X)
            self._reduce(PH_SETUP)
            self._phase(PH_P_FIRST)
            T.halo(self, DVEC_PHAT)
            self._reduce(PH_PIVOT)
            step = self._iteration
            if self.use_graph:
                if self._graph is None:
                    try:
                        self._graph = self._capture()  # captured, not executed
                    except Exception:  # noqa: BLE001  (capture unsupported here: issue op by op)
                        self.use_graph = False
                if self._graph is not None:
                    step = self._graph.replay
            it = 0
            while True:
                step()
                it += 1
                if it % check_every == 0 or it >= max_iterations:
                    rep, done = self._status()
                    if done:
                        break
        rep, done = self._status()
        hist = np.empty(rep.history_len, dtype=np.float64)
        _lib.check(lib.zk_dshard_history(self._h, hist.ctypes.data, rep.history_len))
        if done == 2:  # zero rhs: x = 0 (krylov.py:174-178)
            _lib.check(lib.zk_memset(_lib.context(), self.vec_ptr(DVEC_X), 0, 16 * self.n))
        if gather:
            x = self.transport.gather_x(self)
        else:
            x = np.empty(self.n, dtype=np.complex128)
            _lib.check(lib.zk_memcpy_d2h(_lib.context(), x.ctypes.data, self.vec_ptr(DVEC_X), 16 * self.n))
        history = [float(v) for v in hist]
        report = SolveReport(iterations=int(rep.iterations), final_relative_residual=history[-1],
                             converged=bool(rep.converged), residual_history=history,
                             elapsed_ms=(time.perf_counter() - t0) * 1e3)
        if rep.breakdown:
            what = _BREAKDOWN_WHAT.get(int(rep.breakdown), "recurrence")
            raise BreakdownError(f"{what} numerically zero (|value| < {_BREAKDOWN_EPS:g}) after "
                                 f"{report.iterations} iterations", report=report)
        return x, report


_LAYOUTS = weakref.WeakKeyDictionary()  # CsrMatrix -> {(world, rank): (bounds, layout)}


def solve_bicgstab_sharded(A: CsrMatrix, b, M: Preconditioner | None = None, cfg: SolverConfig | None = None,
                           group=None, transport: str = "nccl"):
    """Row-sharded counterpart of :func:`krylov.solve_bicgstab` for one rank
    of ``group``: every rank passes the whole system and gets the whole
    solution (a ZVector, all-gathered device to device over NCCL) and the
    same report."""
    import torch.distributed as dist
    cfg = cfg or SolverConfig()
    n = A.n
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bvec = np.asarray(b.data if hasattr(b, "data") else b, dtype=np.complex128)
    if bvec.shape[0] != n:
        raise DimensionError(f"matrix is {n}x{n} but right-hand side has {bvec.shape[0]} elements")
    M = M if M is not None else Preconditioner.identity()
    # the partition and the shard layout depend only on the (immutable) matrix
    # and the group size: computed once per matrix; the device shard (upload,
    # SELL layout, workspace) is built on every call
    key = (world, rank)
    cached = _LAYOUTS.get(A, {}).get(key)
    if cached is None:
        bounds = partition_rows(A.ia, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        lo, hi = int(A.ia[r0]), int(A.ia[r1])
        ja_local, halo = localize(A.ja[lo:hi], r0, r1)
        cached = (bounds, (ja_local, halo, halo_plan(rank, bounds, halo, group)))
        _LAYOUTS.setdefault(A, {})[key] = cached
    bounds, layout = cached
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    lo, hi = int(A.ia[r0]), int(A.ia[r1])
    sh = ShardedBiCGStab(bounds, rank, A.ia[r0:r1 + 1] - lo, A.ja[lo:hi], A.aa[lo:hi], A.nnz,
                         jacobi=M.kind == "jacobi", max_iterations=cfg.max_iterations, group=group,
                         transport=transport, layout=layout)
    guess = cfg.initial_guess
    x0 = None if guess is None else np.asarray(guess.data, dtype=np.complex128)[r0:r1]
    minv = M.data[r0:r1] if M.kind == "jacobi" else None
    return sh.solve(bvec[r0:r1], minv, x0, cfg.tolerance, cfg.max_iterations, gather=True)
