"""Host-side logic of the row-sharded solver on CPU: partition,
column renumbering, halo plans -- in process and over a world-size-2 gloo
group -- and a sharded SpMV assembled from the C oracle, bitwise equal to the
unsharded one (the elision decision and every row's order are preserved)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2112_06465_b200 import dist as D, problems

import dist_worker


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_partition(world):
    n, ia, ja, aa, b = problems.helmholtz_fd(3, 41)  # 64000 rows, 16 blocks
    bd = D.partition_rows(ia, world)
    assert bd[0] == 0 and bd[-1] == n and len(bd) == world + 1
    assert np.all(np.diff(bd) > 0)
    assert np.all(bd[:-1] % D.BLOCK == 0)
    nnz = np.diff(ia[bd])
    assert nnz.max() - nnz.min() <= 2 * D.BLOCK * 7  # balanced to within a couple of blocks


def test_partition_rejects_too_many_ranks():
    n, ia, ja, aa, b = problems.helmholtz_fd(3, 17)  # 4096 rows = 1 block
    with pytest.raises(Exception):
        D.partition_rows(ia, 2)


def _shards(ia, ja, world):
    bd = D.partition_rows(ia, world)
    out = []
    for r in range(world):
        r0, r1 = bd[r], bd[r + 1]
        lo, hi = ia[r0], ia[r1]
        jl, halo = D.localize(ja[lo:hi], r0, r1)
        out.append((r0, r1, ia[r0:r1 + 1] - lo, jl, halo, lo, hi))
    return bd, out


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_spmv_bitwise(world):
    O.set_arith(True, 262144)
    n, ia, ja, aa, b = problems.helmholtz_fd(3, 41, frequency=3.0, damping=0.3)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ref = O.spmv(n, n, ia, ja, aa, x)
    bd, shards = _shards(ia, ja, world)
    halos = [s[4] for s in shards]
    # the global SpMV swaps operands (nnz * 16 >= 256 KiB); shards must too
    O.set_arith(True, 1 if ia[-1] * 16 >= 262144 else 1 << 62)
    try:
        parts = []
        for r, (r0, r1, ial, jl, halo, lo, hi) in enumerate(shards):
            plan = D.HaloPlan(r, bd, halo, halos)
            xe = np.empty(r1 - r0 + len(halo), dtype=np.complex128)
            xe[: r1 - r0] = x[r0:r1]
            for q, (off, cnt) in plan.recv.items():  # what peer q sends: its rows at our halo columns
                qp = D.HaloPlan(q, bd, halos[q], halos)
                idx = qp.send[r]
                assert len(idx) == cnt
                xe[r1 - r0 + off: r1 - r0 + off + cnt] = x[bd[q] + idx]
            assert np.array_equal(xe[r1 - r0:], x[halo])
            parts.append(O.spmv(r1 - r0, len(xe), ial, jl, aa[lo:hi], xe))
    finally:
        O.set_arith(True, 262144)
    assert np.concatenate(parts).tobytes() == ref.tobytes()


def test_halo_plan_gloo_world2(tmp_path):
    world, port = 2, _free_port()
    mp.start_processes(dist_worker.plan_worker, args=(world, port, str(tmp_path), 41), nprocs=world,
                       start_method="spawn", join=True)
    n, ia, ja, aa, b = problems.helmholtz_fd(3, 41)
    bd, shards = _shards(ia, ja, world)
    halos = [s[4] for s in shards]
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        want = D.HaloPlan(r, bd, halos[r], halos)
        assert np.array_equal(got["bounds"], bd)
        assert np.array_equal(got["halo"], halos[r])
        assert [tuple(v) for v in got["recv"]] == [(q, o, c) for q, (o, c) in sorted(want.recv.items())]
        for q, idx in want.send.items():
            assert np.array_equal(got[f"send{q}"], idx)
