"""Row-sharded BiCGStab on the device: every rank's solution
slice, iteration count and residual history must be the unsharded
reference's bits.  Ranks share the one GPU of the test box over a gloo group
(host-staged halo/partials transport); the NCCL transport runs at world
size 1 (a single GPU cannot host two NCCL ranks)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2112_06465_b200 as Z
from oracle import oracle as O
from paper_2112_06465_b200 import problems

import dist_worker

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle(case):
    kind, cells, freq, damp, jac, guess, maxit = case
    O.set_arith(True, 262144)
    n, ia, ja, aa, b = problems.helmholtz_fd(3, cells, frequency=freq, damping=damp)
    A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
    minv = np.divide(1.0, A.diagonal()) if jac else None
    x0 = None
    if guess:
        rng = np.random.default_rng(7)
        x0 = rng.standard_normal(n) * 1e-3 + 0j
    if kind == "zero_rhs":
        b = np.zeros(n, dtype=np.complex128)
    return O.bicgstab(n, ia, ja, aa, b, minv, x0, 1e-8, maxit)


CASES = [
    ("jacobi", 33, 4.0, 0.3, True, False, 400),       # 32768 rows, 8 blocks, converges
    ("identity+guess", 33, 2.0, 0.3, False, True, 400),
    ("cap", 33, 4.0, 0.3, True, False, 5),             # stops at max_iterations
    ("zero_rhs", 33, 4.0, 0.3, True, False, 50),       # trivial result: x = 0, history [0.0]
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_sharded_bicgstab_gloo(tmp_path, world, case):
    port = _free_port()
    mp.start_processes(dist_worker.solve_worker, args=(world, port, str(tmp_path), case, "gloo"), nprocs=world,
                       start_method="spawn", join=True)
    xo, hist, it, st, _ = _oracle(case)
    xs = []
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        assert str(got["status"]) == "ok"
        assert int(got["it"]) == it, (r, int(got["it"]), it)
        assert np.asarray(got["hist"]).tobytes() == np.asarray(hist).tobytes(), r
        xs.append(got["x"])
    for x in xs:  # every rank returns the whole (all-gathered) solution
        assert x.tobytes() == xo.tobytes()


def test_sharded_bicgstab_nccl_world1(tmp_path):
    case = CASES[0]
    port = _free_port()
    mp.start_processes(dist_worker.solve_worker, args=(1, port, str(tmp_path), case, "nccl"), nprocs=1,
                       start_method="spawn", join=True)
    xo, hist, it, st, _ = _oracle(case)
    got = np.load(os.path.join(tmp_path, "rank0.npz"))
    assert int(got["it"]) == it
    assert np.asarray(got["hist"]).tobytes() == np.asarray(hist).tobytes()
    assert got["x"].tobytes() == xo.tobytes()
