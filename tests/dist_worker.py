"""Worker for the sharded-solver tests: one rank of a torch.distributed group
(127.0.0.1 rendezvous).  Writes its result to <out>/rank<k>.npz."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def plan_worker(rank, world, port, out, n_cells):
    """CPU only: halo plans over gloo must equal the in-process construction."""
    import torch.distributed as dist

    from paper_2112_06465_b200 import dist as D, problems
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n, ia, ja, aa, b = problems.helmholtz_fd(3, n_cells)
        bounds = D.partition_rows(ia, world)
        r0, r1 = bounds[rank], bounds[rank + 1]
        _, halo = D.localize(ja[ia[r0]:ia[r1]], r0, r1)
        plan = D.halo_plan(rank, bounds, halo)
        np.savez(os.path.join(out, f"rank{rank}.npz"), bounds=bounds, halo=halo,
                 recv=np.array([(q, o, c) for q, (o, c) in sorted(plan.recv.items())], dtype=np.int64).reshape(-1, 3),
                 **{f"send{q}": idx for q, idx in plan.send.items()})
    finally:
        dist.destroy_process_group()


def solve_worker(rank, world, port, out, case, backend):
    """GPU: one rank of the sharded solve (ranks may share one GPU with gloo)."""
    os.environ["ZK_DEVICE"] = "0"
    import torch
    import torch.distributed as dist

    import paper_2112_06465_b200 as Z
    from paper_2112_06465_b200 import dist as D, problems
    if backend == "nccl":
        torch.cuda.set_device(0)
    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        Z.set_arithmetic(True, 262144)
        kind, cells, freq, damp, jac, guess, maxit = case
        n, ia, ja, aa, b = problems.helmholtz_fd(3, cells, frequency=freq, damping=damp)
        if kind == "zero_rhs":
            b = np.zeros(n, dtype=np.complex128)
        A = Z.CsrMatrix(n, n, aa, ja, ia)
        M = Z.build_jacobi(A) if jac else None
        x0 = None
        if guess:
            rng = np.random.default_rng(7)
            x0 = Z.ZVector(rng.standard_normal(n) * 1e-3 + 0j)
        cfg = Z.SolverConfig(tolerance=1e-8, max_iterations=maxit, initial_guess=x0)
        transport = "nccl" if backend == "nccl" else "host"
        status, x, hist, it = "ok", np.zeros(0, np.complex128), [], -1
        try:
            xv, rep = D.solve_bicgstab_sharded(A, Z.ZVector(b), M, cfg, transport=transport)
            assert isinstance(xv, Z.ZVector)
            x, hist, it = xv.data, rep.residual_history, rep.iterations
        except Z.BreakdownError as e:
            status, hist, it = "breakdown", e.report.residual_history, e.report.iterations
        np.savez(os.path.join(out, f"rank{rank}.npz"), x=x, hist=np.asarray(hist), it=it, status=status)
    finally:
        dist.destroy_process_group()
