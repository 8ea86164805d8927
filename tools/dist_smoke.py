"""Sharded solve under torchrun (one process per rank; --backend gloo lets the
ranks share one GPU): compares against the C oracle and prints one line per rank."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--cells", type=int, default=33)
    args = ap.parse_args()
    import torch.distributed as dist
    import paper_2112_06465_b200 as Z
    from paper_2112_06465_b200 import dist as D, problems
    from oracle import oracle as O
    rank = int(os.environ["RANK"])
    os.environ["ZK_DEVICE"] = "0" if args.backend == "gloo" else os.environ.get("LOCAL_RANK", "0")
    if args.backend == "nccl":
        import torch
        torch.cuda.set_device(int(os.environ["ZK_DEVICE"]))
    dist.init_process_group(args.backend)
    n, ia, ja, aa, b = problems.helmholtz_fd(3, args.cells, frequency=4.0, damping=0.3)
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    M = Z.build_jacobi(A)
    cfg = Z.SolverConfig(tolerance=1e-8, max_iterations=400)
    x, rep = D.solve_bicgstab_sharded(A, Z.ZVector(b), M, cfg, transport="nccl" if args.backend == "nccl" else "host")
    O.set_arith(True, 262144)
    xo, hist, it, st, _ = O.bicgstab(n, ia, ja, aa, b, M.data, None, 1e-8, 400)
    print(f"rank {rank}: it {rep.iterations} (oracle {it}) hist_equal {rep.residual_history == hist} "
          f"x_equal {x.data.tobytes() == xo.tobytes()}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
