import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2112_06465_b200 as Z
from oracle import oracle as O
from helpers import random_dominant_system
seeds = iter(range(300, 400))
bad = 0
for n in (10, 50, 200):
    for _ in range(10):
        seed = next(seeds)
        A, dense, b = random_dominant_system(n, 0.1, seed=seed)
        M = Z.build_jacobi(A)
        rng = np.random.default_rng(seed)
        xx = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ys = Z.spmv(A, Z.ZVector(xx)).data
        yo = O.spmv(n, n, A.ia, A.ja, A.aa, xx)
        x, rep = Z.solve_bicgstab(A, b, M, Z.SolverConfig(tolerance=1e-9))
        xo, hist, it, st, _ = O.bicgstab(n, A.ia, A.ja, A.aa, b.data, M.data, None, 1e-9, 1000)
        ok = rep.residual_history == hist
        if not ok or ys.tobytes() != yo.tobytes():
            bad += 1
            k = next((i for i, (a, c) in enumerate(zip(rep.residual_history, hist)) if a != c), None)
            print(f"n={n} seed={seed} spmv_ok={ys.tobytes()==yo.tobytes()} it={rep.iterations}/{it} first_diff={k} "
                  f"gpu={rep.residual_history[:k+2] if k is not None else None} ora={hist[:k+2] if k is not None else None}")
print("bad", bad)
