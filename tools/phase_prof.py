"""Per-phase kernel times of one C4 Jacobi-BiCGStab solve (host-driven loop
with CUDA events around each kernel), plus the graph-launched solve time.
ZK_LIB_PATH selects a variant build."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib, problems  # noqa: E402

m = int(os.environ.get("ZK_PROFILE_M", "200"))
maxit = int(os.environ.get("MAXIT", "1000"))
n, ia, ja, aa, b = problems.helmholtz_27pt(m)
A = Z.CsrMatrix(n, n, aa, ja, ia)
M = Z.build_jacobi(A)
bv = Z.ZVector(b)
cfg = Z.SolverConfig(tolerance=1e-8, max_iterations=maxit)
x, rep = Z.solve_bicgstab(A, bv, M, cfg)
_lib.synchronize()
_lib.event_record(0)
for _ in range(3):
    x, rep = Z.solve_bicgstab(A, bv, M, cfg)
_lib.event_record(1)
solve_ms = _lib.event_elapsed_ms(0, 1) / 3
_lib.profile_enable(True)
x2, rep2 = Z.solve_bicgstab(A, bv, M, cfg)
prof = _lib.profile_read()
_lib.profile_enable(False)
same = rep2.residual_history == rep.residual_history
out = {"same_history": same, "iterations": rep.iterations, "final": rep.final_relative_residual, "solve_ms": round(solve_ms, 2),
       "solves_per_s": round(1e3 / solve_ms, 4),
       "phases_us": {k: round(v[0] / max(v[1], 1) * 1e3, 1) for k, v in prof.items() if v[1]}}
print(json.dumps(out))
