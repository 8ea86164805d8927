"""Driver for ncu captures: the hot kernels of one BASELINE configuration
(ZK_PROFILE_CONFIG, default C4): two plain SpMVs, a 3-iteration solve with
the host-driven loop (so every phase kernel is a separate launch ncu can
see; inside the solver's CUDA graph the conditional WHILE node hides them),
and -- for C4 -- zdotc / znorm2 at 1e8 elements (ZK_PROFILE_NV)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import problems, _lib  # noqa: E402

cfg_name = os.environ.get("ZK_PROFILE_CONFIG", "C4")
n, ia, ja, aa, b = problems.config_problem(cfg_name)
A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
M = Z.build_jacobi(A)
rng = np.random.default_rng(0)
x = Z.ZVector(rng.random(n) + 1j * rng.random(n))
for _ in range(2):
    Z.spmv(A, x)
os.environ["ZK_SOLVER_LOOP"] = "host"
Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-8, max_iterations=3))
if cfg_name == "C4":
    nv = int(os.environ.get("ZK_PROFILE_NV", "100000000"))
    v1 = Z.ZVector._device_new(nv)
    v2 = Z.ZVector._device_new(nv)
    _lib.check(_lib.lib().zk_memset(_lib.context(), v1._dptr_out(), 0, 16 * nv))
    _lib.check(_lib.lib().zk_memset(_lib.context(), v2._dptr_out(), 0, 16 * nv))
    for _ in range(2):
        Z.zdot(v1, v2)
        Z.znorm2(v1)
_lib.synchronize()
print("done")
