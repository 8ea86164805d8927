"""Small driver for ncu captures: one launch of each hot kernel on C4-shaped
inputs (scale via ZK_PROFILE_M, default 200 = full C4)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import problems, _lib  # noqa: E402

m = int(os.environ.get("ZK_PROFILE_M", "200"))
n, ia, ja, aa, b = problems.helmholtz_27pt(m)
A = Z.CsrMatrix(n, n, aa, ja, ia)
M = Z.build_jacobi(A)
rng = np.random.default_rng(0)
x = Z.ZVector(rng.random(n) + 1j * rng.random(n))
for _ in range(2):
    Z.spmv(A, x)
nv = int(os.environ.get("ZK_PROFILE_NV", "100000000"))
v1 = Z.ZVector._device_new(nv)
v2 = Z.ZVector._device_new(nv)
_lib.check(_lib.lib().zk_memset(_lib.context(), v1._dptr_out(), 0, 16 * nv))
_lib.check(_lib.lib().zk_memset(_lib.context(), v2._dptr_out(), 0, 16 * nv))
for _ in range(2):
    Z.zdot(v1, v2)
    Z.znorm2(v1)
del v1, v2
os.environ["ZK_SOLVER_LOOP"] = "host"
Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-8, max_iterations=3))
_lib.synchronize()
print("done")
