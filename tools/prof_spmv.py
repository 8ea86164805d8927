"""One standalone zSpMV launch on C4 for an ncu capture (-k k_spmv -c 1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib, problems  # noqa: E402

m = int(os.environ.get("ZK_PROFILE_M", "200"))
n, ia, ja, aa, b = problems.helmholtz_27pt(m)
A = Z.CsrMatrix(n, n, aa, ja, ia)
rng = np.random.default_rng(42)
x = Z.ZVector(rng.random(n) + 1j * rng.random(n))
for _ in range(int(os.environ.get("REPS", "2"))):
    Z.spmv(A, x)
_lib.synchronize()
print("done")
