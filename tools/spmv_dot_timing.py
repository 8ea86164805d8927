"""C4: plain zSpMV vs the fused SpMV + <w, y> kernel (zk_spmv_dotc) under the
same conditions -- separates the fused-reduction cost from the solver context."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib, problems  # noqa: E402
from paper_2112_06465_b200.sparse import spmv_dot  # noqa: E402

n, ia, ja, aa, b = problems.helmholtz_27pt(200)
A = Z.CsrMatrix(n, n, aa, ja, ia)
rng = np.random.default_rng(0)
x = Z.ZVector(rng.random(n) + 1j * rng.random(n))
w = Z.ZVector(rng.random(n) + 1j * rng.random(n))
res = {}
for name, fn in (("spmv", lambda: Z.spmv(A, x)), ("spmv_dot", lambda: spmv_dot(A, x, w))):
    fn()
    _lib.synchronize()
    _lib.event_record(0)
    for _ in range(10):
        fn()
    _lib.event_record(1)
    res[name + "_us"] = round(_lib.event_elapsed_ms(0, 1) / 10 * 1e3, 1)
print(json.dumps(res))
