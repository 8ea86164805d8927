"""Does the L2 state left by the previous kernel slow the SpMV down?  Times
spmv(A, x) (CUDA events around each kernel) after different predecessors."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib, problems  # noqa: E402

n, ia, ja, aa, b = problems.helmholtz_27pt(int(os.environ.get("ZK_PROFILE_M", "200")))
A = Z.CsrMatrix(n, n, aa, ja, ia)
rng = np.random.default_rng(0)
x = Z.ZVector(rng.random(n) + 1j * rng.random(n))
other = Z.ZVector(rng.random(n) + 1j * rng.random(n))
third = Z.ZVector(rng.random(n) + 1j * rng.random(n))
Z.spmv(A, x)
for v in (other, third):  # upload once, outside the timed region
    Z.zscal(1.0, v)
_lib.synchronize()


def timed(pre, reps=6):
    tp = ts = 0.0
    for _ in range(reps):
        _lib.event_record(0)
        pre()
        _lib.event_record(1)
        Z.spmv(A, x)
        _lib.event_record(2)
        tp += _lib.event_elapsed_ms(0, 1)
        ts += _lib.event_elapsed_ms(1, 2)
    return round(tp / reps * 1e3, 1), round(ts / reps * 1e3, 1)


res = {
    "none": timed(lambda: None),
    "zscal_x": timed(lambda: Z.zscal(1.0, x)),
    "zscal_other": timed(lambda: Z.zscal(1.0, other)),
    "zaxpy_other": timed(lambda: Z.zaxpy(1.0, third, other)),
    "zdot_other": timed(lambda: Z.zdot(other, third)),
    "zscal_other_x": timed(lambda: (Z.zscal(1.0, other), Z.zscal(1.0, x))),
    "zaxpy_other_third": timed(lambda: (Z.zaxpy(1.0, other, third), Z.zscal(1.0, other))),
}
print(json.dumps(res))
