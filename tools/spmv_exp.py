"""Standalone zSpMV on C4 across ring depths (env ZK_NS caps the stage count;
NSS lists the depths to time)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib, problems  # noqa: E402

m = int(os.environ.get("ZK_PROFILE_M", "200"))
n, ia, ja, aa, b = problems.helmholtz_27pt(m)
A = Z.CsrMatrix(n, n, aa, ja, ia)
x = Z.ZVector(np.random.default_rng(0).random(n) + 0j)
bytes_ = 20 * ia[-1] + 4 * (n + 1) + 32 * n
res = {}
for exp in ("0",):
    for ns in os.environ.get("NSS", "4,6,8,10,12").split(","):
        os.environ["ZK_NS"] = ns
        Z.spmv(A, x)
        _lib.synchronize()
        _lib.event_record(0)
        for _ in range(10):
            Z.spmv(A, x)
        _lib.event_record(1)
        us = _lib.event_elapsed_ms(0, 1) / 10 * 1e3
        res[f"exp{exp}_ns{ns}"] = (round(us, 1), round(bytes_ / (us * 1e-6) / 1e9, 1))
print(json.dumps(res))
