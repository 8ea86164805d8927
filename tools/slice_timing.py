"""Experiment build (ZK_EXP>=10): per-slice consumer clock breakdown.
dbg[0] = cycles waiting for the stage, dbg[1] = cycles computing the rows,
dbg[2] = slices, dbg[5]/[6] = non-uniform/uniform slices."""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib, problems  # noqa: E402

L = _lib.load_library()
buf = (ctypes.c_ulonglong * 16)()


def read(reset=True, solver=0):
    L.zk_debug_read(buf, int(reset), int(solver))
    d = list(buf)
    n = max(d[2], 1)
    return {"wait_cyc": round(d[0] / n), "compute_cyc": round(d[1] / n), "slices": d[2],
            "uniform_frac": round(d[6] / max(d[5] + d[6], 1), 3),
            "uni_issue_cyc": round(d[7] / max(d[6], 1)), "uni_gather_lat_cyc": round(d[8] / max(d[6], 1)),
            "uni_compute_cyc": round(d[9] / max(d[6], 1))}


n, ia, ja, aa, b = problems.helmholtz_27pt(200)
A = Z.CsrMatrix(n, n, aa, ja, ia)
x = Z.ZVector(np.random.default_rng(0).random(n) + 0j)
Z.spmv(A, x)
read()
read(solver=1)
for _ in range(3):
    Z.spmv(A, x)
print("plain", json.dumps(read()))
M = Z.build_jacobi(A)
Z.solve_bicgstab(A, Z.ZVector(b), M, Z.SolverConfig(tolerance=1e-8, max_iterations=5))
print("solver(5 it)", json.dumps(read(solver=1)))
import time
_lib.synchronize()
t0 = time.time()
_lib.event_record(0)
for _ in range(3):
    Z.spmv(A, x)
_lib.event_record(1)
print("plain spmv us", round(_lib.event_elapsed_ms(0, 1) / 3 * 1e3, 1))
