"""Where the e2e step's time goes (C4): matrix upload + SELL build (streamed),
solve (incl. b / M^-1 upload), solution readback; plus the raw pinned H2D
rate of this box for reference."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_06465_b200 as Z
from paper_2112_06465_b200 import problems, _lib

n, ia, ja, aa, b = problems.config_problem("C4")
M = Z.build_jacobi(Z.CsrMatrix(n, n, aa, ja, ia, validate=False))
minv = M.data
cfg = Z.SolverConfig(tolerance=1e-8)
for arr in (ia, ja, aa, b, minv):
    _lib.host_register(arr)
def ev(f):
    _lib.synchronize(); _lib.event_record(4); r = f(); _lib.event_record(5)
    return r, _lib.event_elapsed_ms(4, 5)
dev = Z.ZVector._device_new(aa.shape[0])
_, t = ev(lambda: _lib.check(_lib.lib().zk_memcpy_h2d(_lib.context(), dev._dptr_out(), aa.ctypes.data, aa.nbytes)))
print(f"raw pinned H2D: {aa.nbytes / t / 1e6:.1f} GB/s ({aa.nbytes/1e9:.2f} GB in {t:.1f} ms)")
del dev
for k in range(3):
    t0 = time.perf_counter()
    A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
    _, t_up = ev(A._device)
    Me = Z.Preconditioner("jacobi", minv)
    be = Z.ZVector(b)
    (x, rep), t_solve = ev(lambda: Z.solve_bicgstab(A, be, Me, cfg))
    xh, t_rd = ev(lambda: x.data)
    print(f"upload+build {t_up:.1f} ms ({(ia.nbytes + ja.nbytes + aa.nbytes) / t_up / 1e6:.1f} GB/s)  "
          f"solve(incl. b/M upload) {t_solve:.1f} ms  readback {t_rd:.1f} ms  wall {1e3*(time.perf_counter()-t0):.1f} ms")
    del A
