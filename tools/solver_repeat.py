import sys, time
sys.path.insert(0, '/root/repo')
import paper_2112_06465_b200 as Z
from paper_2112_06465_b200 import problems, _lib
n, ia, ja, aa, b = problems.config_problem("C4")
A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
M = Z.build_jacobi(A)
bv = Z.ZVector(b)
cfg = Z.SolverConfig(tolerance=1e-8, max_iterations=1000, l=8)
for name, fn in (("l8", Z.solve_bicgstab_l), ("bicgstab", Z.solve_bicgstab), ("l8", Z.solve_bicgstab_l)):
    ts = []
    for k in range(5):
        _lib.synchronize()
        _lib.event_record(12)
        x, rep = fn(A, bv, M, cfg)
        _lib.event_record(13)
        ts.append(round(_lib.event_elapsed_ms(12, 13), 1))
    print(name, ts, rep.iterations, flush=True)
