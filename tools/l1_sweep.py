"""C2 BLAS-1 sweep only (bench.blas1_sweep): zdotc / zaxpy / zscal / znrm2 at
1e4..1e8 with an L2 flush before every timed launch; prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

peak, _ = bench.peaks()
print(json.dumps(bench.blas1_sweep(peak)))
