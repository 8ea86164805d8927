"""``python -m paper_2112_06465_b200 kernel|spmv|solve ...`` -- the bench CLI
(zlinalg __main__.py / bench.py:399-432) on the device path."""
from .benchtool import main

raise SystemExit(main())
