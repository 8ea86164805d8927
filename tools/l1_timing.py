"""Standalone level-1 timings at 1e8 complex128 elements (GB/s by the SURVEY
8d byte model): zdotc 32 B/elem, znorm2 16, zaxpy 48, zscal 32."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06465_b200 as Z  # noqa: E402
from paper_2112_06465_b200 import _lib  # noqa: E402

nv = int(os.environ.get("NV", "100000000"))
v1 = Z.ZVector._device_new(nv)
v2 = Z.ZVector._device_new(nv)
_lib.check(_lib.lib().zk_memset(_lib.context(), v1._dptr_out(), 0, 16 * nv))
_lib.check(_lib.lib().zk_memset(_lib.context(), v2._dptr_out(), 0, 16 * nv))
res = {}
for name, fn, bpe in (("zdotc", lambda: Z.zdot(v1, v2), 32), ("znorm2", lambda: Z.znorm2(v1), 16),
                      ("zaxpy", lambda: Z.zaxpy(0.5 + 0.25j, v1, v2), 48), ("zscal", lambda: Z.zscal(1.0, v1), 32)):
    fn()
    _lib.synchronize()
    _lib.event_record(0)
    for _ in range(10):
        fn()
    _lib.event_record(1)
    us = _lib.event_elapsed_ms(0, 1) / 10 * 1e3
    res[name] = {"us": round(us, 1), "gbs": round(bpe * nv / (us * 1e-6) / 1e9, 1)}
print(json.dumps(res))
