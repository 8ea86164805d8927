"""Host numpy arithmetic fingerprint (TEST / BENCH INFRASTRUCTURE ONLY).

The reference's bits depend on which complex-multiply loop the host numpy
dispatches: with AVX512F/FMA3 it is the fused formula the
golden vectors and the CUDA kernels use.  This probe detects it by comparing
numpy's product with both restatements in the C oracle, and records the CPU
facts the bench's cpu_baseline reports.
"""
from __future__ import annotations

import os
import platform

import numpy as np

from . import oracle as O


def complex_multiply_formula() -> str:
    rng = np.random.default_rng(12345)
    a = rng.standard_normal(4099) + 1j * rng.standard_normal(4099)
    b = rng.standard_normal(4099) + 1j * rng.standard_normal(4099)
    got = (a * b).tobytes()
    try:
        O.set_arith(True, 262144)
        if O.zaxmy(b, a).tobytes() == got:
            return "fma"
        O.set_arith(False, 262144)
        if O.zaxmy(b, a).tobytes() == got:
            return "plain"
        return "unknown"
    finally:
        O.set_arith(True, 262144)


def host_facts() -> dict:
    try:
        from numpy._core._multiarray_umath import __cpu_dispatch__
    except Exception:  # noqa: BLE001
        __cpu_dispatch__ = []
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {
        "cpu_model": model or platform.processor(),
        "os_cpu_count": os.cpu_count(),
        "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
        "numpy": np.__version__,
        "numpy_dispatch_fma": "FMA3" in __cpu_dispatch__ or "AVX512F" in __cpu_dispatch__,
        "complex_multiply": complex_multiply_formula(),
    }
