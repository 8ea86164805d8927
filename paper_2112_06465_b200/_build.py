"""Build libzk.so in-tree with nvcc for sm_100a (no JIT cache; the .so
travels to the GPU box with the repository snapshot)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
OUT = os.path.join(OUT_DIR, "libzk.so")
SOURCES = ["zk_api.cu", "zk_blas1.cu", "zk_spmv.cu", "zk_bicgstab.cu", "zk_krylov.cu", "zk_plan.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no contraction anywhere -- the arithmetic must be the reference's
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-O2",
         "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def _obj(src, out_dir=OUT_DIR):
    return os.path.join(out_dir, "obj", os.path.splitext(src)[0] + ".o")


def _compile(src, verbose=False, out_dir=OUT_DIR, defines=()):
    obj = _obj(src, out_dir)
    cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return r.stderr


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in os.listdir(d):
            if os.path.getmtime(os.path.join(d, f)) > t:
                return True
    return False


def build(force: bool = False, verbose: bool = False, out_dir: str = OUT_DIR, defines=()) -> str:
    """Build libzk.so into out_dir (default: the package's lib/).  A different
    out_dir + defines builds a kernel variant for A/B experiments."""
    out = os.path.join(out_dir, "libzk.so")
    if out_dir == OUT_DIR and not defines and not force and not _stale():
        return OUT
    os.makedirs(os.path.join(out_dir, "obj"), exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        logs = list(ex.map(lambda s: _compile(s, verbose, out_dir, defines), SOURCES))
    if verbose:
        for s, l in zip(SOURCES, logs):
            if l.strip():
                print(f"== {s}\n{l}", file=sys.stderr)
    tmp = out + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[_obj(s, out_dir) for s in SOURCES], "-lcudart_static", "-lrt", "-ldl",
           "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
