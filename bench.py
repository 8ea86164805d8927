"""Benchmark: Jacobi-preconditioned BiCGStab solves/sec on BASELINE config C4
(car-compartment-scale 27-point Helmholtz, 200^3 = 8M rows, 214M nnz), with
zSpMV / zdotc GB/s against the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl zk|reference]

One step = one complete solve (b -> x, tol 1e-8) through the product path.
With N > 1 (torchrun) the same system is row-sharded over the N GPUs
(strong scaling, paper_2112_06465_b200/dist.py: halo exchange and block
partials over NCCL); the result is bit-for-bit the 1-GPU one.
`value` is timed with CUDA events on the library stream with every input
resident in HBM; `e2e` repeats the solve through the public Python API with
the matrix, right-hand side and preconditioner in pinned host memory (the
device copy of the matrix is dropped before every step, so each step uploads
and re-lays-out all 5.1 GB) and the solution read back.  The matrix (4.6 GB
in the device layout) is far larger than the 126 MB L2, so no flush is
needed between steps.

`--impl reference` times the reference's own CPU algorithm (oracle/port.py,
the same numpy operations as zlinalg) on this host, one BiCGStab iteration
per step, and extrapolates solves/sec with the iteration count of the
configuration (identical on both sides: the GPU path is bitwise the
reference).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "C4"  # the headline; --config C1|C3|C5 runs the other BASELINE systems
WORKLOADS = {
    "C1": "C1: 7-point Helmholtz FD 32^3 (cells=33, frequency 1.5), Jacobi BiCGStab tol 1e-8, x0=0 "
          "(the reference's CPU path)",
    "C3": "C3: cylinder P1-FE Helmholtz (996,369 rows, 14.7M nnz; k=4pi, eps=0.1, point source), "
          "Jacobi BiCGStab tol 1e-8, x0=0",
    "C4": "C4: 27-point Helmholtz 200^3, k^2=100, eps=0.05, Jacobi BiCGStab tol 1e-8, x0=0",
    "C5": "C5: 7-point Helmholtz FD 256^3, 12 points per wavelength, eps=0.3, Jacobi BiCGStab tol 1e-8, x0=0",
}
DATA = {
    "C1": "synthetic: reference 7-point FD assembly (bitwise helmholtz.assemble), unit interior source",
    "C3": "synthetic: generated P1 tetrahedral FE cylinder (Kuhn split), unit point source",
    "C4": "synthetic: generated 27-point Helmholtz stencil, unit interior source, zero Dirichlet",
    "C5": "synthetic: generated 7-point FD stencil, complex damping, unit interior source",
}
TOL = 1e-8
MAXIT = 20000
# Iteration counts of the BASELINE solves, bitwise identical between this GPU
# path and the reference algorithm (provenance in the file).  The GPU arm
# re-measures its count every run and checks it against this record; the
# reference arm needs it to extrapolate its per-iteration time.
ITERATIONS_FILE = os.path.join(ROOT, "tests", "golden", "headline_iterations.json")


def known_iterations(config: str):
    try:
        with open(ITERATIONS_FILE) as fh:
            return json.load(fh).get(config, {}).get("iterations")
    except OSError:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


# ---- distributed plumbing ---------------------------------------------------

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        # ZK_BENCH_TRANSPORT=host: ranks share GPU 0 over gloo (exercises the
        # sharded path on a 1-GPU box; not a performance configuration)
        self.transport = os.environ.get("ZK_BENCH_TRANSPORT", "nccl")
        if self.world > 1 or os.environ.get("ZK_BENCH_SHARDED") == "1":  # (1-rank shard: overhead check)
            import torch
            import torch.distributed as dist
            if self.transport == "nccl":
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                os.environ["ZK_DEVICE"] = "0"
                dist.init_process_group("gloo")
            self.dist, self.torch = dist, torch

    def barrier(self):
        if hasattr(self, "dist"):
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not hasattr(self, "dist"):
            return v
        dev = "cuda" if self.transport == "nccl" else "cpu"
        t = self.torch.tensor([v], dtype=self.torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if hasattr(self, "dist"):
            self.dist.destroy_process_group()


# ---- clocks -------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx = float(f[1])
                except ValueError:
                    continue
                for name, val in zip(names, f[4:8]):
                    if val.lower() == "active":
                        reasons.add(name)
        finally:
            os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


# ---- workload -------------------------------------------------------------------

def build_problem(config: str = CONFIG):
    from paper_2112_06465_b200 import problems
    n, ia, ja, aa, b = problems.config_problem(config)
    return n, ia, ja, aa, b


def algorithmic_bytes(n: int, nnz: int):
    """SURVEY 8d byte model (int32-index CSR, every array counted once)."""
    A = 20 * nnz + 4 * (n + 1) + 16 * n + 16 * n
    Ar = 20 * nnz + 4 * (n + 1)  # matrix stream only
    return {
        "spmv": A,
        "spmv_pivot": A,                      # v = A p^ (plain pipeline)
        "spmv2": A + 32 * n,                  # narrow matrices: t = A x and v = A p^ in one matrix pass
        "res_pass": 32 * n,                   # ||b - A x||: b, A x
        "pivot_first": A,
        "pivot_dot": 32 * n,                  # <r~, v>: r~, v
        "pivot_first_dot": 32 * n,
        "spmv_t": A,                          # t = A s^
        "tt_ts": 32 * n,                      # <t, t>, <t, s>: t, s
        "true_res": A,                        # t = A x (plain pipeline; b is read by the residual pass)
        "p_next": 96 * n,                     # p, v, r, minv -> p, p^
        "true_res_s": Ar + 32 * n,
        "s_update": 80 * n,
        "xr_update": 128 * n,
        "x_alpha": 48 * n,
        "p_first": 96 * n,
        # the minimum of SURVEY 8d (the <r~,v> and <t,s> operands counted with
        # their SpMV); the two reduction passes re-read v and t (+32n)
        "iteration": 3 * A + 336 * n,
    }


def traffic_from_profiles(kernel: str, config: str = CONFIG):
    """DRAM bytes (read + write) per launch of `kernel` on `config`, from the
    committed ncu capture of the current build (profiles/traffic.json:
    {"build": ..., "<config>": {"<kernel>": bytes}}); None when that
    configuration or kernel was not captured."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config, {}).get(kernel)
    except Exception:  # noqa: BLE001
        return None


def run_zk(args, dist: Dist):
    import paper_2112_06465_b200 as Z
    from paper_2112_06465_b200 import _lib

    peak, peak_kind = peaks()
    t0 = time.time()
    n, ia, ja, aa, b = build_problem(args.config)
    nnz = int(ia[-1])
    A = Z.CsrMatrix(n, n, aa, ja, ia)
    M = Z.build_jacobi(A)
    bv = Z.ZVector(b)
    cfg = Z.SolverConfig(tolerance=TOL, max_iterations=MAXIT)
    setup_s = time.time() - t0

    # ---- value: device-resident solves -------------------------------------
    A._device()
    bv._dptr()
    M._device_minv()._dptr()
    for _ in range(args.warmup):
        x, rep = Z.solve_bicgstab(A, bv, M, cfg)
    iters = rep.iterations
    dist.barrier()
    _lib.synchronize()
    l0 = Z.launch_count()
    with Clocks(dist.local) as clk:
        _lib.event_record(0)
        for _ in range(args.steps):
            x, rep = Z.solve_bicgstab(A, bv, M, cfg)
        _lib.event_record(1)
        ms = _lib.event_elapsed_ms(0, 1)
    launches = Z.launch_count() - l0
    _lib.synchronize()
    dist.barrier()
    ms_max = dist.max(ms)
    clocks = clk.summary()
    step_ms = ms_max / args.steps
    value = args.steps / (ms_max / 1e3)

    # ---- e2e: public API, pinned host inputs, fresh upload every step ---------
    pinned = [ia, ja, aa, b, M.data]
    for arr in pinned:
        _lib.host_register(arr)
    e2e_ms = []
    try:
        for k in range(args.steps + 1):
            Ae = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
            Me = Z.Preconditioner("jacobi", M.data)
            be = Z.ZVector(b)
            dist.barrier()
            _lib.synchronize()
            _lib.event_record(2)
            xe, repe = Z.solve_bicgstab(Ae, be, Me, cfg)
            xh = xe.data
            _lib.event_record(3)
            t = _lib.event_elapsed_ms(2, 3)
            if k:  # the first call also builds the solver graph; keep it as warm-up
                e2e_ms.append(t)
            del Ae
    finally:
        for arr in pinned:
            _lib.host_unregister(arr)
    e2e_step = dist.max(sum(e2e_ms) / len(e2e_ms))
    assert repe.iterations == iters and xh.tobytes() == x.data.tobytes()
    h2d = ia.nbytes + ja.nbytes + aa.nbytes + b.nbytes + M.data.nbytes
    d2h = 16 * n + 8 * (iters + 1)

    # ---- per-phase kernel times (host loop with events around each kernel) ----
    _lib.profile_enable(True)
    Z.solve_bicgstab(A, bv, M, cfg)
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    B = algorithmic_bytes(n, nnz)
    phases = {}
    conditional = ("x_alpha", "true_res_s")  # device no-ops unless the s-check fires: no bytes credited
    for name, (tms, cnt) in prof.items():
        if cnt:
            avg = tms / cnt
            entry = {"launches": cnt, "avg_us": round(avg * 1e3, 2), "total_ms": round(tms, 3)}
            if name in B and name not in conditional:
                entry["gbs"] = round(B[name] / (avg * 1e-3) / 1e9, 1)
            phases[name] = entry
    body = [p for p in ("s_update", "x_alpha", "true_res_s", "spmv_t", "tt_ts", "xr_update", "true_res", "res_pass",
                        "p_next", "spmv_pivot", "pivot_dot", "spmv2")
            if p in phases]
    # matrices at most 8 entries wide (no long rows) run the narrow SpMV kernels (zk_spmv.cuh)
    spmv_k = "k_spmv_phase_narrow" if int(np.diff(ia).max()) <= 8 and os.environ.get("ZK_NARROW") != "0" \
        else "k_spmv_phase"
    kernel_names = {"spmv_t": spmv_k, "spmv_pivot": spmv_k, "true_res": spmv_k, "spmv2": "k_spmv2_phase_narrow",
                    "res_pass": "k_res_pass",
                    "s_update": "k_s_update_pipe", "xr_update": "k_xr_update_pipe", "tt_ts": "k_tt_ts_pass",
                    "pivot_dot": "k_pivot_pass", "p_next": "k_p_next"}
    # dominant kernel = the most device time per solve, summed over the
    # phases it runs (k_spmv_phase serves both the K2 and K4 products)
    per_kernel = {}
    for p in body:
        if p in conditional:
            continue
        k = kernel_names.get(p, p)
        kt, kc, kb = per_kernel.get(k, (0.0, 0, 0))
        per_kernel[k] = (kt + prof[p][0], kc + prof[p][1], kb + B[p] * prof[p][1])
    dominant = max(per_kernel, key=lambda k: per_kernel[k][0])
    dom_ms, dom_cnt, dom_bytes = per_kernel[dominant]
    dom_avg_s = dom_ms / dom_cnt / 1e3
    dom_bytes_launch = dom_bytes / dom_cnt
    achieved = dom_bytes_launch / dom_avg_s / 1e9
    iter_s = sum(prof[p][0] for p in body) / max(prof["s_update"][1], 1) / 1e3

    # ---- standalone kernels: zSpMV on C4, zdotc / zaxpy at 1e8 ------------------
    rng = np.random.default_rng(42)
    xs = Z.ZVector(rng.random(n) + 1j * rng.random(n))
    y = Z.spmv(A, xs)
    _lib.synchronize()
    reps = 20
    _lib.event_record(4)
    for _ in range(reps):
        Z.spmv(A, xs)
    _lib.event_record(5)
    spmv_ms = _lib.event_elapsed_ms(4, 5) / reps
    del y
    sweep = blas1_sweep(peak) if not args.no_sweep else {}
    others = {} if args.no_solvers else other_solvers(A, bv, M, B["spmv"])
    sub = {
        "zspmv_gbs": round(B["spmv"] / (spmv_ms * 1e-3) / 1e9, 1),
        "zspmv_frac": round(B["spmv"] / (spmv_ms * 1e-3) / 1e9 / peak, 3),
        "zspmv_us": round(spmv_ms * 1e3, 1),
        "c2_blas1_sweep": sweep,
        "other_solvers": others,
        "bicgstab_iteration_gbs": round(B["iteration"] / iter_s / 1e9, 1),
        "bicgstab_iteration_frac": round(B["iteration"] / iter_s / 1e9 / peak, 3),
        "bicgstab_iteration_us": round(iter_s * 1e6, 1),
        "phases": phases,
    }

    out = {
        "metric": "bicgstab_solves_per_sec",
        "value": round(value, 4),
        "unit": "solves/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128 (f64 re/im pairs)",
        "data": DATA[args.config],
        "config": {"workload": WORKLOADS[args.config], "n": n, "nnz": nnz, "iterations": iters},
        "detail": {
            "converged": bool(rep.converged), "final_rel": rep.final_relative_residual,
            "parallelism": "1 GPU",
            "l2": "inputs larger than L2 (4.6 GB matrix, 126 MB L2): no flush",
            "host_setup_s": round(setup_s, 1),
        },
        "e2e": {"value": round(1.0 / (e2e_step / 1e3), 4), "unit": "solves/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": round(e2e_step, 3),
                "path": "solve_bicgstab(CsrMatrix, ZVector, Preconditioner) from pinned host arrays, x.data read"},
        "roofline": {"bound": "hbm", "kernel": dominant,
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 3), "peak_kind": peak_kind,
                     "bytes_per_launch": int(dom_bytes_launch), "avg_launch_us": round(dom_avg_s * 1e6, 1),
                     "launches_per_solve": int(dom_cnt),
                     "traffic": traffic_from_profiles(dominant, args.config)},
        "clocks": clocks,
        "gpu_launches": int(launches),
        "sub_metrics": sub,
    }
    known = known_iterations(args.config)
    out["parity"] = {"iterations_committed": known,
                     "iterations_match_committed": None if known is None else known == iters}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        cb, detail = cpu_baseline(ia, ja, aa, b, M.data, iters, args.config)
        out["cpu_baseline"] = cb
        # parity of the measured path with the reference algorithm: the CPU
        # sample's first iteration (residual history prefix and x) against a
        # 1-iteration solve of the same system on the GPU, bitwise
        x1, rep1 = Z.solve_bicgstab(A, bv, M, Z.SolverConfig(tolerance=TOL, max_iterations=1))
        same_fp = cb["host"].get("complex_multiply") == "fma"
        hist_ok = np.array(rep1.residual_history).tobytes() == np.array(detail["hist"]).tobytes()
        x_ok = x1.data.tobytes() == detail["x"].tobytes()
        out["parity"].update({"hist_prefix_bitwise": hist_ok, "x_after_1_iteration_bitwise": x_ok,
                              "hist_prefix": detail["hist"], "checked_against": "oracle/port.py (numpy) on this host",
                              "host_fingerprint_matches": same_fp})
        if same_fp and not (hist_ok and x_ok):
            raise SystemExit(f"parity failure: GPU {rep1.residual_history} vs reference algorithm {detail['hist']}")
    if out["parity"]["iterations_match_committed"] is False:
        raise SystemExit(f"iteration count {iters} differs from the committed bitwise record {known}")
    if dist.rank == 0:
        print(json.dumps(out), flush=True)


def run_sharded(args, dist: Dist):
    """N > 1: the C4 system row-sharded over the N GPUs (strong scaling,
    paper_2112_06465_b200/dist.py); every rank gets the unsharded bits."""
    import paper_2112_06465_b200 as Z
    from paper_2112_06465_b200 import _lib, dist as D

    peak, peak_kind = peaks()
    t0 = time.time()
    n, ia, ja, aa, b = build_problem(args.config)
    nnz = int(ia[-1])
    A = Z.CsrMatrix(n, n, aa, ja, ia, validate=False)
    M = Z.build_jacobi(A)
    bounds = D.partition_rows(ia, dist.world)
    r0, r1 = int(bounds[dist.rank]), int(bounds[dist.rank + 1])
    lo, hi = int(ia[r0]), int(ia[r1])
    transport = "nccl" if dist.transport == "nccl" else "host"
    shard = D.ShardedBiCGStab(bounds, dist.rank, ia[r0:r1 + 1] - lo, ja[lo:hi], aa[lo:hi], nnz, jacobi=True,
                              max_iterations=MAXIT, transport=transport)
    b_loc, m_loc = b[r0:r1], M.data[r0:r1]
    setup_s = time.time() - t0
    for _ in range(args.warmup):
        x, rep = shard.solve(b_loc, m_loc, None, TOL, MAXIT)
    dist.barrier()
    _lib.synchronize()
    l0 = Z.launch_count()
    with Clocks(dist.local) as clk:
        _lib.event_record(0)
        for _ in range(args.steps):
            x, rep = shard.solve(b_loc, m_loc, None, TOL, MAXIT)
        _lib.event_record(1)
        ms = _lib.event_elapsed_ms(0, 1)
    launches = Z.launch_count() - l0
    _lib.synchronize()
    dist.barrier()
    ms_max = dist.max(ms)
    step_ms = ms_max / args.steps
    # e2e: the public sharded API from host arrays (partition, shard upload,
    # halo plan, solve, all-gather of x) every step
    e2e_ms = []
    cfg = Z.SolverConfig(tolerance=TOL, max_iterations=MAXIT)
    for k in range(2):
        dist.barrier()
        t1 = time.perf_counter()
        xe, repe = D.solve_bicgstab_sharded(A, b, M, cfg, transport=transport)
        e2e_ms.append((time.perf_counter() - t1) * 1e3)
    e2e_step = dist.max(statistics.median(e2e_ms))
    assert repe.iterations == rep.iterations
    # roofline: zSpMV on this rank's shard (own rows, halo columns)
    xs = Z.ZVector(np.random.default_rng(42).random(shard.n + shard.n_halo) + 0j)
    Z.spmv(shard.A, xs)
    _lib.synchronize()
    _lib.event_record(4)
    for _ in range(10):
        Z.spmv(shard.A, xs)
    _lib.event_record(5)
    spmv_ms = _lib.event_elapsed_ms(4, 5) / 10
    snnz = hi - lo
    sb = 20 * snnz + 4 * (shard.n + 1) + 16 * (shard.n + shard.n_halo) + 16 * shard.n
    out = {
        "metric": "bicgstab_solves_per_sec",
        "value": round(args.steps / (ms_max / 1e3), 4),
        "unit": "solves/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128 (f64 re/im pairs)",
        "data": DATA[args.config],
        "config": {"workload": WORKLOADS[args.config], "n": n, "nnz": nnz, "iterations": rep.iterations},
        "detail": {
            "converged": bool(rep.converged), "final_rel": rep.final_relative_residual,
            "parallelism": f"row-sharded x{dist.world} ({transport}): 4096-aligned nnz-balanced rows, halo "
                           f"exchange before each SpMV, all-gathered block partials folded in global order",
            "shard_rows": [int(v) for v in np.diff(bounds)], "halo_rows_rank0": shard.n_halo,
            "l2": "inputs larger than L2: no flush",
            "host_setup_s": round(setup_s, 1),
        },
        "e2e": {"value": round(1.0 / (e2e_step / 1e3), 4), "unit": "solves/s",
                "h2d_bytes_per_step": int(20 * nnz + 8 * (n + 1) + 32 * n),
                "d2h_bytes_per_step": int(16 * n + 8 * (rep.iterations + 1)),
                "ms_per_step": round(e2e_step, 3),
                "path": "dist.solve_bicgstab_sharded(CsrMatrix, b, Preconditioner) from host arrays: partition, "
                        "shard upload, halo plan, solve, all-gather of x"},
        "roofline": {"bound": "hbm", "kernel": "k_spmv (rank 0 shard)",
                     "achieved": round(sb / (spmv_ms * 1e-3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(sb / (spmv_ms * 1e-3) / 1e9 / peak, 3), "peak_kind": peak_kind,
                     "bytes_per_launch": int(sb), "avg_launch_us": round(spmv_ms * 1e3, 1), "traffic": None},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
    }
    if dist.rank == 0:
        print(json.dumps(out), flush=True)


def other_solvers(A, bv, M, spmv_bytes, steps: int = 3):
    """The paper's other two solvers on the same system:
    BiCGSTAB(8) and TFQMR (krylov.py:298-489), device-resident, timed with
    CUDA events per solve (one graph launch each) after two warm-up solves
    (the first builds the graph; the second was measured up to 35% slow)."""
    import paper_2112_06465_b200 as Z
    from paper_2112_06465_b200 import _lib
    out = {}
    for name, fn, cfg in (("bicgstab_l8", Z.solve_bicgstab_l, Z.SolverConfig(tolerance=TOL, max_iterations=MAXIT, l=8)),
                          ("tfqmr", Z.solve_tfqmr, Z.SolverConfig(tolerance=TOL, max_iterations=MAXIT))):
        for _ in range(2):
            x, rep = fn(A, bv, M, cfg)
        l0 = Z.launch_count()
        _lib.event_record(12)
        for _ in range(steps):
            x, rep = fn(A, bv, M, cfg)
        _lib.event_record(13)
        ms = _lib.event_elapsed_ms(12, 13) / steps
        out[name] = {"solves_per_s": round(1e3 / ms, 4), "ms_per_solve": round(ms, 2),
                     "iterations": rep.iterations, "converged": bool(rep.converged),
                     "final_rel": rep.final_relative_residual,
                     "kernels_per_solve": (Z.launch_count() - l0) // steps, "host_syncs_per_solve": 1}
    return out


# ---- C2: the paper's BLAS-1 study (BASELINE configs[1]) ----------------------------

C2_SIZES = (10_000, 100_000, 1_000_000, 10_000_000, 100_000_000)
C2_BYTES = {"zdotc": 32, "zaxpy": 48, "zscal": 32, "znrm2": 16}  # SURVEY 8d, per element


def blas1_sweep(peak: float, sizes=C2_SIZES):
    """zdotc / zaxpy / zscal / znrm2 at 1e4..1e8 complex128 elements through
    the public API (vecops.py:124-200), inputs from random_zvector (seed 42,
    reference bench.py:137-139).  Each timed launch is bracketed by CUDA
    events on the library stream with a 256 MB L2 flush before it, so small
    sizes measure HBM, not the 126 MB L2; the median of the reps is kept."""
    import paper_2112_06465_b200 as Z
    from paper_2112_06465_b200 import _lib
    flush = Z.ZVector._device_new(16 * 1024 * 1024)  # 256 MB > L2
    res = Z.ZVector._device_new(1)
    out = {}
    for n in sizes:
        rng = np.random.default_rng(42)
        x = Z.ZVector(rng.random(n) + 1j * rng.random(n))
        y = Z.ZVector(rng.random(n) + 1j * rng.random(n))
        alpha = complex(rng.random(), rng.random())
        x._dptr()
        y._dptr()
        L, ctx = _lib.lib(), _lib.context()
        # reductions with their result left in device memory (zk_zdotc_dev):
        # the timed interval holds the kernel, not the host round trip
        ops = {"zdotc": lambda: _lib.check(L.zk_zdotc_dev(ctx, n, x._dptr(), y._dptr(), 1, 4096, 0, res._dptr_out())),
               "zaxpy": lambda: Z.zaxpy(alpha, x, y),
               "zscal": lambda: Z.zscal(alpha, x),
               "znrm2": lambda: _lib.check(L.zk_znorm2_dev(ctx, n, x._dptr(), 4096, 0, res._dptr_out()))}
        reps = 20 if n <= 10_000_000 else 8
        for name, fn in ops.items():
            fn()
            times = []
            for _ in range(reps):
                _lib.check(_lib.lib().zk_memset(_lib.context(), flush._dptr_out(), 1, 16 * 16 * 1024 * 1024))
                _lib.event_record(10)
                fn()
                _lib.event_record(11)
                times.append(_lib.event_elapsed_ms(10, 11))
            ms = statistics.median(times)
            gbs = C2_BYTES[name] * n / (ms * 1e-3) / 1e9
            out[f"{name}_{n:.0e}".replace("+0", "")] = {"us": round(ms * 1e3, 2), "gbs": round(gbs, 1),
                                                          "frac": round(gbs / peak, 3)}
        del x, y
    return out


def cpu_sample(ia, ja, aa, b, minv, iters):
    """One capped solve of the reference algorithm (oracle/port.py): setup +
    one iteration; returns (solves/s extrapolated to `iters`, detail)."""
    from oracle import port
    t0 = time.perf_counter()
    x, hist, conv, t_setup, it_times = port.bicgstab(ia, ja, aa, b, minv, TOL, 1)
    wall = time.perf_counter() - t0
    t_iter = it_times[0]
    per_solve = t_setup + iters * t_iter
    return 1.0 / per_solve, {"setup_s": t_setup, "iteration_s": t_iter, "wall_s": wall, "hist": list(hist), "x": x}


def cpu_baseline(ia, ja, aa, b, minv, iters, config=CONFIG):
    from oracle import fingerprint
    v, d = cpu_sample(ia, ja, aa, b, minv, iters)
    facts = fingerprint.host_facts()
    return {"value": v, "unit": "solves/s", "cores": 1, "kind": "port",
            "sample": (f"reference BiCGStab algorithm (oracle/port.py, numpy, single-threaded like zlinalg) on {config}: "
                       f"setup {d['setup_s']:.2f}s + 1 iteration {d['iteration_s']:.2f}s, extrapolated to "
                       f"{iters} iterations"),
            "host": facts}, d


def run_reference(args, dist: Dist):
    if dist.rank != 0:
        return
    iters = args.iterations if args.iterations is not None else known_iterations(args.config)
    if iters is None:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.config} iteration count unknown; pass --iterations"}))
        return
    n, ia, ja, aa, b = build_problem(args.config)
    diag = np.zeros(n, dtype=np.complex128)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ia))
    hit = rows == ja
    diag[rows[hit]] = aa[hit]
    minv = np.divide(1.0, diag)  # build_jacobi (krylov.py:120)
    from oracle import port
    port.spmv(ia, ja, aa, b, n)  # warm-up (page-in)
    vals, details = [], []
    for _ in range(args.steps):
        v, d = cpu_sample(ia, ja, aa, b, minv, iters)
        vals.append(v)
        details.append(d)
    value = statistics.median(vals)
    sample = (f"reference BiCGStab algorithm (oracle/port.py, numpy) on {args.config}, per step: setup + 1 iteration "
              f"(median iteration {statistics.median(d['iteration_s'] for d in details):.2f}s), extrapolated to "
              f"{iters} iterations")
    out = {"metric": "bicgstab_solves_per_sec", "value": value, "unit": "solves/s", "n_gpus": dist.world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": statistics.median(d["wall_s"] for d in details) * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64 re/im pairs)", "data": "synthetic",
           "config": {"workload": WORKLOADS[args.config], "n": n, "nnz": int(ia[-1]), "iterations": iters},
           "detail": {"iterations_source": "tests/golden/headline_iterations.json (bitwise GPU == oracle)",
                      "parallelism": "1 host core (numpy ufuncs are single-threaded; the hot path calls no BLAS)"},
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "solves/s", "cores": 1, "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _launch_ranks(args) -> int:
    """``--gpus N`` without a torchrun environment: start N ranks on this
    node (torch.distributed.run, 127.0.0.1 rendezvous), one per GPU, and
    return their exit status; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["zk", "reference"], default="zk")
    ap.add_argument("--iterations", type=int, default=None, help="reference arm: override the committed iteration count")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C2 BLAS-1 sweep")
    ap.add_argument("--no-solvers", action="store_true", help="skip the BiCGSTAB(8) / TFQMR lines")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default=CONFIG, help="BASELINE system (default C4)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(_launch_ranks(args))
    dist = Dist() if args.impl == "zk" else _NoDist()
    if args.impl == "zk" and dist.world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={dist.world}")
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif dist.world > 1 or os.environ.get("ZK_BENCH_SHARDED") == "1":
            run_sharded(args, dist)
        else:
            run_zk(args, dist)
    finally:
        dist.close()


class _NoDist(Dist):
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))

    def close(self):
        pass


if __name__ == "__main__":
    main()
