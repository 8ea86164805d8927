/*
 * zk.h -- C ABI of libzk, the B200 (sm_100a) complex128 Krylov hot path.
 *
 * This is the drop-in boundary for the reference package `zlinalg`
 * (/root/reference/pkg/src/zlinalg).  The reference has no FFI of its own:
 * its hot path is the Python module API exported at `__init__.py:8-91`, and
 * each entry point below replaces one of those functions (cited per
 * function).  INTEGRATION.md shows the ctypes binding a maintainer would add
 * to `vecops.py`, `sparse.py` and `krylov.py`; paper_2112_06465_b200/ is that
 * binding, packaged.
 *
 * Conventions
 *  - Plain C types only.  Complex vectors are device pointers to interleaved
 *    little-endian binary64 (re, im) pairs, i.e. numpy complex128 / `<c16`
 *    (cnum.py:1-8, vecops.py:203-207).  Host pointers are marked `_host`.
 *  - Every function returns a zk_status.  Nothing throws across the ABI;
 *    zk_last_error() returns a thread-local message for the last failure.
 *    Status codes map 1:1 onto the reference's exception classes
 *    (errors.py:4-39).
 *  - Argument checks (lengths, indices, parameters) run before any device
 *    work is enqueued, so a failed call never writes an output
 *    (test_vecops.py:110-125: "raises before any write").
 *  - All work is ordered on the context's stream.  Calls returning host
 *    scalars (zdotc/znorm2/bicgstab) synchronise; the others are async.
 *  - Arithmetic reproduces the reference bit for bit: numpy's complex
 *    multiply formula, numpy's pairwise summation order inside each
 *    reduction block, the left fold over blocks and Python's scalar
 *    recurrences.  zk_set_arith() selects the host
 *    numpy fingerprint being reproduced.
 */
#ifndef ZK_H
#define ZK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int zk_status;
#define ZK_OK 0
#define ZK_ERR_DIMENSION 1   /* errors.DimensionError */
#define ZK_ERR_FORMAT 2      /* errors.FormatError */
#define ZK_ERR_PARAMETER 3   /* errors.ParameterError */
#define ZK_ERR_SINGULAR 4    /* errors.SingularPreconditionerError */
#define ZK_ERR_BREAKDOWN 5   /* errors.BreakdownError (report still filled) */
#define ZK_ERR_CUDA 6        /* device / driver failure */
#define ZK_ERR_NOMEM 7       /* device allocation failed */
#define ZK_ERR_NODEVICE 8    /* no CUDA device: there is no CPU fallback */

#define ZK_MODE_BLOCKED 0    /* vecops.BLOCKED */
#define ZK_MODE_SEQUENTIAL 1 /* vecops.SEQUENTIAL */

typedef struct zk_context zk_context;
typedef struct zk_csr zk_csr;

/* ---- context, memory ---------------------------------------------------- */
const char* zk_last_error(void);
const char* zk_version(void);
zk_status zk_context_create(int device, zk_context** out);
zk_status zk_context_destroy(zk_context* ctx);
/* Fingerprint of the numpy being reproduced: use_fma=1 is the AVX512F/FMA3
 * complex multiply (fma(a.re,b.re,-(a.im*b.im)), fma(a.re,b.im,a.im*b.re)),
 * 0 the plain one; elide_bytes is numpy's temporary-elision threshold
 * (NPY_MIN_ELIDE_BYTES, 256 KiB) that swaps SpMV's product operands. */
zk_status zk_set_arith(zk_context* ctx, int use_fma, int64_t elide_bytes);
zk_status zk_malloc(zk_context* ctx, size_t bytes, void** dptr);
zk_status zk_free(zk_context* ctx, void* dptr);
zk_status zk_host_alloc(size_t bytes, void** hptr);   /* pinned */
zk_status zk_host_free(void* hptr);
zk_status zk_memcpy_h2d(zk_context* ctx, void* dst, const void* src_host, size_t bytes);
zk_status zk_memcpy_d2h(zk_context* ctx, void* dst_host, const void* src, size_t bytes);
zk_status zk_memcpy_d2d(zk_context* ctx, void* dst, const void* src, size_t bytes);
zk_status zk_memset(zk_context* ctx, void* dst, int value, size_t bytes);
zk_status zk_synchronize(zk_context* ctx);
/* Kernels launched by this context so far (graph nodes included). */
zk_status zk_launch_count(zk_context* ctx, int64_t* count);
/* Launch stream as an opaque handle (cudaStream_t) for event timing. */
zk_status zk_stream(zk_context* ctx, void** stream);

/* Pin / unpin caller-owned host memory (cudaHostRegister) so uploads run at
 * full PCIe rate. */
zk_status zk_host_register(void* hptr, size_t bytes);
zk_status zk_host_unregister(void* hptr);
/* CUDA events on the context stream, slots 0..31 (device-side timing). */
zk_status zk_event_record(zk_context* ctx, int slot);
zk_status zk_event_elapsed(zk_context* ctx, int start_slot, int stop_slot, double* ms);

/* Solver phase profiling.  While enabled, zk_bicgstab drives the loop from
 * the host and brackets every phase kernel with CUDA events; zk_profile_read
 * returns the accumulated device time and launch count per phase, in this
 * order: setup, p_first, pivot_first, pivot_first_dot, s_update, x_alpha,
 * true_res_s, spmv_t, tt_ts, xr_update, true_res (A x), res_pass, p_next,
 * spmv_pivot, pivot_dot, spmv2 (matrices at most 8 entries wide: A x and A p^
 * in one pass, replacing true_res and spmv_pivot). */
#define ZK_NPHASES 16
zk_status zk_profile_enable(zk_context* ctx, int on);
zk_status zk_profile_read(zk_context* ctx, double* total_ms, int64_t* launches);

/* ---- level-1 kernels (vecops.py) ---------------------------------------- */
/* zscal: x <- F1(x, alpha)                      replaces vecops.zscal  (vecops.py:124-127) */
zk_status zk_zscal(zk_context* ctx, int64_t n, double alpha_re, double alpha_im, double* x);
/* zaxpy: y <- y + F1(alpha, x)                  replaces vecops.zaxpy  (vecops.py:130-134) */
zk_status zk_zaxpy(zk_context* ctx, int64_t n, double alpha_re, double alpha_im,
                   const double* x, double* y);
/* zaxmy: y <- F1(y, x)                          replaces vecops.zaxmy  (vecops.py:137-141) */
zk_status zk_zaxmy(zk_context* ctx, int64_t n, const double* x, double* y);
/* zassign: dst <- src                           replaces vecops.zassign (vecops.py:117-121) */
zk_status zk_zassign(zk_context* ctx, int64_t n, double* dst, const double* src);
/* out <- F1(v, minv)                   replaces Preconditioner.apply (krylov.py:92-100) */
zk_status zk_jacobi_apply(zk_context* ctx, int64_t n, const double* v, const double* minv, double* out);
/* sum cbar(x)*y, cbar = conj when conjugate; block_size in [64, 65536] (power of
 * two) with mode BLOCKED, or mode SEQUENTIAL.  result_host = (re, im).
 *                                                replaces vecops.zdot (vecops.py:165-186) */
zk_status zk_zdotc(zk_context* ctx, int64_t n, const double* x, const double* y, int conjugate,
                   int64_t block_size, int mode, double* result_host);
/*                                                replaces vecops.znorm2 (vecops.py:189-200) */
zk_status zk_znorm2(zk_context* ctx, int64_t n, const double* x, int64_t block_size, int mode,
                    double* result_host);

/* Same reductions, asynchronous: the result lands in device memory
 * (result_dev: 2 doubles for zdotc, 1 for znorm2), stream-ordered, no host
 * wait -- for device-resident pipelines (and kernel-only timing). */
zk_status zk_zdotc_dev(zk_context* ctx, int64_t n, const double* x, const double* y, int conjugate,
                       int64_t block_size, int mode, double* result_dev);
zk_status zk_znorm2_dev(zk_context* ctx, int64_t n, const double* x, int64_t block_size, int mode,
                        double* result_dev);

/* ---- CSR matrix and SpMV (sparse.py) ------------------------------------ */
/* Upload a validated CSR (zero-based int64 ia[n_rows+1], ja[nnz]; complex128
 * aa[nnz]; strictly increasing columns per row -- CsrMatrix._validate,
 * sparse.py:79-103) into the device SELL-32 layout.  Host pointers.
 *                                   device twin of CsrMatrix (sparse.py:60-158) */
zk_status zk_csr_create(zk_context* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                        const int64_t* ia_host, const int64_t* ja_host, const double* aa_host,
                        zk_csr** out);
/* Same, from device-resident CSR arrays (ia/ja int64, aa complex128). */
zk_status zk_csr_create_device(zk_context* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                               const int64_t* ia, const int64_t* ja, const double* aa,
                               zk_csr** out);
zk_status zk_csr_destroy(zk_csr* A);
/* Device bytes held by the matrix (SELL arrays incl. padding). */
zk_status zk_csr_bytes(const zk_csr* A, int64_t* bytes, int64_t* padded_elems);
/* y <- A x (x: n_cols, y: n_rows)               replaces sparse.spmv (sparse.py:217-232) */
zk_status zk_spmv(zk_context* ctx, const zk_csr* A, const double* x, double* y);
/* y <- A x and result = sum cbar(w)*y in ONE pass over A (the SpMV's rows feed
 * the DEFAULT_PLAN block reduction as they are produced): bitwise
 * sparse.spmv(A, x) followed by vecops.zdot(w, y, conjugate) (vecops.py:165-186),
 * the fusion the BiCGStab loop uses for its shadow pivot (krylov.py:267-268). */
zk_status zk_spmv_dotc(zk_context* ctx, const zk_csr* A, const double* x, double* y, const double* w,
                       int conjugate, double* result_host);

/* Jacobi preconditioner on the device: minv[i] = 1 / A[i][i] for
 * i < min(n_rows, n_cols), numpy's complex division bit for bit.  A missing
 * or zero diagonal entry returns ZK_ERR_SINGULAR with *zero_row = the first
 * such row (else -1).          replaces krylov.build_jacobi (krylov.py:106-120) */
zk_status zk_jacobi_build(zk_context* ctx, const zk_csr* A, double* minv, int64_t* zero_row);

/* ---- BiCGStab (krylov.py) ----------------------------------------------- */
typedef struct {
    int64_t iterations;          /* SolveReport.iterations */
    int32_t converged;           /* SolveReport.converged */
    int32_t breakdown;           /* 0 none, 1 rho, 2 omega, 3 shadow pivot, 4 <t,t> */
    double final_relative_residual;
    int64_t history_len;         /* iterations + 1 (entries written to history_host) */
    int64_t kernel_launches;     /* kernels launched by this solve */
} zk_solve_report;

/* Right-preconditioned BiCGStab, device-resident: x, r, r~, p, v, s, t, p^,
 * s^ never leave HBM and the host waits once, for the final report.
 * b: device rhs; minv: device inverse diagonal (Jacobi) or NULL (identity);
 * x0: device initial guess or NULL (zero); x_out: device solution (n).
 * history_host: >= max_iterations + 1 doubles.
 * Returns ZK_OK (converged or not: non-convergence is data, krylov.py:295)
 * or ZK_ERR_BREAKDOWN with the report filled up to the breakdown.
 *                              replaces krylov.solve_bicgstab (krylov.py:213-295) */
zk_status zk_bicgstab(zk_context* ctx, const zk_csr* A, const double* b, const double* minv,
                      const double* x0, double tolerance, int64_t max_iterations, double* x_out,
                      double* history_host, zk_solve_report* report);

/* ---- BiCGSTAB(l) and TFQMR (krylov.py:298-489) ------------------------------
 * Device-resident like zk_bicgstab: one CUDA-graph launch per solve (a
 * conditional WHILE over one outer cycle of BiCGSTAB(l), resp. two TFQMR
 * iterations), scalars and control flow on the device, one host wait.
 * report->breakdown holds a ZK_BD_* code; for ZK_BD_MR *breakdown_index is
 * the basis vector j of "minimal-residual basis vector {j}". */
#define ZK_BD_RHO 1      /* "rho" */
#define ZK_BD_OMEGA 2    /* "omega" */
#define ZK_BD_PIVOT 3    /* "shadow pivot" */
#define ZK_BD_MR 5       /* "minimal-residual basis vector {j}" */
#define ZK_BD_SIGMA 6    /* "sigma = <r~, v>" */
#define ZK_BD_ALPHA 7    /* "alpha" */
#define ZK_BD_TAU 8      /* "quasi-residual tau" */
/*                          replaces krylov.solve_bicgstab_l (krylov.py:298-410); 1 <= ell <= 32 */
zk_status zk_bicgstab_l(zk_context* ctx, const zk_csr* A, const double* b, const double* minv,
                        const double* x0, double tolerance, int64_t max_iterations, int ell, double* x_out,
                        double* history_host, zk_solve_report* report, int32_t* breakdown_index);
/*                          replaces krylov.solve_tfqmr (krylov.py:413-489) */
zk_status zk_tfqmr(zk_context* ctx, const zk_csr* A, const double* b, const double* minv, const double* x0,
                   double tolerance, int64_t max_iterations, double* x_out, double* history_host,
                   zk_solve_report* report);

/* ---- row-sharded BiCGStab (multi-GPU) --------------------------
 * One shard per rank (process / GPU).  The reference has no distributed
 * solver: a shard runs exactly the loop of krylov.solve_bicgstab
 * (krylov.py:213-295) on its rows and the ranks combine every reduction in
 * the unsharded block order, so all ranks -- and the 1-GPU solve and the
 * reference -- produce the same bits.  The library does the device work;
 * the caller's transport (NCCL or host staging, paper_2112_06465_b200/dist.py)
 * moves halos and block partials between the phases:
 *   - A_local: rows [row0, row0 + n) of the matrix, row0 a multiple of 4096
 *     (the reduction block), columns renumbered own rows first ([0, n)) and
 *     the n_halo external columns after, in ascending global order;
 *   - before SETUP / TRUE_RES_S / TRUE_RES the halo of ZK_DVEC_X, before
 *     PIVOT that of ZK_DVEC_PHAT, before SPMV_T that of ZK_DVEC_SHAT must be
 *     current (zk_dshard_pack gathers the entries a peer needs);
 *   - after a phase with a reduction, each rank's ZK_DVEC_PARTIALS is
 *     all-gathered into ZK_DVEC_GATHERED (rank r at r * len(PARTIALS)) and
 *     zk_dshard_finish folds it.  PARTIALS holds two slots of
 *     4 * max_blocks doubles: SPMV_T and TRUE_RES write slot 1, every other
 *     phase slot 0, so TRUE_RES_S + SPMV_T and XR_UPDATE + TRUE_RES can
 *     share one all-gather (finish them in that order).
 * Phases whose work depends on the s-check (X_ALPHA, TRUE_RES_S) are no-ops
 * on the device when it did not fire, so every rank issues the same calls. */
typedef struct zk_dshard zk_dshard;
#define ZK_DVEC_X 0
#define ZK_DVEC_PHAT 1
#define ZK_DVEC_SHAT 2
#define ZK_DVEC_B 3
#define ZK_DVEC_MINV 4
#define ZK_DVEC_PARTIALS 5
#define ZK_DVEC_GATHERED 6
#define ZK_DPHASE_SETUP 0       /* r0 = b - A x0, ||b||, ||r0||, <r0,r0>  (krylov.py:159-168) */
#define ZK_DPHASE_P_FIRST 1     /* p = r (first iteration)                  (krylov.py:263-266) */
#define ZK_DPHASE_PIVOT 2       /* v = A p^, <r~,v> -> alpha                (krylov.py:267-271) */
#define ZK_DPHASE_S_UPDATE 3    /* s, s^, ||s|| -> s-check                  (krylov.py:272-275) */
#define ZK_DPHASE_X_ALPHA 4     /* x += alpha p^ (s-check path)             (krylov.py:274) */
#define ZK_DPHASE_TRUE_RES_S 5  /* ||b - A x|| on the s-check path          (krylov.py:276-279) */
#define ZK_DPHASE_SPMV_T 6      /* t = A s^, <t,t>, <t,s> -> omega           (krylov.py:281-287) */
#define ZK_DPHASE_XR_UPDATE 7   /* x, r updates, <r~,r> -> rho, beta         (krylov.py:288-290, 255-261) */
#define ZK_DPHASE_TRUE_RES 8    /* ||b - A x|| -> record / stop              (krylov.py:291-294) */
#define ZK_DPHASE_P_NEXT 9      /* p, p^ for the next iteration             (krylov.py:263-266) */
zk_status zk_dshard_create(zk_context* ctx, zk_csr* A_local, int64_t n_halo, int64_t nnz_global, int jacobi,
                           int64_t max_iterations, int nranks, int64_t max_blocks, zk_dshard** out);
zk_status zk_dshard_destroy(zk_dshard* shard);
/* Device pointer + length (complex entries; doubles for PARTIALS/GATHERED). */
zk_status zk_dshard_vector(zk_dshard* shard, int which, double** dptr, int64_t* length);
/* Start a solve (b, minv, and x0 when has_x0 already copied into the shard's vectors). */
zk_status zk_dshard_reset(zk_dshard* shard, double tolerance, int64_t max_iterations, int has_x0);
zk_status zk_dshard_phase(zk_dshard* shard, int phase);
/* rank_blocks_host[r]: reduction blocks of rank r (its partials count). */
zk_status zk_dshard_finish(zk_dshard* shard, int phase, const int64_t* rank_blocks_host);
/* out[i] = vec[idx[i]] (device arrays): the entries a peer's halo needs. */
zk_status zk_dshard_pack(zk_dshard* shard, int which, const int64_t* idx, int64_t count, double* out);
/* Synchronises; done = 1 stopped (converged / cap / breakdown), 2 zero rhs. */
zk_status zk_dshard_status(zk_dshard* shard, zk_solve_report* report, int32_t* done);
zk_status zk_dshard_history(zk_dshard* shard, double* history_host, int64_t count);

#ifdef __cplusplus
}
#endif
#endif /* ZK_H */
