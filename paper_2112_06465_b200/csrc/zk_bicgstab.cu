// zk_bicgstab.cu -- device-resident right-preconditioned BiCGStab
// (krylov.py:213-295, _Run krylov.py:139-206), bitwise faithful.
//
// One iteration of the reference (op order in SURVEY 3.2) is fused into five
// grid-wide phases, every vector pass doing all the elementwise work and the
// reduction that follows it:
//
//   K2  v = A p^            + block partials of <r~, v>    -> fold: pivot, alpha
//   K3  s = r - alpha v, s^ = M s, |s|^2 partials           -> fold: s-check
//  [K3x x += alpha p^ ; K6x ||b - A x||  -- only when the s-check fires]
//   K4  t = A s^            + <t,t>, <t,s> partials         -> fold: omega
//   K5  x = (x + alpha p^) + omega s^, r = s - omega t,
//       <r~, r> partials                                    -> fold: rho', beta
//   K61 ||b - A x|| partials (true residual, _Run.true_relative_residual)
//       fused with next iteration's p = ((p - omega v) * beta) + r, p^ = M p
//                                                           -> fold: record, stop?
//
// SpMV phases are persistent TMA-pipelined kernels (zk_spmv.cuh); the
// reduction of each 4096-row block runs on the consumer warps as soon as the
// block's rows are done, while the producer warp keeps streaming the matrix.
// The level-1 phases K3 and K5 run on the TMA-fed block-reduction engine
// (zk_l1pipe.cuh): their input vectors stream into shared memory stage by
// stage (one pairwise subtree per stage) and consumer warps apply the fused
// updates and the numpy-order sums from there.
// The CTA that finishes the last block folds the block partials in order
// and runs the scalar recurrences (Python Cplx arithmetic, zk_common.cuh) on
// a device SolverState.  The loop is a CUDA-graph conditional WHILE node
// whose condition K61 sets, so a solve is one graph launch and the host
// synchronises once.
#include <cstdlib>
#include <cstring>

#include "zk_internal.h"
#include "zk_blockred.cuh"
#include "zk_l1pipe.cuh"
#include "zk_spmv.cuh"

namespace zk {

SellView sell_view(const zk_csr* A, const zk_context* c, size_t extra, int nsv);
size_t pipe_smem_bytes(const SellView& v, size_t extra);
unsigned pipe_grid(const zk_csr* A);
unsigned plain_grid(const zk_csr* A, SellView& v);

enum : int32_t { ST_RUNNING = 0, ST_CONVERGED = 1, ST_NOT_CONVERGED = 2, ST_BREAKDOWN = 3 };
enum : int32_t { BD_NONE = 0, BD_RHO = 1, BD_OMEGA = 2, BD_PIVOT = 3, BD_TT = 4 };

struct SolverState {
    double2 rho, rho_old, alpha, omega, beta;
    double b_norm, tol, last_rel;
    int64_t maxit, iterations, trips;
    int32_t done, status, what, scheck, alpha_applied, trivial_zero;
    unsigned int counter;
    int32_t pad;
};

struct SolverBufs {
    double2 *x, *b, *minv, *r, *rs, *p, *v, *s, *t, *ph, *sh;
    double* partials;  // nblocks * 4 doubles
    double* slots;     // nblocks * 4 doubles at kSlotEmpty between passes (1-GPU streaming fold)
    double* hist;      // hist_cap doubles
    SolverState* st;
    int64_t n, nblocks;
    bool jacobi, fma;
    int dist;          // row-sharded solve: block partials are folded across ranks (k_fold_finish)
    int64_t pslot;     // row-sharded: doubles per partials slot (4 x max blocks of any rank); slot 1 at +pslot
};


struct SolverPlan {
    int64_t n = 0;
    bool jacobi = false;
    int64_t hist_cap = 0;
    SolverBufs bufs{};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool graph_ok = false;
    // arithmetic the graph's kernel parameters were captured with: the FMA
    // fingerprint and numpy's elision swap (SellView::swap, which depends on
    // zk_context::elide_bytes); a change of either rebuilds the graph
    bool graph_fma = true, graph_swap = false;
};

namespace {


__device__ __forceinline__ double2 neg(double2 a) { return make_double2(-a.x, -a.y); }

__device__ __forceinline__ void stop(SolverState* st, int32_t status, int32_t what) {
    st->status = status;
    st->what = what;
    st->done = 1;
}

// ---- SpMV-phase bodies (zk_spmv.cuh reducer pipeline) ----------------------
// Each body stores its row outputs and returns the row's reduction terms;
// finish() receives the in-order folded totals [complex re/im pairs..., reals...]
// in lane 0 of the reducer warp of the CTA that retired the last block.

// ---- setup: r0 = b - A x0, ||b||, ||r0||, <r0, r0> (krylov.py:159-168, 255) ----
struct SetupBody {
    static constexpr int kNC = 1, kNR = 2, kSV = 1;  // staged: b
    static constexpr int kNP = 2 * kNC + kNR;
    SolverBufs B;
    __device__ void row(int64_t row, const double2 (&ax)[1], const double2 (&sv)[1], double2 (&tc)[1], double (&tr)[2]) {
        const double2 b = sv[0];
        const double2 r0 = cadd(b, f1(make_double2(-1.0, 0.0), ax[0], B.fma));
        B.r[row] = r0;
        B.rs[row] = r0;
        tc[0] = f1(conjz(r0), r0, B.fma);
        tr[0] = abs2_np(b);
        tr[1] = abs2_np(r0);
    }
    __device__ void finish(const double* t) {  // [<r0,r0>.re, .im, |b|^2, |r0|^2]
        SolverState* st = B.st;
        st->counter = 0;
        const double bn = __dsqrt_rn(t[2]), rn = __dsqrt_rn(t[3]);
        const double2 tc = make_double2(t[0], t[1]);
        st->b_norm = bn;
        const double h0 = bn > 0.0 ? __ddiv_rn(rn, bn) : 0.0;
        B.hist[0] = h0;
        st->last_rel = h0;
        if (bn == 0.0) {  // trivial_result: zero rhs -> x = 0, history [0.0]
            B.hist[0] = 0.0;
            st->last_rel = 0.0;
            st->trivial_zero = 1;
            stop(st, ST_CONVERGED, BD_NONE);
            return;
        }
        if (h0 <= st->tol) {  // the initial guess already solves
            stop(st, ST_CONVERGED, BD_NONE);
            return;
        }
        // iteration 1: rho = alpha = omega = 1, no breakdown possible
        const double2 one = make_double2(1.0, 0.0);
        st->rho_old = one;
        st->alpha = one;
        st->omega = one;
        st->beta = cmul_py(cdiv_py(tc, one), cdiv_py(one, one));
        st->rho = tc;
    }
};

__global__ void __launch_bounds__(kRedPipeThreads, 1) k_setup(SellView A, SolverBufs B, RedCfg R) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (B.st->done) return;
    SetupBody body{B};
    sell_run<1>(A, B.x, nullptr, body, R, smem);
}

// ---- K1: p update for the first iteration (p = v = 0) ----
// p = ((p + F1(-w, v)) * beta) + F1(1, r); p^ = F1(p, minv)
// (krylov.py:263-266: zaxpy, zscal, zaxpy, M.apply -- separate roundings).
__device__ __forceinline__ void p_update(const SolverBufs& B, double2 mw, double2 beta, int64_t i, double2 p,
                                         double2 v, double2 r, double2 m) {
    const bool fma = B.fma;
    p = cadd(p, f1(mw, v, fma));
    p = f1(p, beta, fma);
    p = cadd(p, f1(make_double2(1.0, 0.0), r, fma));
    B.p[i] = p;
    if (B.jacobi) B.ph[i] = f1(p, m, fma);
}

__global__ void __launch_bounds__(256) k_p_first(SolverBufs B) {
    const SolverState* st = B.st;
    if (st->done) return;
    const double2 mw = neg(st->omega), beta = st->beta;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B.n; i += stride)
        p_update(B, mw, beta, i, B.p[i], B.v[i], B.r[i], B.jacobi ? B.minv[i] : make_double2(0.0, 0.0));
}

// ---- Kp: next iteration's p update (after K5 has formed r and beta) ----
__global__ void __launch_bounds__(256) k_p_next(SolverBufs B) {
    const SolverState* st = B.st;
    if (st->done) return;
    const double2 mw = neg(st->omega), beta = st->beta;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B.n; i += stride)
        p_update(B, mw, beta, i, B.p[i], B.v[i], B.r[i], B.jacobi ? __ldg(B.minv + i) : make_double2(0.0, 0.0));
}

// pivot = <r~, v> -> alpha (krylov.py:268-271); false when the loop stopped
__device__ __forceinline__ void pivot_to_alpha(SolverState* st, double2 pivot) {
    if (small_py(pivot)) {
        stop(st, ST_BREAKDOWN, BD_PIVOT);
        return;
    }
    st->alpha = cdiv_py(st->rho, pivot);
}

// ---- K2 / K4 SpMV: v = A p^, t = A s^ (plain pipeline, all 7 consumer warps) ----
// The reductions that follow them (<r~, v>; <t, t> and <t, s>) run as a
// separate pass on the level-1 engine: the vector was just written and is
// half L2-resident, and the pass costs ~45 us at C4 against the ~150-200 us
// a reducer warp inside the SpMV cost (profiles/r02: 858 -> 2 kernels).
struct PhaseSpmvBody {
    static constexpr int kNC = 0, kNR = 0, kSV = 0;
    double2* __restrict__ y;
    __device__ __forceinline__ void row(int64_t r, const double2 (&v)[1], const double2 (&)[1], double2 (&)[1],
                                        double (&)[1]) {
        y[r] = v[0];
    }
    __device__ __forceinline__ void finish(const double*) {}
};

__global__ void __launch_bounds__(kPipeThreads, 1) k_spmv_phase(SellView A, const double2* __restrict__ x,
                                                                double2* __restrict__ y, const SolverState* st) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (st->done) return;
    PhaseSpmvBody body{y};
    const RedCfg R{};
    sell_run<1>(A, x, nullptr, body, R, smem);
}

template <int WM>
__global__ void __launch_bounds__(32 * NarrowCfg<WM>::warps(1), NarrowCfg<WM>::kMinB)
    k_spmv_phase_narrow(SellView A, const double2* __restrict__ x, double2* __restrict__ y, const SolverState* st) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (st->done) return;
    PhaseSpmvBody body{y};
    narrow_tma_run<WM, 1>(A, x, x, body, smem);
}

// Narrow matrices: K61's A x and K2's A p^ in one pass over the matrix
// (t = A x, v = A p^); the loop body runs Kp before it (launch_body).
struct PhaseSpmv2Body {
    static constexpr int kNC = 0, kNR = 0, kSV = 0;
    double2* __restrict__ y0;
    double2* __restrict__ y1;
    __device__ __forceinline__ void row(int64_t r, const double2 (&v)[2], const double2 (&)[1], double2 (&)[1],
                                        double (&)[1]) {
        y0[r] = v[0];
        y1[r] = v[1];
    }
};

template <int WM>
__global__ void __launch_bounds__(32 * NarrowCfg<WM>::warps(2), NarrowCfg<WM>::kMinB2)
    k_spmv2_phase_narrow(SellView A, const double2* __restrict__ x0, const double2* __restrict__ x1,
                         double2* __restrict__ y0, double2* __restrict__ y1, const SolverState* st) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (st->done) return;
    PhaseSpmv2Body body{y0, y1};
    narrow_tma_run<WM, 2>(A, x0, x1, body, smem);
}

// Wide matrices (experiment, ZK_FUSE2=2): the same two products through the ring.
__global__ void __launch_bounds__(kPipeThreads, 1) k_spmv2_phase(SellView A, const double2* __restrict__ x0,
                                                                 const double2* __restrict__ x1,
                                                                 double2* __restrict__ y0, double2* __restrict__ y1,
                                                                 const SolverState* st) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (st->done) return;
    PhaseSpmv2Body body{y0, y1};
    const RedCfg R{};
    sell_run<2>(A, x0, x1, body, R, smem);
}

// ---- K2 pass: <r~, v> -> pivot, alpha (krylov.py:268-271) ----
// Last kernel of the loop body: sets the graph's WHILE condition (the
// prologue instance, use_cond = 0, runs the first iteration's K2).
struct PivotOp {
    using V = double2;
    static constexpr int NIN = 2;  // r~, v
    bool fma;
    __device__ __forceinline__ double2 apply(int64_t, const double2 (&v)[2]) const {
        return f1(conjz(v[0]), v[1], fma);
    }
};

struct PivotFin {
    static constexpr int kNP = 2;
    SolverBufs B;
    cudaGraphConditionalHandle cond;
    int use_cond;
    __device__ void finish(const double* t) {
        SolverState* st = B.st;
        pivot_to_alpha(st, make_double2(t[0], t[1]));
        if (use_cond) cudaGraphSetConditional(cond, st->done ? 0u : 1u);
    }
};

__global__ void __launch_bounds__(kL1Threads, 1) k_pivot_pass(SolverBufs B, L1View P, cudaGraphConditionalHandle cond,
                                                              int use_cond) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (B.st->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
        return;
    }
    PivotOp op{B.fma};
    PivotFin fin{B, cond, use_cond};
    l1_pipeline(P, op, fin, smem);
}

// ---- K4 pass: <t, t>, <t, s> -> omega (krylov.py:282-287) ----
struct TOp {
    using V = cplx2;
    static constexpr int NIN = 2;  // t, s
    bool fma;
    __device__ __forceinline__ cplx2 apply(int64_t, const double2 (&v)[2]) const {
        const double2 ct = conjz(v[0]);
        return {f1(ct, v[0], fma), f1(ct, v[1], fma)};
    }
};

struct TFin {
    static constexpr int kNP = 4;
    SolverBufs B;
    __device__ void finish(const double* t) {
        SolverState* st = B.st;
        const double2 tt = make_double2(t[0], t[1]), ts = make_double2(t[2], t[3]);
        if (small_py(tt)) {
            stop(st, ST_BREAKDOWN, BD_TT);
            return;
        }
        const double2 w = cdiv_py(ts, tt);
        st->omega = w;
        if (small_py(w)) stop(st, ST_BREAKDOWN, BD_OMEGA);
    }
};

__global__ void __launch_bounds__(kL1Threads, 1) k_tt_ts_pass(SolverBufs B, L1View P) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (B.st->done) return;
    TOp op{B.fma};
    TFin fin{B};
    l1_pipeline(P, op, fin, smem);
}

// ---- true residual ||b + F1(-1, A x)|| / ||b|| (krylov.py:183-186) ----
// MODE 0: on the s-check path (K6x, krylov.py:275-279);  MODE 1: end of
// iteration (K61, krylov.py:288-294), which also runs the next iteration's
// rho/omega breakdown checks (krylov.py:256-259).
template <int MODE>
struct ResBody {
    static constexpr int kNC = 0, kNR = 1, kSV = 1;  // staged: b
    static constexpr int kNP = 2 * kNC + kNR;
    SolverBufs B;
    __device__ void row(int64_t, const double2 (&ax)[1], const double2 (&sv)[1], double2 (&)[1], double (&tr)[1]) {
        tr[0] = abs2_np(cadd(sv[0], f1(make_double2(-1.0, 0.0), ax[0], B.fma)));
    }
    __device__ void finish(const double* t) {
        SolverState* st = B.st;
        st->counter = 0;
        const double rel = __ddiv_rn(__dsqrt_rn(t[0]), st->b_norm);
        if (MODE == 0) {
            if (rel <= st->tol) {
                st->iterations++;
                B.hist[st->iterations] = rel;
                st->last_rel = rel;
                stop(st, ST_CONVERGED, BD_NONE);
            }
            return;
        }
        st->iterations++;
        B.hist[st->iterations] = rel;
        st->last_rel = rel;
        st->scheck = 0;
        st->alpha_applied = 0;
        if (rel <= st->tol) {
            stop(st, ST_CONVERGED, BD_NONE);
        } else if (st->iterations >= st->maxit) {
            stop(st, ST_NOT_CONVERGED, BD_NONE);
        } else if (small_py(st->rho_old)) {
            stop(st, ST_BREAKDOWN, BD_RHO);
        } else if (small_py(st->omega)) {
            stop(st, ST_BREAKDOWN, BD_OMEGA);
        }
    }
};

template <int MODE>
__global__ void __launch_bounds__(kRedPipeThreads, 1) k_true_res(SellView A, SolverBufs B, RedCfg R) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (B.st->done || (MODE == 0 && !B.st->scheck)) return;
    ResBody<MODE> body{B};
    sell_run<1>(A, B.x, nullptr, body, R, smem);
}

// true residual pass: ||b + F1(-1, A x)||^2 over (b, A x) -> record / stop
struct ResOp {
    using V = double;
    static constexpr int NIN = 2;  // b, A x
    bool fma;
    __device__ __forceinline__ double apply(int64_t, const double2 (&v)[2]) const {
        return abs2_np(cadd(v[0], f1(make_double2(-1.0, 0.0), v[1], fma)));
    }
};

__global__ void __launch_bounds__(kL1Threads, 1) k_res_pass(SolverBufs B, L1View P) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (B.st->done) return;
    ResOp op{B.fma};
    ResBody<1> fin{B};
    l1_pipeline(P, op, fin, smem);
}

__global__ void k_fill_empty(double* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = __longlong_as_double((long long)kSlotEmpty);
}

// ---- K3: s = r + F1(-alpha, v); s^ = M s; ||s|| -> s-check (krylov.py:272-275) ----
// s-check decision from the folded ||s||^2 (krylov.py:275)
struct SUpdFinish {
    static constexpr int kNP = 1;
    SolverBufs B;
    __device__ void finish(const double* t) {
        SolverState* st = B.st;
        st->counter = 0;
        st->scheck = (__ddiv_rn(__dsqrt_rn(t[0]), st->b_norm) <= st->tol) ? 1 : 0;
    }
};

// K3 on the TMA-fed engine (zk_l1pipe.cuh): staged r, v, minv
struct SUpdPipeOp {
    using V = double;
    static constexpr int NIN = 3;
    double2* s;
    double2* sh;
    double2 ma;
    bool jacobi, fma;
    __device__ __forceinline__ double apply(int64_t e, const double2 (&v)[3]) const {
        const double2 sv = cadd(v[0], f1(ma, v[1], fma));
        s[e] = sv;
        if (jacobi) sh[e] = f1(sv, v[2], fma);
        return abs2_np(sv);
    }
};

__global__ void __launch_bounds__(kL1Threads, 1) k_s_update_pipe(SolverBufs B, L1View P) {
    extern __shared__ __align__(128) unsigned char smem[];
    SolverState* st = B.st;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->trips++;  // loop-body executions (launch accounting)
    if (st->done) return;
    SUpdPipeOp op{B.s, B.sh, neg(st->alpha), B.jacobi, B.fma};
    SUpdFinish fin{B};
    l1_pipeline(P, op, fin, smem);
}

// ---- K3x: x = x + F1(alpha, p^), only on the s-check path (krylov.py:274) ----
__global__ void __launch_bounds__(256) k_x_alpha(SolverBufs B) {
    SolverState* st = B.st;
    if (st->done || !st->scheck) return;
    const double2 a = st->alpha;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B.n; i += stride)
        B.x[i] = cadd(B.x[i], f1(a, B.ph[i], B.fma));
    if (blockIdx.x == 0 && threadIdx.x == 0) st->alpha_applied = 1;
}

// ---- K5: x, r updates and <r~, r> -> rho', beta (krylov.py:288-290, 255-261) ----
// rho' = <r~, r> -> rho, beta of the next iteration (krylov.py:255-261)
struct XrFinish {
    static constexpr int kNP = 2;
    SolverBufs B;
    __device__ void finish(const double* t) {
        SolverState* st = B.st;
        st->counter = 0;
        const double2 rho_next = make_double2(t[0], t[1]);
        const double2 rho = st->rho, a = st->alpha, w = st->omega;
        st->rho_old = rho;
        st->rho = rho_next;
        // beta for the next iteration (speculative: K61 stops before it is
        // used if the loop ends, and breaks down on krylov.py:256-259's checks)
        if (!small_py(rho) && !small_py(w)) st->beta = cmul_py(cdiv_py(rho_next, rho), cdiv_py(a, w));
    }
};

// K5 on the TMA-fed engine: staged x, p^, s^, s, t, r~ (p^ is staged even when
// the s-check path already applied alpha p^: that path runs at most once)
struct XrPipeOp {
    using V = double2;
    static constexpr int NIN = 6;
    double2* x;
    double2* r;
    double2 a, w, mw;
    bool applied, fma;
    __device__ __forceinline__ double2 apply(int64_t e, const double2 (&v)[6]) const {
        double2 xv = v[0];
        if (!applied) xv = cadd(xv, f1(a, v[1], fma));
        xv = cadd(xv, f1(w, v[2], fma));
        x[e] = xv;
        const double2 rv = cadd(v[3], f1(mw, v[4], fma));
        r[e] = rv;
        return f1(conjz(v[5]), rv, fma);
    }
};

__global__ void __launch_bounds__(kL1Threads, 1) k_xr_update_pipe(SolverBufs B, L1View P) {
    extern __shared__ __align__(128) unsigned char smem[];
    SolverState* st = B.st;
    if (st->done) return;
    const double2 a = st->alpha, w = st->omega;
    XrPipeOp op{B.x, B.r, a, w, neg(w), st->alpha_applied != 0, B.fma};
    XrFinish fin{B};
    l1_pipeline(P, op, fin, smem);
}

// ---- ordered fold of block partials + the phase's scalar recurrences ----------
// `gathered` holds the block partials of every rank (rank r at r*maxb*NP, its
// counts[r] blocks first) -- one rank for the 1-GPU level-1 phases, all
// ranks (all-gathered) for the row-sharded solve.  That is the global block
// order of the unsharded vector (rank row ranges are 4096-aligned), so one
// warp folding them in order reproduces vecops.py:159-161 exactly.
constexpr int kMaxRanks = 64;
struct RankCounts {
    int64_t n[kMaxRanks];
};

template <class Fin>
__global__ void __launch_bounds__(32) k_fold_finish(Fin fin, const double* __restrict__ gathered, int nranks,
                                                    int64_t rank_stride, RankCounts counts, int phase_gate) {
    __shared__ double scratch[2 * kFoldStage];
    const SolverState* st = fin.B.st;
    if (st->done || (phase_gate == 1 && !st->scheck)) return;
    constexpr int NP = Fin::kNP;
    double tot = 0.0;
    bool first = true;
    for (int r = 0; r < nranks; ++r) {
        if (counts.n[r] <= 0) continue;
        warp_fold_cont(gathered + (int64_t)r * rank_stride, NP, counts.n[r], scratch, tot, first);
        first = false;
    }
    double t[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) t[c] = __shfl_sync(0xffffffffu, tot, c);
    if (threadIdx.x == 0) fin.finish(t);
}

}  // namespace

namespace {

template <class K>
void smem_attr(K kernel, size_t bytes) {
    ZK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

struct Launch {
    zk_context* c;
    SolverPlan* P;
    // ring geometry + dynamic smem of the SpMV-phase kernels (their reducer
    // stashes and staged vectors differ): setup, K2, K4, K6x/K61
    SellView As, Ar;
    size_t smem_s, smem_r;
    RedCfg red, red1;          // reducer-warp SpMV kernels: partials slot 0 / slot 1 (row-sharded)
    PlanPtrs pc, pr;
    unsigned nb, ew, pg;      // blocks, elementwise grid, fused-reduction SpMV grid
    unsigned ppg = 1;         // plain SpMV grid (pipeline blocks may be smaller than 4096 rows)
    RankCounts one;           // {nblocks}: the 1-GPU fold's partial count
    // K3 / K5 and the K2 / K4 reduction passes on the TMA-fed engine (zk_l1pipe.cuh)
    L1View l1s, l1x, l1p, l1t;
    size_t smem_l1s = 0, smem_l1x = 0, smem_l1p = 0, smem_l1t = 0;
    unsigned grid_l1s = 0, grid_l1x = 0, grid_l1p = 0, grid_l1t = 0;
    SellView Apl;             // plain SpMV phases (K2, K4, K61 products)
    bool fuse2;               // narrow matrices: K61 + K2 products in one pass (PH_SPMV2)
    size_t smem_pl = 0;
    L1View l1r;               // true-residual pass
    size_t smem_l1r = 0;
    unsigned grid_l1r = 0;
};

// Phase events for zk_profile_enable: ev[k] is recorded before phase k's
// kernel and ev[k+1] after it (prologue phases 0-2, body phases 3-10).
// Solver phases, in zk_profile_read order (include/zk.h ZK_NPHASES):
enum Phase : int {
    PH_SETUP, PH_P_FIRST, PH_PIVOT_FIRST, PH_PIVOT_FIRST_DOT,          // prologue
    PH_S_UPDATE, PH_X_ALPHA, PH_TRUE_RES_S, PH_SPMV_T, PH_TT_TS, PH_XR_UPDATE,
    PH_TRUE_RES, PH_RES_PASS, PH_P_NEXT, PH_SPMV_PIVOT, PH_PIVOT_DOT,
    PH_SPMV2,  // narrow matrices: t = A x and v = A p^ in one pass
    PH_COUNT
};

// Events bracketing each phase's kernel (host-driven profiling loop only).
struct PhaseEvents {
    cudaEvent_t beg[PH_COUNT] = {}, end[PH_COUNT] = {};
    bool used[PH_COUNT] = {};
    bool on = false;
    cudaStream_t s = nullptr;
    void b(int k) {
        if (on) {
            ZK_CUDA(cudaEventRecord(beg[k], s));
            used[k] = true;
        }
    }
    void e(int k) {
        if (on) ZK_CUDA(cudaEventRecord(end[k], s));
    }
};

// Wraps one kernel launch in its phase's events (a no-op without profiling).
struct PhaseScope {
    PhaseEvents* pe;
    int k;
    PhaseScope(PhaseEvents* p, int kk) : pe(p), k(kk) {
        if (pe) pe->b(k);
    }
    ~PhaseScope() {
        if (pe) pe->e(k);
    }
};

// A plain SpMV phase: the narrow kernels for matrices at most 16 wide, else the ring.
inline void spmv_phase(const Launch& L, cudaStream_t s, const double2* x, double2* y, const SolverState* st) {
    if (L.Apl.narrow_w) ZK_NARROW_LAUNCH(k_spmv_phase_narrow, L.Apl, 1, s, L.Apl, x, y, st);
    else k_spmv_phase<<<L.ppg, kPipeThreads, L.smem_pl, s>>>(L.Apl, x, y, st);
}

void launch_prologue(const Launch& L, cudaStream_t s, PhaseEvents* pe = nullptr) {
    SolverBufs B = L.P->bufs;
    { PhaseScope ps(pe, PH_SETUP); k_setup<<<L.pg, kRedPipeThreads, L.smem_s, s>>>(L.As, B, L.red); }
    { PhaseScope ps(pe, PH_P_FIRST); k_p_first<<<L.ew, 256, 0, s>>>(B); }
    { PhaseScope ps(pe, PH_PIVOT_FIRST); spmv_phase(L, s, B.ph, B.v, B.st); }
    { PhaseScope ps(pe, PH_PIVOT_FIRST_DOT); k_pivot_pass<<<L.grid_l1p, kL1Threads, L.smem_l1p, s>>>(B, L.l1p, 0, 0); }
}
constexpr int kPrologueKernels = 4;

// One iteration: K3, [K3x, K6x], K4 (SpMV + pass), K5, K61 (A x into t +
// the residual pass: record / stop), Kp, K2 (SpMV + pivot pass; sets the
// WHILE condition).  K61 is a plain SpMV + pass like K2/K4 (786 vs 794 us for
// the reducer-warp SpMV on C4); one matrix pass for K61's A x and K2's A p^
// measured slower (1703 vs 799 + 716 us: two gathered vectors make the
// consumers the bottleneck).
void launch_body(const Launch& L, cudaStream_t s, cudaGraphConditionalHandle cond, int use_cond,
                 PhaseEvents* pe = nullptr) {
    SolverBufs B = L.P->bufs;
    { PhaseScope ps(pe, PH_S_UPDATE); k_s_update_pipe<<<L.grid_l1s, kL1Threads, L.smem_l1s, s>>>(B, L.l1s); }
    { PhaseScope ps(pe, PH_X_ALPHA); k_x_alpha<<<L.ew, 256, 0, s>>>(B); }
    { PhaseScope ps(pe, PH_TRUE_RES_S); k_true_res<0><<<L.pg, kRedPipeThreads, L.smem_r, s>>>(L.Ar, B, L.red); }
    { PhaseScope ps(pe, PH_SPMV_T); spmv_phase(L, s, B.sh, B.t, B.st); }
    { PhaseScope ps(pe, PH_TT_TS); k_tt_ts_pass<<<L.grid_l1t, kL1Threads, L.smem_l1t, s>>>(B, L.l1t); }
    { PhaseScope ps(pe, PH_XR_UPDATE); k_xr_update_pipe<<<L.grid_l1x, kL1Threads, L.smem_l1x, s>>>(B, L.l1x); }
    if (L.fuse2) {
        // Kp first (it reads v and writes p, p^ only; the residual pass's
        // stop decision only ever skips it, and p is not part of the result),
        // then t = A x and v = A p^ in one matrix pass, then both passes
        { PhaseScope ps(pe, PH_P_NEXT); k_p_next<<<L.ew, 256, 0, s>>>(B); }
        {
            PhaseScope ps(pe, PH_SPMV2);
            if (L.Apl.narrow_w)
                ZK_NARROW_LAUNCH(k_spmv2_phase_narrow, L.Apl, 2, s, L.Apl, B.x, B.ph, B.t, B.v, B.st);
            else
                k_spmv2_phase<<<L.ppg, kPipeThreads, L.smem_pl, s>>>(L.Apl, B.x, B.ph, B.t, B.v, B.st);
        }
        { PhaseScope ps(pe, PH_RES_PASS); k_res_pass<<<L.grid_l1r, kL1Threads, L.smem_l1r, s>>>(B, L.l1r); }
        {
            PhaseScope ps(pe, PH_PIVOT_DOT);
            k_pivot_pass<<<L.grid_l1p, kL1Threads, L.smem_l1p, s>>>(B, L.l1p, cond, use_cond);
        }
        return;
    }
    { PhaseScope ps(pe, PH_TRUE_RES); spmv_phase(L, s, B.x, B.t, B.st); }
    { PhaseScope ps(pe, PH_RES_PASS); k_res_pass<<<L.grid_l1r, kL1Threads, L.smem_l1r, s>>>(B, L.l1r); }
    { PhaseScope ps(pe, PH_P_NEXT); k_p_next<<<L.ew, 256, 0, s>>>(B); }
    { PhaseScope ps(pe, PH_SPMV_PIVOT); spmv_phase(L, s, B.ph, B.v, B.st); }
    {
        PhaseScope ps(pe, PH_PIVOT_DOT);
        k_pivot_pass<<<L.grid_l1p, kL1Threads, L.smem_l1p, s>>>(B, L.l1p, cond, use_cond);
    }
}
// launches per loop trip
inline int body_kernels(const Launch& L) { return L.fuse2 ? 10 : 11; }

void accumulate(zk_context* c, PhaseEvents& pe) {
    for (int k = 0; k < PH_COUNT; ++k) {
        if (!pe.used[k]) continue;
        ZK_CUDA(cudaEventSynchronize(pe.end[k]));
        float ms = 0.f;
        ZK_CUDA(cudaEventElapsedTime(&ms, pe.beg[k], pe.end[k]));
        c->prof_ms[k] += ms;
        c->prof_n[k] += 1;
        pe.used[k] = false;
    }
}

void set_attrs(const Launch& L) {
    smem_attr(k_setup, L.smem_s);
    smem_attr(k_spmv_phase, L.smem_pl);
    ZK_NARROW_ATTR(k_spmv_phase_narrow);
    ZK_NARROW_ATTR(k_spmv2_phase_narrow);
    smem_attr(k_spmv2_phase, L.smem_pl);
    smem_attr(k_res_pass, L.smem_l1r);
    smem_attr(k_pivot_pass, L.smem_l1p);
    smem_attr(k_tt_ts_pass, L.smem_l1t);
    smem_attr(k_true_res<0>, L.smem_r);
    smem_attr(k_s_update_pipe, L.smem_l1s);
    smem_attr(k_xr_update_pipe, L.smem_l1x);
}

bool use_graph() {
    const char* e = std::getenv("ZK_SOLVER_LOOP");
    return !(e && std::strcmp(e, "host") == 0);
}

void build_graph(const Launch& L) {
    SolverPlan* P = L.P;
    cudaStream_t s = L.c->stream;
    cudaGraph_t g;
    ZK_CUDA(cudaGraphCreate(&g, 0));
    // prologue captured into its own graph, embedded as a child node
    cudaGraph_t gp;
    ZK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    launch_prologue(L, s);
    ZK_CUDA(cudaStreamEndCapture(s, &gp));
    cudaGraphNode_t npro;
    ZK_CUDA(cudaGraphAddChildGraphNode(&npro, g, nullptr, 0, gp));
    ZK_CUDA(cudaGraphDestroy(gp));
    cudaGraphConditionalHandle cond;
    ZK_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t nloop;
    ZK_CUDA(cudaGraphAddNode(&nloop, g, &npro, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    ZK_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    launch_body(L, s, cond, 1);
    cudaGraph_t body_out;
    ZK_CUDA(cudaStreamEndCapture(s, &body_out));
    ZK_CUDA(cudaGraphInstantiate(&P->exec, g, 0));
    P->graph = g;
    P->graph_ok = true;
}

}  // namespace


void destroy_solver_plan(zk_context* c, SolverPlan* P) {
    if (!P) return;
    if (P->exec) cudaGraphExecDestroy(P->exec);
    if (P->graph) cudaGraphDestroy(P->graph);
    SolverBufs& B = P->bufs;
    void* ptrs[] = {B.x, B.b, B.minv, B.r, B.rs, B.p, B.v, B.s, B.t, B.partials, B.slots, B.hist, B.st};
    for (void* p : ptrs)
        if (p) c->alloc.free(p);
    if (B.jacobi) {
        c->alloc.free(B.ph);
        c->alloc.free(B.sh);
    }
    delete P;
}

static SolverPlan* get_plan(zk_context* c, zk_csr* A, bool jacobi, int64_t maxit) {
    SolverPlan*& slot = A->solver[jacobi ? 1 : 0];
    if (slot && slot->hist_cap < maxit + 1) {
        destroy_solver_plan(c, slot);
        slot = nullptr;
    }
    if (slot) return slot;
    SolverPlan* P = new SolverPlan();
    const int64_t n = A->n_rows;
    P->n = n;
    P->jacobi = jacobi;
    P->hist_cap = maxit + 1 > 1024 ? maxit + 1 : 1024;
    SolverBufs& B = P->bufs;
    const size_t vb = sizeof(double2) * (size_t)(n ? n : 1);
    auto vec = [&]() { return static_cast<double2*>(c->alloc.alloc(vb)); };
    B.n = n;
    B.nblocks = (n + kBlock - 1) / kBlock;
    B.jacobi = jacobi;
    B.fma = c->fma != 0;
    B.x = vec(); B.b = vec(); B.r = vec(); B.rs = vec(); B.p = vec(); B.v = vec(); B.s = vec(); B.t = vec();
    B.minv = jacobi ? vec() : nullptr;
    B.ph = jacobi ? vec() : B.p;   // identity: M.apply is a copy, bitwise equal
    B.sh = jacobi ? vec() : B.s;
    B.partials = static_cast<double*>(c->alloc.alloc(sizeof(double) * 4 * (size_t)(B.nblocks ? B.nblocks : 1)));
    B.slots = static_cast<double*>(c->alloc.alloc(sizeof(double) * 4 * (size_t)(B.nblocks ? B.nblocks : 1)));
    k_fill_empty<<<64, 256, 0, c->stream>>>(B.slots, 4 * (B.nblocks ? B.nblocks : 1));
    ZK_CUDA(cudaGetLastError());
    B.hist = static_cast<double*>(c->alloc.alloc(sizeof(double) * P->hist_cap));
    B.st = static_cast<SolverState*>(c->alloc.alloc(sizeof(SolverState)));
    slot = P;
    return P;
}

// Kernel geometry of every solver phase for matrix A and plan P (and the
// kernels' shared-memory attributes).
static Launch make_launch(zk_context* c, zk_csr* A, SolverPlan* P) {
    SolverBufs& B = P->bufs;
    const int64_t n = A->n_rows;
    Launch L;
    L.c = c;
    L.P = P;
    const size_t ex_s = RedSmem<1, 2>::kBytes, ex_r = RedSmem<0, 1>::kBytes;
    L.As = sell_view(A, c, ex_s, 1);
    L.As.sv[0] = B.b;
    L.Ar = sell_view(A, c, ex_r, 1);
    L.Ar.sv[0] = B.b;
    L.Apl = sell_view(A, c, 0, 0);
    L.ppg = plain_grid(A, L.Apl);
    {
        const char* e = std::getenv("ZK_FUSE2");  // A/B switch (experiments only)
        L.fuse2 = (L.Apl.narrow_w && !(e && e[0] == '0')) || (e && e[0] == '2');
    }
    L.smem_s = pipe_smem_bytes(L.As, ex_s);
    L.smem_pl = pipe_smem_bytes(L.Apl, 0);
    L.smem_r = pipe_smem_bytes(L.Ar, ex_r);
    L.pc = c->plans_for(n, kBlock, kComplex);
    L.pr = c->plans_for(n, kBlock, kReal);
    L.red = RedCfg{L.pc, L.pr, B.partials, &B.st->counter, B.dist, B.dist ? nullptr : B.slots};
    L.red1 = RedCfg{L.pc, L.pr, B.partials + B.pslot, &B.st->counter, B.dist, B.dist ? nullptr : B.slots};
    L.nb = (unsigned)B.nblocks;
    L.one = RankCounts{};
    L.one.n[0] = B.nblocks;
    L.pg = pipe_grid(A);
    int64_t ewg = (n + 255) / 256;
    int64_t cap = (int64_t)num_sms() * 8;
    L.ew = (unsigned)(ewg < 1 ? 1 : (ewg > cap ? cap : ewg));
    {
        double* slots = B.dist ? nullptr : B.slots;
        // row-sharded: two partials slots, so two reductions can share one
        // all-gather (K6x + K4, K5 + K61; dist.py) -- slot 0: K3, K5, K2;
        // slot 1: K4's and K61's passes
        double* partials = B.dist ? B.partials : nullptr;
        double* partials1 = B.dist ? B.partials + B.pslot : nullptr;
        // K3 stages r, v (and minv); K5 x, p^, s^ (identity: s^ is s), s, t, r~
        const double2* in3[3] = {B.r, B.v, B.jacobi ? B.minv : nullptr};
        const int8_t al3[3] = {0, 0, 0};
        const double2* in5[6] = {B.x, B.ph, B.jacobi ? B.sh : nullptr, B.s, B.t, B.rs};
        const int8_t al5[6] = {0, 0, 3, 0, 0, 0};
        // K2 pass stages r~, v; K4 pass t, s
        const double2* inp[2] = {B.rs, B.v};
        const double2* int_[2] = {B.t, B.s};
        const double2* inr[2] = {B.b, B.t};  // residual pass: b, A x (in t)
        const int8_t al2[2] = {0, 0};
        if (n > 0 && (!l1_view(c, n, kReal, in3, al3, 3, slots, partials, L.l1s, L.smem_l1s, L.grid_l1s) ||
                      !l1_view(c, n, kComplex, in5, al5, 6, slots, partials, L.l1x, L.smem_l1x, L.grid_l1x) ||
                      !l1_view(c, n, kComplex, inp, al2, 2, slots, partials, L.l1p, L.smem_l1p, L.grid_l1p) ||
                      !l1_view(c, n, kComplex, int_, al2, 2, slots, partials1, L.l1t, L.smem_l1t, L.grid_l1t,
                               (int)sizeof(cplx2)) ||
                      !l1_view(c, n, kReal, inr, al2, 2, slots, partials1, L.l1r, L.smem_l1r, L.grid_l1r)))
            throw ZkError{ZK_ERR_CUDA, "level-1 engine geometry"};
    }
    set_attrs(L);
    return L;
}

// Runs the solve; x_out/history_host/report filled.  Returns ZK_OK or
// ZK_ERR_BREAKDOWN.
int bicgstab_device(zk_context* c, zk_csr* A, const double2* b, const double2* minv, const double2* x0, double tol,
                    int64_t maxit, double2* x_out, double* history_host, zk_solve_report* rep) {
    const int64_t n = A->n_rows;
    SolverPlan* P = get_plan(c, A, minv != nullptr, maxit);
    SolverBufs& B = P->bufs;
    const bool swap = A->nnz_elide * 16 >= c->elide_bytes;
    B.fma = c->fma != 0;
    if (P->graph_ok && (P->graph_fma != B.fma || P->graph_swap != swap)) {  // arithmetic changed since capture
        if (P->exec) cudaGraphExecDestroy(P->exec);
        if (P->graph) cudaGraphDestroy(P->graph);
        P->exec = nullptr;
        P->graph = nullptr;
        P->graph_ok = false;
    }
    cudaStream_t s = c->stream;
    const size_t vb = sizeof(double2) * (size_t)n;
    ZK_CUDA(cudaMemcpyAsync(B.b, b, vb, cudaMemcpyDeviceToDevice, s));
    if (minv) ZK_CUDA(cudaMemcpyAsync(B.minv, minv, vb, cudaMemcpyDeviceToDevice, s));
    if (x0) ZK_CUDA(cudaMemcpyAsync(B.x, x0, vb, cudaMemcpyDeviceToDevice, s));
    else ZK_CUDA(cudaMemsetAsync(B.x, 0, vb, s));
    ZK_CUDA(cudaMemsetAsync(B.p, 0, vb, s));
    ZK_CUDA(cudaMemsetAsync(B.v, 0, vb, s));
    SolverState h;
    std::memset(&h, 0, sizeof(h));
    h.tol = tol;
    h.maxit = maxit;
    ZK_CUDA(cudaMemcpyAsync(B.st, &h, sizeof(h), cudaMemcpyHostToDevice, s));

    Launch L = make_launch(c, A, P);
    SolverState out;
    if (use_graph() && !c->profile) {
        if (!P->graph_ok) {
            build_graph(L);
            P->graph_fma = B.fma;
            P->graph_swap = swap;
        }
        ZK_CUDA(cudaGraphLaunch(P->exec, s));
        ZK_CUDA(cudaMemcpyAsync(&out, B.st, sizeof(out), cudaMemcpyDeviceToHost, s));
        ZK_CUDA(cudaStreamSynchronize(s));
    } else {  // host-driven loop (ZK_SOLVER_LOOP=host, or phase profiling)
        PhaseEvents pe;
        pe.on = c->profile;
        pe.s = s;
        if (pe.on)
            for (int k = 0; k < PH_COUNT; ++k) {
                ZK_CUDA(cudaEventCreate(&pe.beg[k]));
                ZK_CUDA(cudaEventCreate(&pe.end[k]));
            }
        launch_prologue(L, s, &pe);
        ZK_CUDA(cudaGetLastError());
        if (pe.on) accumulate(c, pe);
        for (;;) {
            launch_body(L, s, 0, 0, &pe);
            ZK_CUDA(cudaGetLastError());
            ZK_CUDA(cudaMemcpyAsync(&out, B.st, sizeof(out), cudaMemcpyDeviceToHost, s));
            ZK_CUDA(cudaStreamSynchronize(s));
            if (pe.on) accumulate(c, pe);
            if (out.done) break;
        }
        if (pe.on)
            for (int k = 0; k < PH_COUNT; ++k) {
                cudaEventDestroy(pe.beg[k]);
                cudaEventDestroy(pe.end[k]);
            }
    }
    c->launches += kPrologueKernels + body_kernels(L) * out.trips;
    const int64_t it = out.iterations;
    ZK_CUDA(cudaMemcpyAsync(history_host, B.hist, sizeof(double) * (it + 1), cudaMemcpyDeviceToHost, s));
    if (out.trivial_zero) ZK_CUDA(cudaMemsetAsync(x_out, 0, vb, s));
    else ZK_CUDA(cudaMemcpyAsync(x_out, B.x, vb, cudaMemcpyDeviceToDevice, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    rep->iterations = it;
    rep->converged = out.status == ST_CONVERGED;
    rep->breakdown = out.status == ST_BREAKDOWN ? out.what : 0;
    rep->final_relative_residual = history_host[it];
    rep->history_len = it + 1;
    rep->kernel_launches = kPrologueKernels + body_kernels(L) * out.trips;
    return out.status == ST_BREAKDOWN ? ZK_ERR_BREAKDOWN : ZK_OK;
}

// ---- row-sharded BiCGStab: one shard per rank ---------------------
// The local matrix holds rows [row0, row0 + n) with columns renumbered own
// rows first ([0, n)) and halo columns after ([n, n + n_halo), ascending
// global order); the vectors an SpMV gathers (x, p^, s^) carry the halo
// region, which the caller's transport fills before each SpMV phase.  Every
// reduction phase leaves its block partials in `partials` (dist = 1); the
// caller all-gathers them (rank r's maxb*NP doubles at r*maxb*NP) and
// dist_finish folds them in global block order and runs the scalar
// recurrences, identically on every rank.
struct DistSolver {  // behind zk_dshard
    zk_context* c = nullptr;
    zk_csr* A = nullptr;
    SolverPlan* P = nullptr;
    Launch L{};
    int64_t n = 0, n_ext = 0, maxb = 0;
    int nranks = 0;
    double* gathered = nullptr;
};

DistSolver* dist_create(zk_context* c, zk_csr* A, int64_t n_halo, int64_t nnz_global, bool jacobi, int64_t maxit,
                        int nranks, int64_t maxb) {
    DistSolver* D = new DistSolver();
    D->c = c;
    D->A = A;
    D->n = A->n_rows;
    D->n_ext = A->n_rows + n_halo;
    D->nranks = nranks;
    D->maxb = maxb;
    A->nnz_elide = nnz_global;  // numpy's elision decision is the unsharded matrix's
    SolverPlan* P = new SolverPlan();
    P->n = D->n;
    P->jacobi = jacobi;
    P->hist_cap = maxit + 1 > 1024 ? maxit + 1 : 1024;
    SolverBufs& B = P->bufs;
    const size_t vb = sizeof(double2) * (size_t)(D->n_ext ? D->n_ext : 1);
    auto vec = [&]() {
        double2* v = static_cast<double2*>(c->alloc.alloc(vb));
        ZK_CUDA(cudaMemsetAsync(v, 0, vb, c->stream));
        return v;
    };
    B.n = D->n;
    B.nblocks = (D->n + kBlock - 1) / kBlock;
    B.jacobi = jacobi;
    B.fma = c->fma != 0;
    B.dist = 1;
    B.x = vec(); B.b = vec(); B.r = vec(); B.rs = vec(); B.p = vec(); B.v = vec(); B.s = vec(); B.t = vec();
    B.minv = jacobi ? vec() : nullptr;
    B.ph = jacobi ? vec() : B.p;
    B.sh = jacobi ? vec() : B.s;
    const int64_t pb = maxb > B.nblocks ? maxb : B.nblocks;
    B.pslot = 4 * (pb ? pb : 1);
    B.partials = static_cast<double*>(c->alloc.alloc(sizeof(double) * 2 * (size_t)B.pslot));
    ZK_CUDA(cudaMemsetAsync(B.partials, 0, sizeof(double) * 2 * (size_t)B.pslot, c->stream));
    B.hist = static_cast<double*>(c->alloc.alloc(sizeof(double) * P->hist_cap));
    B.st = static_cast<SolverState*>(c->alloc.alloc(sizeof(SolverState)));
    D->gathered = static_cast<double*>(c->alloc.alloc(sizeof(double) * 2 * (size_t)B.pslot * (size_t)nranks));
    D->P = P;
    D->L = make_launch(c, A, P);
    return D;
}

void dist_destroy(DistSolver* D) {
    if (!D) return;
    D->c->alloc.free(D->gathered);
    destroy_solver_plan(D->c, D->P);
    delete D;
}

void* dist_vector(DistSolver* D, int which, int64_t* len) {
    SolverBufs& B = D->P->bufs;
    switch (which) {
        case ZK_DVEC_X: *len = D->n_ext; return B.x;
        case ZK_DVEC_PHAT: *len = D->n_ext; return B.ph;
        case ZK_DVEC_SHAT: *len = D->n_ext; return B.sh;
        case ZK_DVEC_B: *len = D->n; return B.b;
        case ZK_DVEC_MINV: *len = B.jacobi ? D->n : 0; return B.minv;
        case ZK_DVEC_PARTIALS: *len = 2 * B.pslot; return B.partials;
        case ZK_DVEC_GATHERED: *len = 2 * B.pslot * (int64_t)D->nranks; return D->gathered;
        default: throw ZkError{ZK_ERR_PARAMETER, "unknown shard vector"};
    }
}

void dist_reset(DistSolver* D, double tol, int64_t maxit, bool has_x0) {
    SolverBufs& B = D->P->bufs;
    if (maxit + 1 > D->P->hist_cap) throw ZkError{ZK_ERR_PARAMETER, "max_iterations above the shard's capacity"};
    // the launch parameters carry the arithmetic fingerprint (SellView::fma,
    // ::swap, SolverBufs::fma): rebuild them in case zk_set_arith changed it
    B.fma = D->c->fma != 0;
    D->L = make_launch(D->c, D->A, D->P);
    cudaStream_t s = D->c->stream;
    const size_t vb = sizeof(double2) * (size_t)D->n_ext;
    if (!has_x0) ZK_CUDA(cudaMemsetAsync(B.x, 0, vb, s));
    ZK_CUDA(cudaMemsetAsync(B.p, 0, vb, s));
    ZK_CUDA(cudaMemsetAsync(B.v, 0, vb, s));
    SolverState h;
    std::memset(&h, 0, sizeof(h));
    h.tol = tol;
    h.maxit = maxit;
    ZK_CUDA(cudaMemcpyAsync(B.st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
}

void dist_phase(DistSolver* D, int phase) {
    const Launch& L = D->L;
    cudaStream_t s = D->c->stream;
    SolverBufs& B = D->P->bufs;
    if (D->n == 0) throw ZkError{ZK_ERR_DIMENSION, "empty shard"};
    switch (phase) {
        case ZK_DPHASE_SETUP: k_setup<<<L.pg, kRedPipeThreads, L.smem_s, s>>>(L.As, B, L.red); break;
        case ZK_DPHASE_P_FIRST: k_p_first<<<L.ew, 256, 0, s>>>(B); break;
        case ZK_DPHASE_PIVOT:
            spmv_phase(L, s, B.ph, B.v, B.st);
            ZK_CUDA(cudaGetLastError());
            D->c->launches++;
            k_pivot_pass<<<L.grid_l1p, kL1Threads, L.smem_l1p, s>>>(B, L.l1p, 0, 0);
            break;
        case ZK_DPHASE_S_UPDATE: k_s_update_pipe<<<L.grid_l1s, kL1Threads, L.smem_l1s, s>>>(B, L.l1s); break;
        case ZK_DPHASE_X_ALPHA: k_x_alpha<<<L.ew, 256, 0, s>>>(B); break;
        case ZK_DPHASE_TRUE_RES_S: k_true_res<0><<<L.pg, kRedPipeThreads, L.smem_r, s>>>(L.Ar, B, L.red); break;
        case ZK_DPHASE_SPMV_T:
            spmv_phase(L, s, B.sh, B.t, B.st);
            ZK_CUDA(cudaGetLastError());
            D->c->launches++;
            k_tt_ts_pass<<<L.grid_l1t, kL1Threads, L.smem_l1t, s>>>(B, L.l1t);
            break;
        case ZK_DPHASE_XR_UPDATE: k_xr_update_pipe<<<L.grid_l1x, kL1Threads, L.smem_l1x, s>>>(B, L.l1x); break;
        case ZK_DPHASE_TRUE_RES:  // A x into t, residual pass -> slot 1
            spmv_phase(L, s, B.x, B.t, B.st);
            ZK_CUDA(cudaGetLastError());
            D->c->launches++;
            k_res_pass<<<L.grid_l1r, kL1Threads, L.smem_l1r, s>>>(B, L.l1r);
            break;
        case ZK_DPHASE_P_NEXT: k_p_next<<<L.ew, 256, 0, s>>>(B); break;
        default: throw ZkError{ZK_ERR_PARAMETER, "unknown solver phase"};
    }
    ZK_CUDA(cudaGetLastError());
    D->c->launches++;
}

void dist_finish(DistSolver* D, int phase, const int64_t* rank_blocks) {
    if (D->nranks > kMaxRanks) throw ZkError{ZK_ERR_PARAMETER, "too many ranks"};
    RankCounts rc{};
    for (int r = 0; r < D->nranks; ++r) rc.n[r] = rank_blocks[r];
    SolverBufs& B = D->P->bufs;
    cudaStream_t s = D->c->stream;
    const int nr = D->nranks;
    const int64_t rs = 2 * B.pslot;                        // doubles per rank in `gathered`
    const double* g0 = D->gathered;                         // slot 0
    const double* g1 = D->gathered + B.pslot;               // slot 1 (K4, K61)
    switch (phase) {
        case ZK_DPHASE_SETUP: k_fold_finish<<<1, 32, 0, s>>>(SetupBody{B}, g0, nr, rs, rc, 0); break;
        case ZK_DPHASE_PIVOT: k_fold_finish<<<1, 32, 0, s>>>(PivotFin{B, 0, 0}, g0, nr, rs, rc, 0); break;
        case ZK_DPHASE_S_UPDATE: k_fold_finish<<<1, 32, 0, s>>>(SUpdFinish{B}, g0, nr, rs, rc, 0); break;
        case ZK_DPHASE_TRUE_RES_S: k_fold_finish<<<1, 32, 0, s>>>(ResBody<0>{B}, g0, nr, rs, rc, 1); break;
        case ZK_DPHASE_SPMV_T: k_fold_finish<<<1, 32, 0, s>>>(TFin{B}, g1, nr, rs, rc, 0); break;
        case ZK_DPHASE_XR_UPDATE: k_fold_finish<<<1, 32, 0, s>>>(XrFinish{B}, g0, nr, rs, rc, 0); break;
        case ZK_DPHASE_TRUE_RES: k_fold_finish<<<1, 32, 0, s>>>(ResBody<1>{B}, g1, nr, rs, rc, 0); break;
        default: throw ZkError{ZK_ERR_PARAMETER, "phase has no reduction"};
    }
    ZK_CUDA(cudaGetLastError());
    D->c->launches++;
}

__global__ void k_pack(const double2* __restrict__ v, const int64_t* __restrict__ idx, int64_t count,
                       double2* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v[idx[i]];
}

void dist_pack(DistSolver* D, int which, const int64_t* idx, int64_t count, double2* out) {
    if (count <= 0) return;
    int64_t len;
    const double2* v = static_cast<const double2*>(dist_vector(D, which, &len));
    const int64_t g = (count + 255) / 256;
    k_pack<<<(unsigned)(g < 4096 ? g : 4096), 256, 0, D->c->stream>>>(v, idx, count, out);
    ZK_CUDA(cudaGetLastError());
    D->c->launches++;
}

void dist_status(DistSolver* D, zk_solve_report* rep, int32_t* done) {
    SolverState out;
    cudaStream_t s = D->c->stream;
    ZK_CUDA(cudaMemcpyAsync(&out, D->P->bufs.st, sizeof(out), cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    rep->iterations = out.iterations;
    rep->converged = out.status == ST_CONVERGED;
    rep->breakdown = out.status == ST_BREAKDOWN ? out.what : 0;
    rep->history_len = out.iterations + 1;
    rep->final_relative_residual = out.last_rel;
    rep->kernel_launches = 0;
    *done = out.done ? (out.trivial_zero ? 2 : 1) : 0;
}

void dist_history(DistSolver* D, double* host, int64_t count) {
    if (count > D->P->hist_cap) throw ZkError{ZK_ERR_PARAMETER, "history longer than the shard's capacity"};
    ZK_CUDA(cudaMemcpyAsync(host, D->P->bufs.hist, sizeof(double) * count, cudaMemcpyDeviceToHost, D->c->stream));
    ZK_CUDA(cudaStreamSynchronize(D->c->stream));
}

}  // namespace zk
