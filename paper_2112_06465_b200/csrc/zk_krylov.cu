// zk_krylov.cu -- device-resident BiCGSTAB(l) (krylov.py:298-410) and TFQMR
// (krylov.py:413-489), bitwise faithful to the reference.
//
// The loops are not transcriptions run from the host: every vector and every
// scalar of the recurrences lives on the device, and a whole solve is ONE
// CUDA-graph launch with ONE host synchronisation.  The host captures the
// loop body once per (matrix, solver, l, preconditioner) -- one outer cycle
// of BiCGSTAB(l), two iterations of TFQMR (the two iterations alternate the
// roles of the uvec / u_old buffers, so no copy is needed) -- into the body
// of a device-side conditional WHILE node.  Control flow the reference
// expresses with `if`/`return`/`raise` (breakdowns, the early residual
// probe inside the BiCG part, TFQMR's convergence after a half-step) is
// device-side predication: every kernel of the body carries a Gate on the
// solver's state words (zk_common.cuh) and returns at once when the solve
// has stopped or the branch it belongs to is not taken.
//
// Kernels used per step:
//   * SpMV phases: the persistent TMA pipeline of zk_spmv.cuh with bodies
//     for r0 = b - A x0 (+ ||b||, ||r0||, <r0, r0>) and y = A z (+ a copy);
//     the BiCG pivot <r~, A z> and the true residual ||b - A x|| / ||b||
//     (whose finish() does the reference's bookkeeping) are passes on the
//     level-1 engine after a plain SpMV.
//   * Reductions: the block-plan kernels of zk_blas1.cu with a Gate,
//     writing their scalar into the state block (streaming ordered fold).
//   * Elementwise: k_pairs (a batch of independent zscal+zaxpy / zaxpy
//     updates on distinct vectors in one pass), k_mr_update (the whole
//     minimal-residual update of BiCGSTAB(l): acc, r0, u0 in one pass over
//     the 2l+3 vectors instead of 3l zaxpy passes), k_curx
//     (x = x0 + M^-1 acc), k_jac (M^-1 v), k_tf_v (TFQMR's v update).
//   * Scalars: k_kscalar, one thread, Python's Cplx arithmetic (cmul_py,
//     cdiv_py, zk_common.cuh) in the reference's operation order.
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
double* fold_slots(zk_context* c, int64_t count);
void zdot_device(zk_context* c, int64_t n, const double2* x, const double2* y, bool conj, int64_t block, int mode,
                 double2* result, Gate gate);
void znorm2_device(zk_context* c, int64_t n, const double2* x, int64_t block, int mode, double* result, Gate gate);

// Breakdown codes (include/zk.h ZK_BD_*; oracle/zk_oracle.c uses the same).
enum : int32_t { KB_RHO = 1, KB_OMEGA = 2, KB_PIVOT = 3, KB_MR = 5, KB_SIGMA = 6, KB_ALPHA = 7, KB_TAU = 8 };
enum : int32_t { KS_RUNNING = 0, KS_CONVERGED = 1, KS_NOT_CONVERGED = 2, KS_BREAKDOWN = 3 };

struct KState {
    int32_t done, flag;  // Gate words: the solve stopped; the branch flag (l: residual probe; TFQMR: half converged)
    int32_t status, what, what_j, trivial;
    int64_t maxit, iterations, trips;
    double b_norm, tol, r0_norm, rel, theta, tau, c, nrm;
    double2 rho, alpha, omega, beta, eta, coefd, dot;
    double2 rho_prev;  // TFQMR, narrow matrices: rho before KO_T_BETA_CALC (its check is deferred)
};

// MR scalars of BiCGSTAB(l), indexed as in krylov.py:366-391 (l <= kMaxEll).
constexpr int kMaxEll = 32;
struct KMr {
    double2 tau[(kMaxEll + 1) * (kMaxEll + 1)];
    double sigma[kMaxEll + 1];
    double2 gp[kMaxEll + 1], gm[kMaxEll + 1], gpp[kMaxEll + 1];
};

enum KSolver : int32_t { KSV_BICGSTABL = 0, KSV_TFQMR = 1 };

namespace {

__device__ __forceinline__ double2 negz(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double2 rz(double v) { return make_double2(v, 0.0); }

__device__ __forceinline__ void kstop(KState* st, int32_t status, int32_t what = 0, int32_t j = 0) {
    st->status = status;
    st->what = what;
    st->what_j = j;
    st->done = 1;
}

// ---- SpMV-phase bodies (zk_spmv.cuh reducer pipeline) -----------------------

// _Run.__init__ (krylov.py:147-168): r0 = b + F1(-1, A x0) into up to three
// vectors, ||b||, ||r0|| and <r0, r0> (TFQMR's first rho, krylov.py:436);
// trivial_result (krylov.py:171-181) and the solver's initial scalars.
struct KSetupBody {
    static constexpr int kNC = 1, kNR = 2, kSV = 1;  // staged: b
    static constexpr int kNP = 2 * kNC + kNR;
    double2* out0;
    double2* out1;
    double2* out2;
    KState* st;
    double* hist;
    int32_t solver;
    bool fma;
    __device__ void row(int64_t row, const double2 (&ax)[1], const double2 (&sv)[1], double2 (&tc)[1],
                        double (&tr)[2]) {
        const double2 b = sv[0];
        const double2 r0 = cadd(b, f1(make_double2(-1.0, 0.0), ax[0], fma));
        out0[row] = r0;
        if (out1) out1[row] = r0;
        if (out2) out2[row] = r0;
        tc[0] = f1(conjz(r0), r0, fma);
        tr[0] = abs2_np(b);
        tr[1] = abs2_np(r0);
    }
    __device__ void finish(const double* t) {  // [<r0,r0>.re, .im, |b|^2, |r0|^2]
        const double bn = __dsqrt_rn(t[2]), rn = __dsqrt_rn(t[3]);
        st->b_norm = bn;
        st->r0_norm = rn;
        const double h0 = bn > 0.0 ? __ddiv_rn(rn, bn) : 0.0;
        hist[0] = h0;
        st->rel = h0;
        if (bn == 0.0) {  // zero rhs: x = 0, history [0.0]
            hist[0] = 0.0;
            st->rel = 0.0;
            st->trivial = 1;
            kstop(st, KS_CONVERGED);
            return;
        }
        if (h0 <= st->tol) {  // the initial guess already solves: x = x0
            kstop(st, KS_CONVERGED);
            return;
        }
        if (solver == KSV_BICGSTABL) {  // krylov.py:333-335
            st->rho = rz(1.0);
            st->alpha = rz(0.0);
            st->omega = rz(1.0);
        } else {  // krylov.py:432-436
            st->theta = 0.0;
            st->eta = rz(0.0);
            st->tau = rn;
            st->rho = make_double2(t[0], t[1]);
        }
    }
};

// y = A x (and a second copy: TFQMR's v = uvec.copy(), krylov.py:431)
struct KPlainBody {
    static constexpr int kNC = 0, kNR = 0, kSV = 0;
    static constexpr int kNP = 0;
    double2* y;
    double2* y2;
    __device__ __forceinline__ void row(int64_t r, const double2 (&v)[1], const double2 (&)[1], double2 (&)[1],
                                        double (&)[1]) {
        y[r] = v[0];
        if (y2) y2[r] = v[0];
    }
    __device__ void finish(const double*) {}
};

// Two products from one matrix pass (narrow matrices, TFQMR): y0 = A x0, y1 = A x1.
struct KPlain2Body {
    static constexpr int kNC = 0, kNR = 0, kSV = 0;
    double2* y0;
    double2* y1;
    __device__ __forceinline__ void row(int64_t r, const double2 (&v)[2], const double2 (&)[1], double2 (&)[1],
                                        double (&)[1]) {
        y0[r] = v[0];
        y1[r] = v[1];
    }
};

// _Run.true_relative_residual (krylov.py:183-186) and what the caller does with it:
//   MODE 0  BiCGSTAB(l) residual probe (krylov.py:355-360): record + stop only when converged
//   MODE 1  BiCGSTAB(l) end of cycle (krylov.py:403-407): record; stop when converged or at the cap
//   MODE 2  TFQMR half-step (krylov.py:462-465): keep rel, flag convergence
template <int MODE>
struct KResBody {
    static constexpr int kNC = 0, kNR = 1, kSV = 1;  // staged: b
    static constexpr int kNP = 1;
    KState* st;
    double* hist;
    bool fma;
    __device__ void row(int64_t, const double2 (&ax)[1], const double2 (&sv)[1], double2 (&)[1], double (&tr)[1]) {
        tr[0] = abs2_np(cadd(sv[0], f1(make_double2(-1.0, 0.0), ax[0], fma)));
    }
    __device__ void finish(const double* t) {
        const double rel = __ddiv_rn(__dsqrt_rn(t[0]), st->b_norm);
        if (MODE == 2) {
            st->rel = rel;
            if (rel <= st->tol) st->flag = 1;
            return;
        }
        if (MODE == 0 && !(rel <= st->tol)) return;
        st->iterations++;
        hist[st->iterations] = rel;
        st->rel = rel;
        if (rel <= st->tol) kstop(st, KS_CONVERGED);
        else if (MODE == 1 && st->iterations >= st->maxit) kstop(st, KS_NOT_CONVERGED);
    }
};

// True residual as a pass over (b, A x) on the level-1 engine, after a plain
// SpMV wrote A x: the same terms and order as KResBody's fused reduction.
struct KResOp {
    using V = double;
    static constexpr int NIN = 2;  // b, A x
    bool fma;
    __device__ __forceinline__ double apply(int64_t, const double2 (&v)[2]) const {
        return abs2_np(cadd(v[0], f1(make_double2(-1.0, 0.0), v[1], fma)));
    }
};

template <int MODE>
__global__ void __launch_bounds__(kL1Threads, 1) k_kres_pass(L1View P, KResBody<MODE> fin, bool fma, Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    KResOp op{fma};
    l1_pipeline(P, op, fin, smem);
}

template <class Body>
__global__ void __launch_bounds__(kRedPipeThreads, 1) k_kspmv_red(SellView A, const double2* __restrict__ x, Body body,
                                                                   RedCfg R, Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    sell_run<1>(A, x, nullptr, body, R, smem);
}

__global__ void __launch_bounds__(kPipeThreads, 1) k_kspmv(SellView A, const double2* __restrict__ x, KPlainBody body,
                                                           Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    const RedCfg R{};
    sell_run<1>(A, x, nullptr, body, R, smem);
}

template <int WM>
__global__ void __launch_bounds__(32 * NarrowCfg<WM>::warps(1), NarrowCfg<WM>::kMinB)
    k_kspmv_narrow(SellView A, const double2* __restrict__ x, KPlainBody body, Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    narrow_tma_run<WM, 1>(A, x, x, body, smem);
}

template <int WM>
__global__ void __launch_bounds__(32 * NarrowCfg<WM>::warps(2), NarrowCfg<WM>::kMinB2)
    k_kspmv2_narrow(SellView A, const double2* __restrict__ x0, const double2* __restrict__ x1, KPlain2Body body,
                    Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    narrow_tma_run<WM, 2>(A, x0, x1, body, smem);
}

// ---- elementwise kernels -------------------------------------------------------

constexpr int kEwThreads = 256;
constexpr int kMaxPairs = 12;

// One update per op on vector y_k: y = S(y) + F1(cb, x) where S(y) = F1(y, ca)
// (zscal, vecops.py:124-127) when the op scales, else y; then zaxpy
// (vecops.py:130-134).  Coefficients are device scalars (null cb = (1, 0),
// Cplx(1.0)), optionally negated (Cplx.__neg__, exact).  The ops of one
// launch touch distinct y vectors, except that an op may follow another on
// the same y (each thread applies the ops of its element in order).
struct PairOp {
    const double2* x;
    double2* y;
    const double2* ca;
    const double2* cb;
    int32_t flags;
};
enum : int32_t { PF_SCALE = 1, PF_NEG_A = 2, PF_NEG_B = 4 };
struct Pairs {
    PairOp op[kMaxPairs];
    int32_t n;
};

__global__ void __launch_bounds__(kEwThreads) k_pairs(Pairs P, int64_t n, bool fma, Gate gate) {
    if (gate.skip()) return;
    // ops staged in shared memory (a dynamically indexed kernel parameter
    // would be copied to local memory per thread)
    __shared__ double2 ca[kMaxPairs], cb[kMaxPairs];
    __shared__ const double2* xs[kMaxPairs];
    __shared__ double2* ys[kMaxPairs];
    __shared__ int32_t fl[kMaxPairs];
    const int np = P.n;
    if (threadIdx.x < (unsigned)np) {
        const PairOp o = P.op[threadIdx.x];
        double2 a = o.ca ? *o.ca : rz(1.0), b = o.cb ? *o.cb : rz(1.0);
        if (o.flags & PF_NEG_A) a = negz(a);
        if (o.flags & PF_NEG_B) b = negz(b);
        ca[threadIdx.x] = a;
        cb[threadIdx.x] = b;
        xs[threadIdx.x] = o.x;
        ys[threadIdx.x] = o.y;
        fl[threadIdx.x] = o.flags;
    }
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        for (int k = 0; k < np; ++k) {
            double2* yp = ys[k];
            double2 y = yp[i];
            if (fl[k] & PF_SCALE) y = f1(y, ca[k], fma);
            yp[i] = cadd(y, f1(cb[k], __ldg(xs[k] + i), fma));
        }
    }
}

// M^-1 v (Preconditioner.apply, krylov.py:92-100: F1(v, minv))
__global__ void __launch_bounds__(kEwThreads) k_jac(int64_t n, const double2* __restrict__ v,
                                                    const double2* __restrict__ m, double2* __restrict__ out, bool fma,
                                                    Gate gate) {
    if (gate.skip()) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = f1(__ldg(v + i), __ldg(m + i), fma);
}

// current_x(acc) = x0.copy(); zaxpy(1, M.apply(acc), x)  (krylov.py:323-326)
__global__ void __launch_bounds__(kEwThreads) k_curx(int64_t n, const double2* __restrict__ x0,
                                                     const double2* __restrict__ acc, const double2* __restrict__ m,
                                                     double2* __restrict__ x, bool fma, Gate gate) {
    if (gate.skip()) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 a = __ldg(acc + i);
        if (m) a = f1(a, __ldg(m + i), fma);
        x[i] = cadd(__ldg(x0 + i), f1(rz(1.0), a, fma));
    }
}

// BiCGSTAB(l) minimal-residual update (krylov.py:393-400), all three vectors
// in one pass: acc += gm1 r0 (old r0); r0 -= gp_l r_l; u0 -= gm_l u_l; then
// for j = 1..l-1: u0 -= gm_j u_j, acc += gpp_j r_j, r0 -= gp_j r_j -- each
// vector's updates in the reference's order, one rounding per zaxpy.
struct MrVecs {
    double2* r[kMaxEll + 1];
    double2* u[kMaxEll + 1];
};

__global__ void __launch_bounds__(kEwThreads) k_mr_update(MrVecs V, int ell, int64_t n, double2* __restrict__ acc,
                                                          const KMr* __restrict__ mr, bool fma, Gate gate) {
    if (gate.skip()) return;
    __shared__ double2 ngm[kMaxEll + 1], ngp[kMaxEll + 1], gpp[kMaxEll + 1];
    __shared__ const double2* rv[kMaxEll + 1];
    __shared__ const double2* uv[kMaxEll + 1];
    for (int j = threadIdx.x; j <= ell; j += blockDim.x) {
        ngm[j] = negz(mr->gm[j]);
        ngp[j] = negz(mr->gp[j]);
        gpp[j] = mr->gpp[j];
        rv[j] = V.r[j];
        uv[j] = V.u[j];
    }
    __syncthreads();
    const double2 gm1 = negz(ngm[1]);
    double2* r0p = V.r[0];
    double2* u0p = V.u[0];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 r0 = r0p[i];
        double2 a = cadd(acc[i], f1(gm1, r0, fma));
        r0 = cadd(r0, f1(ngp[ell], __ldg(rv[ell] + i), fma));
        double2 u0 = cadd(u0p[i], f1(ngm[ell], __ldg(uv[ell] + i), fma));
        for (int j = 1; j < ell; ++j) {
            u0 = cadd(u0, f1(ngm[j], __ldg(uv[j] + i), fma));
            const double2 rj = __ldg(rv[j] + i);
            a = cadd(a, f1(gpp[j], rj, fma));
            r0 = cadd(r0, f1(ngp[j], rj, fma));
        }
        acc[i] = a;
        r0p[i] = r0;
        u0p[i] = u0;
    }
}

// TFQMR: v = beta * (u_old + beta * v) + u_new  (krylov.py:485-489: zscal,
// zaxpy, zscal, zaxpy -- four roundings, in that order)
__global__ void __launch_bounds__(kEwThreads) k_tf_v(int64_t n, double2* __restrict__ v,
                                                     const double2* __restrict__ uold,
                                                     const double2* __restrict__ unew, const KState* st, bool fma,
                                                     Gate gate) {
    if (gate.skip()) return;
    const double2 beta = st->beta, one = rz(1.0);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 t = f1(v[i], beta, fma);
        t = cadd(t, f1(one, __ldg(uold + i), fma));
        t = f1(t, beta, fma);
        v[i] = cadd(t, f1(one, __ldg(unew + i), fma));
    }
}

// ---- scalar recurrences -------------------------------------------------------
enum KOp : int32_t {
    // BiCGSTAB(l)
    KO_L_CYCLE = 0,   // omega check; rho = -omega * rho                (krylov.py:340-342)
    KO_L_BETA = 1,    // rho check; beta = alpha * (rho'/rho); rho = rho' (krylov.py:346-350)
    KO_L_ALPHA = 2,   // pivot check; alpha = rho / pivot                (krylov.py:352-355)
    KO_L_PROBE = 3,   // flag = ||r0|| / ||b|| <= tol                     (krylov.py:359)
    KO_L_TAU = 4,     // tau[i][j] = <r_i, r_j> / sigma[i]               (krylov.py:371-373)
    KO_L_SIGMA = 5,   // sigma[j] = <r_j, r_j>.re, check                 (krylov.py:375-377)
    KO_L_GAMMAP = 6,  // gamma'[j] = <r_j, r_0> / sigma[j]               (krylov.py:378)
    KO_L_GAMMA = 7,   // gamma, omega, gamma''                           (krylov.py:379-391)
    // TFQMR
    KO_T_ALPHA = 10,  // sigma check; alpha; alpha check; d coefficient  (krylov.py:439-444, 452)
    KO_T_COEFD = 11,  // d coefficient for the second half-step          (krylov.py:452)
    KO_T_THETA = 12,  // tau check; theta, c, tau, eta                   (krylov.py:454-459)
    KO_T_BETA = 14,   // rho check; beta = rho'/rho; rho = rho'           (krylov.py:469-473)
    KO_T_END = 15,    // iteration cap                                   (krylov.py:438)
    // TFQMR with the end-of-iteration products moved ahead of the second residual
    KO_T_BETA_CALC = 16,  // beta = rho'/rho; rho = rho' (rho kept for the check)  (krylov.py:471-473)
    KO_T_BETA_CHK = 17,   // rho check, in the reference's place after record     (krylov.py:469-470)
};

__global__ void k_kscalar(KState* st, KMr* mr, int32_t op, int32_t i, int32_t j, Gate gate) {
    if (gate.skip()) return;
    switch (op) {
        case KO_L_CYCLE:
            if (small_py(st->omega)) { kstop(st, KS_BREAKDOWN, KB_OMEGA); return; }
            st->rho = cmul_py(negz(st->omega), st->rho);
            return;
        case KO_L_BETA: {
            const double2 rn = st->dot;
            if (small_py(st->rho)) { kstop(st, KS_BREAKDOWN, KB_RHO); return; }
            st->beta = cmul_py(st->alpha, cdiv_py(rn, st->rho));
            st->rho = rn;
            return;
        }
        case KO_L_ALPHA: {
            const double2 pivot = st->dot;
            if (small_py(pivot)) { kstop(st, KS_BREAKDOWN, KB_PIVOT); return; }
            st->alpha = cdiv_py(st->rho, pivot);
            return;
        }
        case KO_L_PROBE:
            st->flag = (__ddiv_rn(st->nrm, st->b_norm) <= st->tol) ? 1 : 0;
            return;
        case KO_L_TAU:
            mr->tau[i * (kMaxEll + 1) + j] = cdiv_py(st->dot, rz(mr->sigma[i]));
            return;
        case KO_L_SIGMA: {
            const double sg = st->dot.x;
            mr->sigma[j] = sg;
            if (small_py(sg)) kstop(st, KS_BREAKDOWN, KB_MR, j);
            return;
        }
        case KO_L_GAMMAP:
            mr->gp[j] = cdiv_py(st->dot, rz(mr->sigma[j]));
            return;
        case KO_L_GAMMA: {
            const int ell = i;
            for (int k = 0; k <= ell; ++k) mr->gm[k] = rz(0.0);
            mr->gm[ell] = mr->gp[ell];
            st->omega = mr->gm[ell];
            for (int jj = ell - 1; jj >= 1; --jj) {
                double2 s = rz(0.0);
                for (int ii = jj + 1; ii <= ell; ++ii) s = cadd(s, cmul_py(mr->tau[jj * (kMaxEll + 1) + ii], mr->gm[ii]));
                mr->gm[jj] = make_double2(__dsub_rn(mr->gp[jj].x, s.x), __dsub_rn(mr->gp[jj].y, s.y));
            }
            for (int jj = 1; jj < ell; ++jj) {
                double2 s = rz(0.0);
                for (int ii = jj + 1; ii < ell; ++ii)
                    s = cadd(s, cmul_py(mr->tau[jj * (kMaxEll + 1) + ii], mr->gm[ii + 1]));
                mr->gpp[jj] = cadd(mr->gm[jj + 1], s);
            }
            return;
        }
        case KO_T_ALPHA: {
            const double2 sigma = st->dot;
            if (small_py(sigma)) { kstop(st, KS_BREAKDOWN, KB_SIGMA); return; }
            const double2 alpha = cdiv_py(st->rho, sigma);
            if (small_py(alpha)) { kstop(st, KS_BREAKDOWN, KB_ALPHA); return; }
            st->alpha = alpha;
            st->flag = 0;
            st->rel = __longlong_as_double(0x7FF0000000000000ll);  // math.inf
            st->coefd = cdiv_py(cmul_py(st->eta, rz(__dmul_rn(st->theta, st->theta))), alpha);
            return;
        }
        case KO_T_COEFD:
            st->coefd = cdiv_py(cmul_py(st->eta, rz(__dmul_rn(st->theta, st->theta))), st->alpha);
            return;
        case KO_T_THETA: {
            if (small_py(st->tau)) { kstop(st, KS_BREAKDOWN, KB_TAU); return; }
            const double theta = __ddiv_rn(st->nrm, st->tau);
            const double c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(theta, theta))));
            st->theta = theta;
            st->c = c;
            st->tau = __dmul_rn(__dmul_rn(st->tau, theta), c);
            st->eta = cmul_py(st->alpha, rz(__dmul_rn(c, c)));
            return;
        }
        case KO_T_BETA: {
            const double2 rn = st->dot;
            if (small_py(st->rho)) { kstop(st, KS_BREAKDOWN, KB_RHO); return; }
            st->beta = cdiv_py(rn, st->rho);
            st->rho = rn;
            return;
        }
        case KO_T_BETA_CALC:
            st->rho_prev = st->rho;
            st->beta = cdiv_py(st->dot, st->rho);
            st->rho = st->dot;
            return;
        case KO_T_BETA_CHK:
            if (small_py(st->rho_prev)) kstop(st, KS_BREAKDOWN, KB_RHO);
            return;
        case KO_T_END:
            if (st->iterations >= st->maxit) kstop(st, KS_NOT_CONVERGED);
            return;
        default:
            return;
    }
}

// TFQMR run.record(rel) + convergence stop (krylov.py:466-468)
__global__ void k_krecord(KState* st, double* hist, Gate gate) {
    if (gate.skip()) return;
    st->iterations++;
    hist[st->iterations] = st->rel;
    if (st->flag) kstop(st, KS_CONVERGED);
}

// Last kernel of the loop body: continue while the solve runs.
__global__ void k_kloop_end(KState* st, cudaGraphConditionalHandle cond) {
    st->trips++;
    cudaGraphSetConditional(cond, st->done ? 0u : 1u);
}

__global__ void k_kfill(double* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = __longlong_as_double((long long)kSlotEmpty);
}

}  // namespace

// ---- host side -----------------------------------------------------------------

struct KrylovPlan {
    int32_t solver = 0, ell = 0;
    bool jacobi = false;
    int64_t n = 0, hist_cap = 0;
    // vectors (device, n each)
    double2 *x = nullptr, *x0 = nullptr, *b = nullptr, *minv = nullptr, *rs = nullptr, *tmp = nullptr;
    double2* ax = nullptr;         // A x of the true residual
    double2* r[kMaxEll + 1] = {};  // l: r[0..l]
    double2* u[kMaxEll + 1] = {};  // l: u[0..l]
    double2* acc = nullptr;
    double2 *w = nullptr, *y = nullptr, *d = nullptr, *z = nullptr, *v = nullptr, *U[2] = {};  // TFQMR
    double* hist = nullptr;
    KState* st = nullptr;
    KMr* mr = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool graph_fma = true, graph_swap = false;
    int64_t body_kernels = 0, prologue_kernels = 0;
};

namespace {

struct KLaunch {
    zk_context* c;
    const zk_csr* A;
    KrylovPlan* P;
    bool fma;
    int64_t n;
    unsigned ew, pg;
    PlanPtrs pc, pr;
    double* slots;
    int64_t count = 0;  // kernels enqueued
    cudaStream_t s;
    bool fuse2 = false;  // narrow matrix: TFQMR's A x and A z in one pass (t_iteration)

    Gate live() const { return Gate{&P->st->done, Gate::kLive}; }
    Gate nofl() const { return Gate{&P->st->done, Gate::kLiveNoFlag}; }
    Gate onfl() const { return Gate{&P->st->done, Gate::kLiveFlag}; }

    void check() {
        ZK_CUDA(cudaGetLastError());
        ++count;
    }

    template <class Body>
    void spmv_red(const double2* x, Body body, const double2* staged, Gate g) {
        constexpr int NC = Body::kNC, NR = Body::kNR;
        const size_t extra = RedSmem<NC, NR>::kBytes;
        SellView v = sell_view(A, c, extra, Body::kSV);
        v.sv[0] = staged;
        const size_t smem = pipe_smem_bytes(v, extra);
        ZK_CUDA(cudaFuncSetAttribute(k_kspmv_red<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const RedCfg R{pc, pr, nullptr, nullptr, 0, slots};
        k_kspmv_red<Body><<<pg, kRedPipeThreads, smem, s>>>(v, x, body, R, g);
        check();
    }
    void spmv(const double2* x, double2* y, double2* y2, Gate g) {
        SellView v = sell_view(A, c, 0, 0);
        const unsigned grid = plain_grid(A, v);
        if (v.narrow_w) {
            ZK_NARROW_ATTR(k_kspmv_narrow);
            ZK_NARROW_LAUNCH(k_kspmv_narrow, v, 1, s, v, x, KPlainBody{y, y2}, g);
            check();
            return;
        }
        const size_t smem = pipe_smem_bytes(v, 0);
        ZK_CUDA(cudaFuncSetAttribute(k_kspmv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_kspmv<<<grid, kPipeThreads, smem, s>>>(v, x, KPlainBody{y, y2}, g);
        check();
    }
    // op(v) = spmv(A, M.apply(v)) into out; identity M.apply is a copy (bitwise v)
    void op(const double2* vin, double2* out, Gate g) {
        const double2* src = vin;
        if (P->jacobi) {
            jac(vin, P->tmp, g);
            src = P->tmp;
        }
        spmv(src, out, nullptr, g);
    }
    void op_dot(const double2* vin, double2* out, Gate g) {  // + pivot = <r~, out>
        // plain SpMV + the engine's dot: the per-element terms and the plan
        // order are KDotBody's, and the pass costs less than a reducer warp
        op(vin, out, g);
        dot(P->rs, out, g);
    }
    void jac(const double2* vin, double2* out, Gate g) {
        k_jac<<<ew, kEwThreads, 0, s>>>(n, vin, P->minv, out, fma, g);
        check();
    }
    void dot(const double2* x, const double2* y, Gate g) {
        zdot_device(c, n, x, y, true, kBlock, ZK_MODE_BLOCKED, &P->st->dot, g);
        ++count;
    }
    void nrm(const double2* x, Gate g) {
        znorm2_device(c, n, x, kBlock, ZK_MODE_BLOCKED, &P->st->nrm, g);
        ++count;
    }
    void scalar(int32_t op, int32_t i, int32_t j, Gate g) {
        k_kscalar<<<1, 1, 0, s>>>(P->st, P->mr, op, i, j, g);
        check();
    }
    void pairs(const Pairs& p, Gate g) {
        if (p.n == 0) return;
        k_pairs<<<ew, kEwThreads, 0, s>>>(p, n, fma, g);
        check();
    }
    // y0 = A x0 and y1 = A x1 in one pass over a narrow matrix
    void spmv2(const double2* x0, const double2* x1, double2* y0, double2* y1, Gate g) {
        SellView v = sell_view(A, c, 0, 0);
        plain_grid(A, v);
        if (!v.narrow_w) throw ZkError{ZK_ERR_CUDA, "internal: two-vector SpMV needs a narrow matrix"};
        ZK_NARROW_ATTR(k_kspmv2_narrow);
        ZK_NARROW_LAUNCH(k_kspmv2_narrow, v, 2, s, v, x0, x1, KPlain2Body{y0, y1}, g);
        check();
    }
    template <int MODE>
    void true_res(Gate g) {  // A x into ax, then the residual pass (as the BiCGStab loop does)
        spmv(P->x, P->ax, nullptr, g);
        res_pass<MODE>(g);
    }
    template <int MODE>
    void res_pass(Gate g) {  // the residual pass over (b, ax)
        const double2* in[2] = {P->b, P->ax};
        const int8_t alias[2] = {0, 0};
        L1View v;
        size_t smem;
        unsigned grid;
        if (!l1_view(c, n, kReal, in, alias, 2, slots, nullptr, v, smem, grid))
            throw ZkError{ZK_ERR_CUDA, "level-1 engine geometry"};
        ZK_CUDA(cudaFuncSetAttribute(k_kres_pass<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_kres_pass<MODE><<<grid, kL1Threads, smem, s>>>(v, KResBody<MODE>{P->st, P->hist, fma}, fma, g);
        check();
    }
    void curx(Gate g) {
        k_curx<<<ew, kEwThreads, 0, s>>>(n, P->x0, P->acc, P->jacobi ? P->minv : nullptr, P->x, fma, g);
        check();
    }
};

void add_pair(Pairs& p, const double2* x, double2* y, const double2* ca, const double2* cb, int32_t flags) {
    if (p.n >= kMaxPairs) throw ZkError{ZK_ERR_PARAMETER, "internal: too many fused updates"};
    p.op[p.n++] = PairOp{x, y, ca, cb, flags};
}

// ---- BiCGSTAB(l) -------------------------------------------------------------------
void l_prologue(KLaunch& L) {
    KrylovPlan* P = L.P;
    const Gate always{&P->st->done, Gate::kAlways};
    L.spmv_red(P->x, KSetupBody{P->r[0], P->rs, nullptr, P->st, P->hist, KSV_BICGSTABL, L.fma}, P->b, always);
}

// One outer cycle (krylov.py:339-407).
void l_body(KLaunch& L) {
    KrylovPlan* P = L.P;
    KState* st = P->st;
    const int ell = P->ell;
    const Gate G = L.live();
    L.scalar(KO_L_CYCLE, 0, 0, G);
    for (int j = 0; j < ell; ++j) {
        L.dot(P->rs, P->r[j], G);  // rho' = <r~, r_j>
        L.scalar(KO_L_BETA, 0, j, G);
        Pairs pu{};
        for (int i = 0; i <= j; ++i) add_pair(pu, P->r[i], P->u[i], &st->beta, nullptr, PF_SCALE | PF_NEG_A);
        L.pairs(pu, G);                        // u_i = u_i * (-beta) + r_i
        L.op_dot(P->u[j], P->u[j + 1], G);     // u_{j+1} = A M^-1 u_j, pivot = <r~, u_{j+1}>
        L.scalar(KO_L_ALPHA, 0, j, G);
        Pairs pr{};
        for (int i = 0; i <= j; ++i) add_pair(pr, P->u[i + 1], P->r[i], nullptr, &st->alpha, PF_NEG_B);
        add_pair(pr, P->u[0], P->acc, nullptr, &st->alpha, 0);
        L.pairs(pr, G);                        // r_i -= alpha u_{i+1}; acc += alpha u_0
        L.op(P->r[j], P->r[j + 1], G);         // r_{j+1} = A M^-1 r_j
        L.nrm(P->r[0], G);
        L.scalar(KO_L_PROBE, 0, j, G);         // ||r_0|| / ||b|| <= tol ?
        L.curx(L.onfl());                      // x = x0 + M^-1 acc
        L.true_res<0>(L.onfl());               // converged -> record, stop
    }
    for (int j = 1; j <= ell; ++j) {  // modified Gram-Schmidt (krylov.py:369-378)
        for (int i = 1; i < j; ++i) {
            L.dot(P->r[i], P->r[j], G);
            L.scalar(KO_L_TAU, i, j, G);
            Pairs pt{};
            add_pair(pt, P->r[i], P->r[j], nullptr, &P->mr->tau[i * (kMaxEll + 1) + j], PF_NEG_B);
            L.pairs(pt, G);
        }
        L.dot(P->r[j], P->r[j], G);
        L.scalar(KO_L_SIGMA, 0, j, G);
        L.dot(P->r[j], P->r[0], G);
        L.scalar(KO_L_GAMMAP, 0, j, G);
    }
    L.scalar(KO_L_GAMMA, ell, 0, G);
    MrVecs V{};
    for (int k = 0; k <= ell; ++k) {
        V.r[k] = P->r[k];
        V.u[k] = P->u[k];
    }
    k_mr_update<<<L.ew, kEwThreads, 0, L.s>>>(V, ell, L.n, P->acc, P->mr, L.fma, G);
    L.check();
    L.curx(G);
    L.true_res<1>(G);
}

// ---- TFQMR ---------------------------------------------------------------------------
void t_prologue(KLaunch& L) {
    KrylovPlan* P = L.P;
    const Gate always{&P->st->done, Gate::kAlways};
    L.spmv_red(P->x, KSetupBody{P->w, P->y, P->rs, P->st, P->hist, KSV_TFQMR, L.fma}, P->b, always);
    const Gate G = L.live();
    if (P->jacobi) L.jac(P->y, P->z, G);             // z = M y
    L.spmv(P->z, P->U[0], P->v, G);                    // uvec = A z; v = uvec.copy()
}

// One iteration (krylov.py:438-489) with uvec in U[p] and the next one in U[1-p].
void t_iteration(KLaunch& L, int p) {
    KrylovPlan* P = L.P;
    KState* st = P->st;
    const Gate G = L.live(), H = L.nofl();
    double2* Uc = P->U[p];
    double2* Un = P->U[1 - p];
    L.dot(P->rs, P->v, G);  // sigma
    L.scalar(KO_T_ALPHA, 0, 0, G);
    for (int half = 0; half < 2; ++half) {
        const Gate g = half == 0 ? G : H;
        if (half == 1) {
            if (!L.fuse2) {
                Pairs py{};
                add_pair(py, P->v, P->y, nullptr, &st->alpha, PF_NEG_B);
                L.pairs(py, g);                          // y -= alpha v
                if (P->jacobi) L.jac(P->y, P->z, g);     // z = M y
                L.spmv(P->z, Uc, nullptr, g);            // uvec = A z
            }
            L.scalar(KO_T_COEFD, 0, 0, g);
        }
        Pairs pw{};
        add_pair(pw, Uc, P->w, nullptr, &st->alpha, PF_NEG_B);              // w -= alpha uvec
        add_pair(pw, P->z, P->d, &st->coefd, nullptr, PF_SCALE);             // d = d * coef + z
        L.pairs(pw, g);
        L.nrm(P->w, g);
        L.scalar(KO_T_THETA, 0, 0, g);
        Pairs px{};
        add_pair(px, P->d, P->x, nullptr, &st->eta, 0);                      // x += eta d
        L.pairs(px, g);
        if (half == 1 && L.fuse2) {
            // ... and the end of the iteration's rho', beta, y, z ahead of the
            // second residual (the rho check stays after the record, below), so
            // A x and the next uvec = A z share one pass too
            L.dot(P->rs, P->w, g);  // rho'
            L.scalar(KO_T_BETA_CALC, 0, 0, g);
            Pairs py{};
            add_pair(py, P->w, P->y, &st->beta, nullptr, PF_SCALE);          // y = y * beta + w
            L.pairs(py, g);
            if (P->jacobi) L.jac(P->y, P->z, g);
            L.spmv2(P->x, P->z, P->ax, Un, g);       // A x (residual), uvec' = A M^-1 y
            L.res_pass<2>(g);
        } else if (half == 0 && L.fuse2) {
            // narrow matrix: the second half-step's y, z updates move ahead of the
            // first half-step's residual (they read v, alpha and y only; if the
            // residual converges they are dead, as in the reference's break), so
            // A x and the second half-step's A z share one matrix pass
            Pairs py{};
            add_pair(py, P->v, P->y, nullptr, &st->alpha, PF_NEG_B);
            L.pairs(py, g);                          // y -= alpha v
            if (P->jacobi) L.jac(P->y, P->z, g);     // z = M y
            L.spmv2(P->x, P->z, P->ax, Uc, g);       // A x (residual), uvec = A z
            L.res_pass<2>(g);
        } else {
            L.true_res<2>(g);
        }
    }
    k_krecord<<<1, 1, 0, L.s>>>(st, P->hist, G);
    L.check();
    if (L.fuse2) {
        L.scalar(KO_T_BETA_CHK, 0, 0, G);
    } else {
        L.dot(P->rs, P->w, G);  // rho'
        L.scalar(KO_T_BETA, 0, 0, G);
        Pairs py{};
        add_pair(py, P->w, P->y, &st->beta, nullptr, PF_SCALE);              // y = y * beta + w
        L.pairs(py, G);
        if (P->jacobi) L.jac(P->y, P->z, G);
        L.spmv(P->z, Un, nullptr, G);                                        // uvec' = A M^-1 y
    }
    k_tf_v<<<L.ew, kEwThreads, 0, L.s>>>(L.n, P->v, Uc, Un, st, L.fma, G);
    L.check();
    L.scalar(KO_T_END, 0, 0, G);
}

void t_body(KLaunch& L) {
    t_iteration(L, 0);
    t_iteration(L, 1);
}

template <class T>
T* kalloc(zk_context* c, size_t count) {
    return static_cast<T*>(c->alloc.alloc(sizeof(T) * (count ? count : 1)));
}

}  // namespace

void destroy_krylov_plan(zk_context* c, KrylovPlan* P) {
    if (!P) return;
    if (P->exec) cudaGraphExecDestroy(P->exec);
    if (P->graph) cudaGraphDestroy(P->graph);
    void* ptrs[] = {P->x, P->x0, P->b, P->minv, P->rs, P->tmp, P->ax, P->acc, P->w, P->y, P->d, P->v, P->U[0],
                    P->U[1], P->hist, P->st, P->mr};
    for (void* p : ptrs)
        if (p) c->alloc.free(p);
    if (P->jacobi && P->z) c->alloc.free(P->z);
    for (int k = 0; k <= kMaxEll; ++k) {
        if (P->r[k]) c->alloc.free(P->r[k]);
        if (P->u[k]) c->alloc.free(P->u[k]);
    }
    delete P;
}

static KrylovPlan* get_kplan(zk_context* c, zk_csr* A, int32_t solver, int32_t ell, bool jacobi, int64_t maxit) {
    KrylovPlan*& slot = A->kplan[solver * 2 + (jacobi ? 1 : 0)];
    if (slot && (slot->hist_cap < maxit + 1 || (solver == KSV_BICGSTABL && slot->ell != ell))) {
        destroy_krylov_plan(c, slot);
        slot = nullptr;
    }
    if (slot) return slot;
    KrylovPlan* P = new KrylovPlan();
    const int64_t n = A->n_rows;
    P->solver = solver;
    P->ell = ell;
    P->jacobi = jacobi;
    P->n = n;
    P->hist_cap = maxit + 1 > 1024 ? maxit + 1 : 1024;
    auto vec = [&]() { return kalloc<double2>(c, (size_t)n); };
    P->x = vec();
    P->x0 = vec();
    P->b = vec();
    P->rs = vec();
    P->ax = vec();
    P->minv = jacobi ? vec() : nullptr;
    P->tmp = jacobi ? vec() : nullptr;
    if (solver == KSV_BICGSTABL) {
        for (int k = 0; k <= ell; ++k) {
            P->r[k] = vec();
            P->u[k] = vec();
        }
        P->acc = vec();
    } else {
        P->w = vec();
        P->y = vec();
        P->d = vec();
        P->v = vec();
        P->U[0] = vec();
        P->U[1] = vec();
        P->z = jacobi ? vec() : P->y;  // identity: z = M.apply(y) is y, bitwise
    }
    P->hist = kalloc<double>(c, (size_t)P->hist_cap);
    P->st = kalloc<KState>(c, 1);
    P->mr = kalloc<KMr>(c, 1);
    ZK_CUDA(cudaMemsetAsync(P->mr, 0, sizeof(KMr), c->stream));
    slot = P;
    return P;
}

static void build_kgraph(zk_context* c, const zk_csr* A, KrylovPlan* P) {
    KLaunch L{c, A, P, c->fma != 0, P->n, 0, 0, {}, {}, nullptr, 0, c->stream};
    int64_t ewg = (P->n + kEwThreads - 1) / kEwThreads;
    const int64_t cap = (int64_t)num_sms() * 8;
    L.ew = (unsigned)(ewg < 1 ? 1 : (ewg > cap ? cap : ewg));
    L.pg = pipe_grid(A);
    {
        // ZK_FUSE2=0: no two-vector SpMV (A/B)
        SellView v = sell_view(A, c, 0, 0);
        plain_grid(A, v);
        const char* e = std::getenv("ZK_FUSE2");
        L.fuse2 = v.narrow_w != 0 && !(e && e[0] == '0');
    }
    // everything that may allocate or upload happens before the capture
    L.pc = c->plans_for(P->n, kBlock, kComplex);
    L.pr = c->plans_for(P->n, kBlock, kReal);
    const int64_t nb = (P->n + kBlock - 1) / kBlock;
    L.slots = fold_slots(c, 4 * (nb ? nb : 1));
    ZK_CUDA(cudaStreamSynchronize(c->stream));
    cudaStream_t s = c->stream;
    cudaGraph_t g;
    ZK_CUDA(cudaGraphCreate(&g, 0));
    cudaGraph_t gp;
    ZK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    if (P->solver == KSV_BICGSTABL) l_prologue(L);
    else t_prologue(L);
    ZK_CUDA(cudaStreamEndCapture(s, &gp));
    P->prologue_kernels = L.count;
    L.count = 0;
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
    if (P->solver == KSV_BICGSTABL) l_body(L);
    else t_body(L);
    k_kloop_end<<<1, 1, 0, s>>>(P->st, cond);
    L.check();
    cudaGraph_t body_out;
    ZK_CUDA(cudaStreamEndCapture(s, &body_out));
    P->body_kernels = L.count;
    ZK_CUDA(cudaGraphInstantiate(&P->exec, g, 0));
    P->graph = g;
}

// Runs one solve.  Returns ZK_OK or ZK_ERR_BREAKDOWN; report->breakdown is the
// ZK_BD_* code (and report_j the basis-vector index for ZK_BD_MR).
int krylov_device(zk_context* c, zk_csr* A, int solver, int ell, const double2* b, const double2* minv,
                  const double2* x0, double tol, int64_t maxit, double2* x_out, double* history_host,
                  zk_solve_report* rep, int32_t* what_j) {
    if (ell > kMaxEll) throw ZkError{ZK_ERR_PARAMETER, "polynomial degree l above " + std::to_string(kMaxEll)};
    const int64_t n = A->n_rows;
    KrylovPlan* P = get_kplan(c, A, solver, solver == KSV_BICGSTABL ? ell : 0, minv != nullptr, maxit);
    const bool fma = c->fma != 0, swap = A->nnz_elide * 16 >= c->elide_bytes;
    if (P->exec && (P->graph_fma != fma || P->graph_swap != swap)) {  // captured with another fingerprint
        cudaGraphExecDestroy(P->exec);
        cudaGraphDestroy(P->graph);
        P->exec = nullptr;
        P->graph = nullptr;
    }
    cudaStream_t s = c->stream;
    const size_t vb = sizeof(double2) * (size_t)n;
    ZK_CUDA(cudaMemcpyAsync(P->b, b, vb, cudaMemcpyDeviceToDevice, s));
    if (minv) ZK_CUDA(cudaMemcpyAsync(P->minv, minv, vb, cudaMemcpyDeviceToDevice, s));
    if (x0) ZK_CUDA(cudaMemcpyAsync(P->x0, x0, vb, cudaMemcpyDeviceToDevice, s));
    else ZK_CUDA(cudaMemsetAsync(P->x0, 0, vb, s));
    ZK_CUDA(cudaMemcpyAsync(P->x, P->x0, vb, cudaMemcpyDeviceToDevice, s));
    if (solver == KSV_BICGSTABL) {
        for (int k = 0; k <= ell; ++k) ZK_CUDA(cudaMemsetAsync(P->u[k], 0, vb, s));
        ZK_CUDA(cudaMemsetAsync(P->acc, 0, vb, s));
    } else {
        ZK_CUDA(cudaMemsetAsync(P->d, 0, vb, s));
    }
    KState h;
    std::memset(&h, 0, sizeof(h));
    h.tol = tol;
    h.maxit = maxit;
    ZK_CUDA(cudaMemcpyAsync(P->st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    if (!P->exec) {
        build_kgraph(c, A, P);
        P->graph_fma = fma;
        P->graph_swap = swap;
    }
    ZK_CUDA(cudaGraphLaunch(P->exec, s));
    KState out;
    ZK_CUDA(cudaMemcpyAsync(&out, P->st, sizeof(out), cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    const int64_t launches = P->prologue_kernels + P->body_kernels * out.trips;
    c->launches += launches;
    const int64_t it = out.iterations;
    ZK_CUDA(cudaMemcpyAsync(history_host, P->hist, sizeof(double) * (it + 1), cudaMemcpyDeviceToHost, s));
    if (out.trivial) ZK_CUDA(cudaMemsetAsync(x_out, 0, vb, s));
    else ZK_CUDA(cudaMemcpyAsync(x_out, P->x, vb, cudaMemcpyDeviceToDevice, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    rep->iterations = it;
    rep->converged = out.status == KS_CONVERGED;
    rep->breakdown = out.status == KS_BREAKDOWN ? out.what : 0;
    rep->final_relative_residual = history_host[it];
    rep->history_len = it + 1;
    rep->kernel_launches = launches;
    *what_j = out.what_j;
    return out.status == KS_BREAKDOWN ? ZK_ERR_BREAKDOWN : ZK_OK;
}

}  // namespace zk
