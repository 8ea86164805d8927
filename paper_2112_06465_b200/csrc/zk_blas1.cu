// zk_blas1.cu -- level-1 kernels (vecops.py:117-200) for sm_100a.
//
// Elementwise kernels are HBM-bound streams: grid-stride over double2
// (16-byte, coalesced) with 4 independent elements per thread in flight.
// Reductions run one CTA per ReductionPlan block (numpy's pairwise order,
// zk_blockred.cuh) and a one-warp kernel folds the block partials in order.
#include <cstdlib>
#include <cstring>

#include "zk_internal.h"
#include "zk_blockred.cuh"
#include "zk_l1pipe.cuh"

namespace zk {

namespace {

constexpr int kEwThreads = 256;
constexpr int kEwUnroll = 4;

inline int ew_grid(int64_t n) {
    int64_t per = (int64_t)kEwThreads * kEwUnroll;
    int64_t g = (n + per - 1) / per;
    int64_t cap = (int64_t)num_sms() * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

template <class F>
__device__ __forceinline__ void ew_loop(int64_t n, F f) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (kEwUnroll - 1) * stride < n; i += kEwUnroll * stride) {
#pragma unroll
        for (int u = 0; u < kEwUnroll; ++u) f(i + u * stride);
    }
    for (; i < n; i += stride) f(i);
}

__global__ void k_zscal(int64_t n, double2 a, double2* __restrict__ x, bool fma) {
    ew_loop(n, [&](int64_t i) { x[i] = f1(x[i], a, fma); });
}

__global__ void k_zaxpy(int64_t n, double2 a, const double2* __restrict__ x, double2* __restrict__ y, bool fma) {
    ew_loop(n, [&](int64_t i) { y[i] = cadd(y[i], f1(a, ldg2(x + i), fma)); });
}

__global__ void k_zaxmy(int64_t n, const double2* __restrict__ x, double2* __restrict__ y, bool fma) {
    ew_loop(n, [&](int64_t i) { y[i] = f1(y[i], ldg2(x + i), fma); });
}

__global__ void k_jacobi(int64_t n, const double2* __restrict__ v, const double2* __restrict__ m,
                         double2* __restrict__ out, bool fma) {
    ew_loop(n, [&](int64_t i) { out[i] = f1(ldg2(v + i), ldg2(m + i), fma); });
}

constexpr int kRedThreads = 288;  // 65 complex / 33 real leaves x lanes fit one pass

struct DotOp {
    const double2* __restrict__ x;
    const double2* __restrict__ y;
    bool conj, fma;
    struct Item { double2 x, y; };
    static constexpr int U = 8;
    __device__ Item load(int64_t e) const { return {__ldg(x + e), __ldg(y + e)}; }
    __device__ void apply(int64_t, const Item& it, double2 (&v)[1]) const {
        double2 a = it.x;
        if (conj) a.y = -a.y;  // np.conj
        v[0] = f1(a, it.y, fma);
    }
};

struct Norm2Op {
    const double2* __restrict__ x;
    struct Item { double2 x; };
    static constexpr int U = 8;
    __device__ Item load(int64_t e) const { return {__ldg(x + e)}; }
    __device__ void apply(int64_t, const Item& it, double (&v)[1]) const { v[0] = abs2_np(it.x); }
};

// Block partials, one CTA per reduction block, and a streaming ordered fold.
// Every thread runs its (leaf, lane) items, then warp 0 alone combines the
// tree (__syncwarp only) and publishes the block's partial into its slot;
// the other warps exit.  The left fold of the partials (vecops.py:159-161)
// is a serial chain of nb dependent adds (~17 cycles each on B200,
// measured: ~180 us for 24414 blocks), so instead of a fold kernel after
// the pass, CTA 0's warp 0 folds WHILE the pass runs: it polls the slots in
// block order, adds each as it appears and re-marks it empty for the next
// call.  Only the last few partials are folded after the last CTA ends.
// No fence or atomic per CTA: each slot is its own flag, holding the empty
// marker (a signalling NaN, which arithmetic never produces -- results of
// NaN operands are quiet NaNs) until its value lands.  CTA 0 waits only for
// CTAs that need no resources it holds, so it cannot deadlock.
template <typename V, class Op>
__device__ __forceinline__ void block_partial(PlanPtrs plans, int64_t n, int64_t nb, int64_t block, const Op& op,
                                              V* nodes, double* slots, V* result, bool sqrt_result) {
    constexpr int NC = sizeof(V) / sizeof(double);
    const int64_t blk = blockIdx.x;
    const int64_t base = blk * block;
    const char* plan = (base + block <= n) ? plans.full : plans.tail;
    V v0[1];
    if (threadIdx.x == 0) {
        typename Op::Item it = op.load(base);
        op.apply(base, it, v0);
    }
    leaf_phase<V, 1>(plan, base + 1, op, nodes, blockDim.x);
    __syncthreads();
    if ((threadIdx.x >> 5) != 0) return;
    V pw[1];
    warp_tree<V, 1>(plan, nodes, pw);
    if ((threadIdx.x & 31) == 0) {
        const V p = plan_hdr(plan)->L > 0 ? VT<V>::add(v0[0], pw[0]) : v0[0];
        const double* pd = reinterpret_cast<const double*>(&p);
#pragma unroll
        for (int c = 0; c < NC; ++c) slot_store(slots + blk * NC + c, pd[c]);
    }
    if (blk != 0) return;
    double r[NC];
    stream_fold<NC>(slots, nb, r);
    if ((threadIdx.x & 31) == 0) {
        if constexpr (NC == 1) {
            *reinterpret_cast<double*>(result) = sqrt_result ? __dsqrt_rn(r[0]) : r[0];
        } else {
            *result = make_double2(r[0], r[1]);
        }
    }
}

__global__ void __launch_bounds__(kRedThreads, 2) k_zdot_blocks(int64_t n, int64_t nb, const double2* __restrict__ x,
                                                              const double2* __restrict__ y, bool conj, int64_t block,
                                                              PlanPtrs plans, double* slots, double2* result,
                                                              bool fma, Gate gate) {
    extern __shared__ double2 nodes_c[];
    if (gate.skip()) return;  // launch-uniform: every CTA returns, no slot is written
    block_partial<double2>(plans, n, nb, block, DotOp{x, y, conj, fma}, nodes_c, slots, result, false);
}

__global__ void __launch_bounds__(kRedThreads, 3) k_znorm2_blocks(int64_t n, int64_t nb, const double2* __restrict__ x,
                                                                int64_t block, PlanPtrs plans, double* slots,
                                                                double* result, Gate gate) {
    extern __shared__ double nodes_r[];
    if (gate.skip()) return;
    block_partial<double>(plans, n, nb, block, Norm2Op{x}, nodes_r, slots, result, true);
}

// ---- DEFAULT_PLAN (4096) reductions on the TMA-fed engine (zk_l1pipe.cuh) ----
struct DotPipeOp {
    using V = double2;
    static constexpr int NIN = 2;
    bool conj, fma;
    __device__ __forceinline__ double2 apply(int64_t, const double2 (&v)[2]) const {
        double2 a = v[0];
        if (conj) a.y = -a.y;  // np.conj
        return f1(a, v[1], fma);
    }
};

struct NormPipeOp {
    using V = double;
    static constexpr int NIN = 1;
    __device__ __forceinline__ double apply(int64_t, const double2 (&v)[1]) const { return abs2_np(v[0]); }
};

struct DotFin {
    static constexpr int kNP = 2;
    double2* result;
    __device__ void finish(const double* t) { *result = make_double2(t[0], t[1]); }
};

struct NormFin {
    static constexpr int kNP = 1;
    double* result;
    __device__ void finish(const double* t) { *result = __dsqrt_rn(t[0]); }
};

__global__ void __launch_bounds__(kL1Threads, 1) k_zdot_pipe(L1View P, DotPipeOp op, DotFin fin, Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    l1_pipeline(P, op, fin, smem);
}

__global__ void __launch_bounds__(kL1Threads, 1) k_znorm2_pipe(L1View P, NormPipeOp op, NormFin fin, Gate gate) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (gate.skip()) return;
    l1_pipeline(P, op, fin, smem);
}

__global__ void k_fill_empty(double* slots, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        slots[i] = __longlong_as_double((long long)kSlotEmpty);
}

// SEQUENTIAL plan (vecops.py:175-183): a CPython left-to-right loop with the
// plain (non-FMA) complex product, starting from 0j.  Correctness path only.
__global__ void k_zdot_seq(int64_t n, const double2* __restrict__ x, const double2* __restrict__ y, bool conj,
                           double2* result) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        double2 a = x[i];
        if (conj) a.y = -a.y;
        acc = cadd(acc, cmul_py(a, y[i]));
    }
    *result = acc;
}

// vecops.py:194-198: acc += re*re + im*im (Python floats), then math.sqrt.
__global__ void k_znorm2_seq(int64_t n, const double2* __restrict__ x, double* result) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, abs2_np(x[i]));
    *result = __dsqrt_rn(acc);
}

}  // namespace

void launch_zscal(zk_context* c, int64_t n, double2 a, double2* x) {
    if (n <= 0) return;
    k_zscal<<<ew_grid(n), kEwThreads, 0, c->stream>>>(n, a, x, c->fma);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

void launch_zaxpy(zk_context* c, int64_t n, double2 a, const double2* x, double2* y) {
    if (n <= 0) return;
    k_zaxpy<<<ew_grid(n), kEwThreads, 0, c->stream>>>(n, a, x, y, c->fma);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

void launch_zaxmy(zk_context* c, int64_t n, const double2* x, double2* y) {
    if (n <= 0) return;
    k_zaxmy<<<ew_grid(n), kEwThreads, 0, c->stream>>>(n, x, y, c->fma);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

void launch_jacobi(zk_context* c, int64_t n, const double2* v, const double2* m, double2* out) {
    if (n <= 0) return;
    k_jacobi<<<ew_grid(n), kEwThreads, 0, c->stream>>>(n, v, m, out, c->fma);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

int plan_nnodes(zk_context* c, int32_t L, int32_t kind);

// Slots for the streaming fold, all holding the empty marker between calls
// (the folder re-marks each slot it consumes).
double* fold_slots(zk_context* c, int64_t count) {
    if (count > c->slots_n) {
        if (c->slots) c->alloc.free(c->slots);
        c->slots = static_cast<double*>(c->alloc.alloc(sizeof(double) * count));
        c->slots_n = count;
        k_fill_empty<<<ew_grid(count), kEwThreads, 0, c->stream>>>(c->slots, count);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
    }
    return c->slots;
}

// Engine geometry for a DEFAULT_PLAN pass over n elements with the given
// staged inputs; false when the plans do not fit the engine (tail block with
// more stages than a full one), so the caller takes the block-per-CTA path.
bool l1_view(zk_context* c, int64_t n, int32_t kind, const double2* const* in, const int8_t* alias, int nin_op,
             double* slots, double* partials, L1View& P, size_t& smem, unsigned& grid, int vbytes, int fine) {
    if (n <= 0) return false;
    const PlanPtrs p = c->plans_for(n, kBlock, kind);
    const PlanHeader* hf = reinterpret_cast<const PlanHeader*>(c->plan_host(kBlock - 1, kind));
    const int64_t nb = (n + kBlock - 1) / kBlock;
    const int32_t tail_len = (int32_t)(n - (nb - 1) * kBlock) - 1;
    const PlanHeader* ht = reinterpret_cast<const PlanHeader*>(c->plan_host(tail_len, kind));
    int staged_inputs = 0;
    for (int v = 0; v < nin_op; ++v) staged_inputs += in[v] != nullptr;
    if (fine < 0) {
        // finer stages (half-size ring slots, twice as many in flight) for ops
        // that stage many vectors; ZK_L1FINE = 0 / 1 / 2: never / default / always
        const char* e = std::getenv("ZK_L1FINE");
        const int mode = e ? std::atoi(e) : 1;
        fine = mode == 2 ? 1 : (mode == 0 ? 0 : (staged_inputs >= 4 ? 1 : 0));
    }
    if (ht->nstages[fine] > hf->nstages[fine]) return false;
    std::memset(&P, 0, sizeof(P));
    P.n = n;
    P.nblocks = nb;
    P.plans = p;
    int staged = 0;
    for (int v = 0; v < nin_op; ++v) {
        P.in[v] = in[v];
        P.alias[v] = alias ? alias[v] : 0;
        if (in[v]) ++staged;
    }
    P.nin = staged;
    P.fine = fine;
    P.smax = fine ? kStageMaxElemsFine : kStageMaxElems;
    P.slot_bytes = staged * P.smax * 16;
    const size_t head = l1_head_bytes(vbytes ? vbytes : (kind == kComplex ? 16 : 8));
    const size_t limit = 227 * 1024 - kL1StaticSmem;
    int ns = (int)((limit - head) / (size_t)P.slot_bytes);
    if (ns > L1Smem<double>::kMaxSlots) ns = L1Smem<double>::kMaxSlots;
    if (ns < 2) return false;
    P.ns = ns;
    P.slots = slots;
    P.partials = partials;
    smem = head + (size_t)ns * P.slot_bytes;
    const int64_t g = nb < num_sms() ? nb : num_sms();
    grid = (unsigned)g;
    return true;
}

void zdot_device(zk_context* c, int64_t n, const double2* x, const double2* y, bool conj, int64_t block,
                 int mode, double2* result, Gate gate) {
    if (mode == ZK_MODE_BLOCKED && block == kBlock) {
        const int64_t nb = (n + kBlock - 1) / kBlock;
        const double2* in[2] = {x, x == y ? nullptr : y};
        const int8_t alias[2] = {0, 0};
        L1View P;
        size_t smem;
        unsigned grid;
        if (l1_view(c, n, kComplex, in, alias, 2, fold_slots(c, 2 * nb), nullptr, P, smem, grid)) {
            ZK_CUDA(cudaFuncSetAttribute(k_zdot_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_zdot_pipe<<<grid, kL1Threads, smem, c->stream>>>(P, DotPipeOp{conj, c->fma != 0}, DotFin{result}, gate);
            ZK_CUDA(cudaGetLastError());
            c->launches++;
            return;
        }
    }
    if (mode == ZK_MODE_SEQUENTIAL) {
        k_zdot_seq<<<1, 1, 0, c->stream>>>(n, x, y, conj, result);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
        return;
    }
    int64_t nb = (n + block - 1) / block;
    PlanPtrs p = c->plans_for(n, block, kComplex);
    int nnodes = plan_nnodes(c, (int32_t)(block - 1), kComplex);
    int tail = (int32_t)(n - (nb - 1) * block) - 1;
    int nn2 = plan_nnodes(c, tail, kComplex);
    if (nn2 > nnodes) nnodes = nn2;
    const size_t smem = (size_t)nnodes * sizeof(double2);
    double* slots = fold_slots(c, 2 * nb);
    if (smem > 48 * 1024)
        ZK_CUDA(cudaFuncSetAttribute(k_zdot_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_zdot_blocks<<<(unsigned)nb, kRedThreads, smem, c->stream>>>(n, nb, x, y, conj, block, p, slots, result, c->fma,
                                                                  gate);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

void znorm2_device(zk_context* c, int64_t n, const double2* x, int64_t block, int mode, double* result, Gate gate) {
    if (mode == ZK_MODE_BLOCKED && block == kBlock) {
        const int64_t nb = (n + kBlock - 1) / kBlock;
        const double2* in[1] = {x};
        L1View P;
        size_t smem;
        unsigned grid;
        if (l1_view(c, n, kReal, in, nullptr, 1, fold_slots(c, nb), nullptr, P, smem, grid)) {
            ZK_CUDA(cudaFuncSetAttribute(k_znorm2_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_znorm2_pipe<<<grid, kL1Threads, smem, c->stream>>>(P, NormPipeOp{}, NormFin{result}, gate);
            ZK_CUDA(cudaGetLastError());
            c->launches++;
            return;
        }
    }
    if (mode == ZK_MODE_SEQUENTIAL) {
        k_znorm2_seq<<<1, 1, 0, c->stream>>>(n, x, result);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
        return;
    }
    int64_t nb = (n + block - 1) / block;
    PlanPtrs p = c->plans_for(n, block, kReal);
    int nnodes = plan_nnodes(c, (int32_t)(block - 1), kReal);
    int tail = (int32_t)(n - (nb - 1) * block) - 1;
    int nn2 = plan_nnodes(c, tail, kReal);
    if (nn2 > nnodes) nnodes = nn2;
    const size_t smem = (size_t)nnodes * sizeof(double);
    double* slots = fold_slots(c, nb);
    if (smem > 48 * 1024)
        ZK_CUDA(cudaFuncSetAttribute(k_znorm2_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_znorm2_blocks<<<(unsigned)nb, kRedThreads, smem, c->stream>>>(n, nb, x, block, p, slots, result, gate);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

}  // namespace zk
