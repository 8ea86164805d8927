// zk_spmv.cuh -- SELL-32 complex128 SpMV engine (device side, sm_100a).
//
// Layout (built once per matrix by zk_csr_create, zk_spmv.cu): rows are cut
// into 32-row slices; slice s stores its rows column-major, element k of
// slice-row r at aa[slice_off[s] + 32*k + r] (double2) and ja[...] (int32),
// padded to the slice's longest row.  A slice is therefore two contiguous
// chunks (32*W*16 B of values, 32*W*4 B of column indices).  Rows longer than
// 65 entries ("long rows", absent from stencil and FE matrices) live in a
// side CSR and are summed by one thread with the full pairwise recursion.
//
// Pipeline (the matrix is the HBM stream; everything else is cache-resident):
// kernels are persistent, one CTA per SM, 8 consumer warps + 1 producer warp.
// The producer's elected lane streams the CTA's slices into a shared-memory
// ring with 1-D TMA bulk copies (cp.async.bulk, L2 evict-first so the
// streamed matrix does not push x out of L2), each stage guarded by a
// full/empty mbarrier pair; so up to NS x 17 KB of matrix is in flight per SM
// without costing a register.  Consumer warp w takes every 8th slice of the
// current 4096-row block, one thread per row, gathers x through L1/L2 with
// one group of products prefetched ahead, and hands each row value to the
// kernel's epilogue.  After a block's rows are done the consumer warps run
// the block's fused reduction (named barrier 1) while the producer keeps
// prefetching the next block.
//
// Arithmetic (sparse.py:217-232 + numpy): the product of
// entry k is F1(aa_k, x[ja_k]) -- or F1(x[ja_k], aa_k) once numpy's
// temporary elision kicks in (nnz*16 >= 256 KiB) -- and a row with L
// entries sums as v0 + PW(v1..v_{L-1}); for L-1 <= 64 that is one pairwise
// leaf: four lane accumulators over full groups of four, (l0+l1)+(l2+l3),
// then the leftovers in order.  One thread evaluates exactly that sequence
// in registers, so results do not depend on the launch geometry.
#pragma once
#include "zk_common.cuh"
#include "zk_pipe.cuh"

namespace zk {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;  // 256
constexpr int kPipeThreads = kConsumers + 32;    // + producer warp
constexpr int kMaxStages = 32;
constexpr int kBarBytes = 2 * kMaxStages * 8;
constexpr int kSmemLimit = 227 * 1024;

struct SellView {
    int64_t n_rows, n_cols, nslices, nblocks;
    const double2* __restrict__ aa;
    const int32_t* __restrict__ ja;
    const int64_t* __restrict__ slice_off;
    const uint8_t* __restrict__ rowlen;
    const int32_t* __restrict__ long_row;
    const int32_t* __restrict__ long_blk_ptr;
    const int64_t* __restrict__ long_ia;
    const int32_t* __restrict__ long_ja;
    const double2* __restrict__ long_aa;
    int32_t stage_bytes;  // ring stage size (widest slice of the matrix, 128 B rounded)
    int32_t ja_off;       // byte offset of the column indices inside a stage
    int32_t ns;           // ring stages for this launch (a multiple of cw)
    int32_t cw;           // consumer warps that take slices (stage st is only ever read by warp st % cw)
    bool swap;            // numpy elided the gathered temporary: prod = F1(x[ja], aa)
    bool fma;
};

__device__ __forceinline__ double2 spmv_prod(const SellView& A, double2 a, double2 xv) {
    return A.swap ? f1(xv, a, A.fma) : f1(a, xv, A.fma);
}

// Row sum of a short row from a ring stage (element k at [32*k + lane]).
__device__ __forceinline__ double2 stage_row(const SellView& A, const double2* __restrict__ x,
                                             const double2* saa, const int32_t* sja, int lane, int len) {
    if (len == 0) return make_double2(0.0, 0.0);
    double2 v0 = spmv_prod(A, saa[lane], __ldg(x + sja[lane]));
    const int L = len - 1;
    if (L == 0) return v0;
    double2 s;
    if (L < 4) {
        s = make_double2(-0.0, -0.0);
        for (int k = 1; k <= L; ++k) s = cadd(s, spmv_prod(A, saa[32 * k + lane], __ldg(x + sja[32 * k + lane])));
        return cadd(v0, s);
    }
    const int G = L >> 2;
    double2 cx[4], r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) cx[q] = __ldg(x + sja[32 * (1 + q) + lane]);
    for (int g = 0; g < G; ++g) {
        double2 nx[4];
        const int kn = 1 + 4 * (g + 1);
        if (g + 1 < G) {
#pragma unroll
            for (int q = 0; q < 4; ++q) nx[q] = __ldg(x + sja[32 * (kn + q) + lane]);
        }
        const int kc = 1 + 4 * g;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double2 p = spmv_prod(A, saa[32 * (kc + q) + lane], cx[q]);
            r[q] = (g == 0) ? p : cadd(r[q], p);
        }
        if (g + 1 < G) {
#pragma unroll
            for (int q = 0; q < 4; ++q) cx[q] = nx[q];
        }
    }
    s = cadd(cadd(r[0], r[1]), cadd(r[2], r[3]));
    for (int k = 1 + 4 * G; k <= L; ++k) s = cadd(s, spmv_prod(A, saa[32 * k + lane], __ldg(x + sja[32 * k + lane])));
    return cadd(v0, s);
}

__device__ __forceinline__ double2 long_prod(const SellView& A, const double2* __restrict__ x, int64_t idx) {
    return spmv_prod(A, A.long_aa[idx], __ldg(x + A.long_ja[idx]));
}

// numpy CDOUBLE_pairwise_sum over products [s, s+L) of the side CSR.
static __device__ double2 long_pw(const SellView& A, const double2* __restrict__ x, int64_t s, int64_t L) {
    if (L < 4) {
        double2 acc = make_double2(-0.0, -0.0);
        for (int64_t k = 0; k < L; ++k) acc = cadd(acc, long_prod(A, x, s + k));
        return acc;
    }
    if (L <= 64) {
        double2 r0 = long_prod(A, x, s), r1 = long_prod(A, x, s + 1);
        double2 r2 = long_prod(A, x, s + 2), r3 = long_prod(A, x, s + 3);
        const int64_t G = L / 4;
        for (int64_t g = 1; g < G; ++g) {
            r0 = cadd(r0, long_prod(A, x, s + 4 * g));
            r1 = cadd(r1, long_prod(A, x, s + 4 * g + 1));
            r2 = cadd(r2, long_prod(A, x, s + 4 * g + 2));
            r3 = cadd(r3, long_prod(A, x, s + 4 * g + 3));
        }
        double2 acc = cadd(cadd(r0, r1), cadd(r2, r3));
        for (int64_t k = 4 * G; k < L; ++k) acc = cadd(acc, long_prod(A, x, s + k));
        return acc;
    }
    const int64_t h = (L - L % 8) / 2;
    double2 a = long_pw(A, x, s, h);
    double2 b = long_pw(A, x, s + h, L - h);
    return cadd(a, b);
}

__device__ __forceinline__ double2 long_row_sum(const SellView& A, const double2* __restrict__ x, int li) {
    const int64_t lo = A.long_ia[li], L = A.long_ia[li + 1] - lo;
    double2 v0 = long_prod(A, x, lo);
    return cadd(v0, long_pw(A, x, lo + 1, L - 1));
}

// Persistent pipelined SpMV over the CTA's 4096-row blocks (blk = blockIdx.x,
// +gridDim.x, ...).  body.row(row, value) is called once per row by the
// consumer thread that computed it; body.block_done(blk) is called by all
// consumer threads after every row of the block is done (named barrier 1
// already passed).  The producer warp exits when it has issued every slice.
// `smem` points at kBarBytes + ns*stage_bytes bytes of dynamic shared memory.
template <class Body>
__device__ __forceinline__ void sell_pipeline(const SellView& A, const double2* __restrict__ x, Body& body,
                                              unsigned char* smem) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    unsigned char* ring = smem + kBarBytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ns = A.ns;
    constexpr int kSlicesPerBlock = kBlock / kSlice;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == kConsumerWarps) {  // producer
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int64_t i = 0;
            for (int64_t blk = blockIdx.x; blk < A.nblocks; blk += gridDim.x) {
                const int64_t s_lo = blk * kSlicesPerBlock;
                const int64_t s_hi = (s_lo + kSlicesPerBlock < A.nslices) ? s_lo + kSlicesPerBlock : A.nslices;
                for (int64_t s = s_lo; s < s_hi; ++s, ++i) {
                    const int st = (int)(i % ns);
                    const int64_t u = i / ns;
                    if (u) mbar_wait(&empty[st], (uint32_t)((u - 1) & 1));
                    const int64_t off0 = __ldg(A.slice_off + s);
                    const uint32_t cnt = (uint32_t)(__ldg(A.slice_off + s + 1) - off0);
                    mbar_arrive_expect_tx(&full[st], cnt * 20u);
                    if (cnt) {
                        unsigned char* stage = ring + (size_t)st * A.stage_bytes;
                        bulk_g2s(stage, A.aa + off0, cnt * 16u, &full[st], pol);
                        bulk_g2s(stage + A.ja_off, A.ja + off0, cnt * 4u, &full[st], pol);
                    }
                }
            }
        }
        return;
    }
    // Slice i of the CTA's sequence goes to stage i % ns and to warp i % cw.
    // Because ns is a multiple of cw, every stage has exactly one consumer
    // warp and that warp meets the stage's uses in order -- required by the
    // parity wait, which cannot tell use u from use u+2.
    const int cw = A.cw;
    int64_t ibase = 0;
    for (int64_t blk = blockIdx.x; blk < A.nblocks; blk += gridDim.x) {
        const int64_t s_lo = blk * kSlicesPerBlock;
        const int64_t s_hi = (s_lo + kSlicesPerBlock < A.nslices) ? s_lo + kSlicesPerBlock : A.nslices;
        const int nsl = (int)(s_hi - s_lo);
        const int j0 = warp < cw ? (int)(((int64_t)warp - ibase % cw + cw) % cw) : nsl;
        for (int j = j0; j < nsl; j += cw) {
            const int64_t i = ibase + j;
            const int st = (int)(i % ns);
            const int64_t row = (s_lo + j) * kSlice + lane;
            const int len = A.rowlen[row];
            mbar_wait(&full[st], (uint32_t)((i / ns) & 1));
            const unsigned char* stage = ring + (size_t)st * A.stage_bytes;
            if (row < A.n_rows && len != 255) {
                double2 v = stage_row(A, x, reinterpret_cast<const double2*>(stage),
                                      reinterpret_cast<const int32_t*>(stage + A.ja_off), lane, len);
                body.row(row, v);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        ibase += nsl;
        if (A.long_blk_ptr) {
            const int lb = A.long_blk_ptr[blk], le = A.long_blk_ptr[blk + 1];
            for (int li = lb + (int)threadIdx.x; li < le; li += kConsumers)
                body.row((int64_t)A.long_row[li], long_row_sum(A, x, li));
        }
        named_sync(1, kConsumers);
        body.block_done(blk);
    }
}

}  // namespace zk
