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

constexpr int kConsumerWarps = 7;  // + 1 producer = 8 warps: 2 per SMSP, so up to 255 registers/thread
constexpr int kConsumers = kConsumerWarps * 32;  // 256
constexpr int kPipeThreads = kConsumers + 32;    // + producer warp
constexpr int kMaxStages = 32;
constexpr int kBarBytes = 2 * kMaxStages * 8 + 2 * kMaxStages * 4;  // full, empty mbarriers + stage tags, widths
constexpr int kSmemLimit = 227 * 1024;
constexpr int kFullCols = 33;  // widest row handled by the whole-row prefetch path
// Reduction windows: 28 slices (4 per consumer warp, 896 rows).  With a
// 2048-row stash ring a window never overwrites rows a pending leaf (<= 128
// elements) or the previous window's leaf pass still reads (896*2+128 < 2048).
constexpr int kWindowSlices = 4 * kConsumerWarps;
constexpr int kStashRows = 2048;

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
    int32_t cm;           // pairwise groups (4 columns each) per ring chunk; 0 = whole slice per stage
    int32_t nch;          // chunks per slice (from the widest slice)
    int32_t stage_bytes;  // (1 + 4 cm) columns x 32 rows x 20 B, 128 B rounded
    int32_t ja_off;       // byte offset of the column indices inside a stage
    int32_t rl_off;       // byte offset of the slice's 32 row lengths inside a stage (cm == 0)
    int32_t ns;           // ring stages for this launch
    uint32_t ns_magic;    // floor(2^32 / ns) + 1: i / ns = umulhi(i, ns_magic) for i < 2^27
    int32_t win;          // slices per reduction window (kWindowSlices, or a whole block with long rows)
    bool swap;            // numpy elided the gathered temporary: prod = F1(x[ja], aa)
    bool fma;
};

__device__ __forceinline__ double2 spmv_prod(const SellView& A, double2 a, double2 xv) {
    return A.swap ? f1(xv, a, A.fma) : f1(a, xv, A.fma);
}

// Per-row accumulator of numpy's order, fed chunk by chunk (chunk c holds
// columns [c0, c1) of the slice; chunk boundaries sit on pairwise-group
// boundaries, so a group of four never straddles two chunks).
struct RowAcc {
    double2 v0, r0, r1, r2, r3, s;
    int L, G;
    bool combined;

    __device__ __forceinline__ void init(int len) {
        L = len - 1;
        G = L >= 4 ? (L >> 2) : 0;
        combined = false;
        s = make_double2(-0.0, -0.0);
    }

    // saa/sja: the chunk's stage; element (k - c0) of this lane's row at [32*(k-c0) + lane]
    __device__ __forceinline__ void chunk(const SellView& A, const double2* __restrict__ x, const double2* saa,
                                          const int32_t* sja, int lane, int c, int c0) {
        const int len = L + 1;
        if (len <= 0) return;
        auto prod = [&](int k) {
            const int e = 32 * (k - c0) + lane;
            return spmv_prod(A, saa[e], __ldg(x + sja[e]));
        };
        if (c == 0) v0 = prod(0);
        if (L < 4) {  // sequential from -0.0 (2L < 8); len <= 4 <= 1+4cm: all in chunk 0
            if (c == 0)
                for (int k = 1; k <= L; ++k) s = cadd(s, prod(k));
            return;
        }
        const int g_lo = (c == 0) ? 0 : A.cm * c;
        const int g_hi = A.cm * (c + 1);
        int g = g_lo;
        if (g < G) {
            double2 cx[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) cx[q] = __ldg(x + sja[32 * (1 + 4 * g + q - c0) + lane]);
            for (; g < g_hi && g < G; ++g) {
                double2 nx[4];
                const bool more = (g + 1 < g_hi) && (g + 1 < G);
                if (more) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) nx[q] = __ldg(x + sja[32 * (5 + 4 * g + q - c0) + lane]);
                }
                const int kb = 32 * (1 + 4 * g - c0) + lane;
                const double2 p0 = spmv_prod(A, saa[kb], cx[0]);
                const double2 p1 = spmv_prod(A, saa[kb + 32], cx[1]);
                const double2 p2 = spmv_prod(A, saa[kb + 64], cx[2]);
                const double2 p3 = spmv_prod(A, saa[kb + 96], cx[3]);
                if (g == 0) {
                    r0 = p0; r1 = p1; r2 = p2; r3 = p3;
                } else {
                    r0 = cadd(r0, p0); r1 = cadd(r1, p1); r2 = cadd(r2, p2); r3 = cadd(r3, p3);
                }
                if (more) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) cx[q] = nx[q];
                }
            }
        }
        if (G >= g_lo && G < g_hi) {  // this chunk holds the end of the full groups: combine, add leftovers
            s = cadd(cadd(r0, r1), cadd(r2, r3));
            combined = true;
            for (int k = 1 + 4 * G; k <= L; ++k) s = cadd(s, prod(k));
        }
    }

    // Whole row in one chunk (width <= kFullCols).  The row's x gathers are
    // issued in two batches (v0 + groups 0..3, then groups 4..7 and the
    // leftovers), each batch fully in flight before its first product: two
    // L1/L2 round trips per row instead of one per group.
    __device__ __forceinline__ void full_row(const SellView& A, const double2* __restrict__ x, const double2* saa,
                                             const int32_t* sja, int lane) {
        const int len = L + 1;
        if (len <= 0) return;
        double2 xs[17];
#pragma unroll
        for (int k = 0; k < 17; ++k)
            if (k < len) xs[k] = __ldg(x + sja[32 * k + lane]);
        asm volatile("" ::: "memory");  // keep the value loads below the gathers (register pressure)
        v0 = spmv_prod(A, saa[lane], xs[0]);
        if (L < 4) {
#pragma unroll
            for (int k = 1; k < 4; ++k)
                if (k <= L) s = cadd(s, spmv_prod(A, saa[32 * k + lane], xs[k]));
            return;
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int kb = 1 + 16 * half;  // first column of this batch
            if (half == 1) {
                if (L < 17) break;
#pragma unroll
                for (int t = 0; t < 16; ++t)
                    if (kb + t <= L) xs[1 + t] = __ldg(x + sja[32 * (kb + t) + lane]);
                asm volatile("" ::: "memory");
            }
            // batch columns kb .. kb+15 live in xs[1 .. 16]
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
                const int g = 4 * half + gg;
                if (g < G) {
                    const double2 p0 = spmv_prod(A, saa[32 * (kb + 4 * gg) + lane], xs[1 + 4 * gg]);
                    const double2 p1 = spmv_prod(A, saa[32 * (kb + 4 * gg + 1) + lane], xs[2 + 4 * gg]);
                    const double2 p2 = spmv_prod(A, saa[32 * (kb + 4 * gg + 2) + lane], xs[3 + 4 * gg]);
                    const double2 p3 = spmv_prod(A, saa[32 * (kb + 4 * gg + 3) + lane], xs[4 + 4 * gg]);
                    if (g == 0) {
                        r0 = p0; r1 = p1; r2 = p2; r3 = p3;
                    } else {
                        r0 = cadd(r0, p0); r1 = cadd(r1, p1); r2 = cadd(r2, p2); r3 = cadd(r3, p3);
                    }
                } else if (g == G) {  // full groups done: combine, then the (< 4) leftovers
                    s = cadd(cadd(r0, r1), cadd(r2, r3));
                    combined = true;
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        if (4 * gg + j < 16 && kb + 4 * gg + j <= L)
                            s = cadd(s, spmv_prod(A, saa[32 * (kb + 4 * gg + j) + lane], xs[1 + 4 * gg + j]));
                }
            }
        }
    }

    __device__ __forceinline__ double2 result() {
        if (L < 0) return make_double2(0.0, 0.0);
        if (L == 0) return v0;
        if (L >= 4 && !combined) s = cadd(cadd(r0, r1), cadd(r2, r3));
        return cadd(v0, s);
    }
};

__device__ __forceinline__ double2 long_prod(const SellView& A, const double2* __restrict__ x, int64_t idx) {
    return spmv_prod(A, A.long_aa[idx], __ldg(x + A.long_ja[idx]));
}

// numpy CDOUBLE_pairwise_sum over products [s, s+L) of the side CSR,
// evaluated iteratively (explicit post-order stack; no device recursion, so
// the calling kernels keep their register allocation).
static __device__ __noinline__ double2 long_pw(const SellView& A, const double2* __restrict__ x, int64_t s, int64_t L) {
    int64_t fs[40], fl[40];
    int8_t fphase[40];
    double2 vals[40];
    int sp = 0, vp = 0;
    fs[0] = s;
    fl[0] = L;
    fphase[0] = 0;
    sp = 1;
    while (sp > 0) {
        const int64_t cs = fs[sp - 1], cl = fl[sp - 1];
        if (cl <= 64) {  // leaf
            double2 acc;
            if (cl < 4) {
                acc = make_double2(-0.0, -0.0);
                for (int64_t k = 0; k < cl; ++k) acc = cadd(acc, long_prod(A, x, cs + k));
            } else {
                double2 r0 = long_prod(A, x, cs), r1 = long_prod(A, x, cs + 1);
                double2 r2 = long_prod(A, x, cs + 2), r3 = long_prod(A, x, cs + 3);
                const int64_t G = cl / 4;
                for (int64_t g = 1; g < G; ++g) {
                    r0 = cadd(r0, long_prod(A, x, cs + 4 * g));
                    r1 = cadd(r1, long_prod(A, x, cs + 4 * g + 1));
                    r2 = cadd(r2, long_prod(A, x, cs + 4 * g + 2));
                    r3 = cadd(r3, long_prod(A, x, cs + 4 * g + 3));
                }
                acc = cadd(cadd(r0, r1), cadd(r2, r3));
                for (int64_t k = 4 * G; k < cl; ++k) acc = cadd(acc, long_prod(A, x, cs + k));
            }
            vals[vp++] = acc;
            --sp;
            continue;
        }
        const int64_t h = (cl - cl % 8) / 2;
        if (fphase[sp - 1] == 0) {  // descend left
            fphase[sp - 1] = 1;
            fs[sp] = cs; fl[sp] = h; fphase[sp] = 0; ++sp;
        } else if (fphase[sp - 1] == 1) {  // descend right
            fphase[sp - 1] = 2;
            fs[sp] = cs + h; fl[sp] = cl - h; fphase[sp] = 0; ++sp;
        } else {  // both halves done: combine left + right
            const double2 b = vals[--vp];
            const double2 a = vals[--vp];
            vals[vp++] = cadd(a, b);
            --sp;
        }
    }
    return vals[0];
}

__device__ __forceinline__ double2 long_row_sum(const SellView& A, const double2* __restrict__ x, int li) {
    const int64_t lo = A.long_ia[li], L = A.long_ia[li + 1] - lo;
    double2 v0 = long_prod(A, x, lo);
    return cadd(v0, long_pw(A, x, lo + 1, L - 1));
}

// ---- fast row path (whole slice per stage, FMA fingerprint) --------------
// One thread, one row of length len <= W4 (W4 = the slice width rounded up to
// 4, warp-uniform, a compile-time constant here).  All gathers of the row
// are issued before the first product; the pairwise order is evaluated with
// predication instead of branches: element k (>= 1) belongs to lane
// accumulator q = (k-1)%4 while its group g = (k-1)/4 is below G = L/4,
// else (g == G) it is leftover q, added after the (l0+l1)+(l2+l3) combine.
template <bool SWAP>
__device__ __forceinline__ double2 prod_fma(double2 a, double2 xv) {
    return SWAP ? f1(xv, a, true) : f1(a, xv, true);
}

template <int W4, bool SWAP>
__device__ __forceinline__ double2 row_fast(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                            int lane, int len) {
    constexpr int B1 = W4 < 28 ? W4 : 28;  // gathers in flight per batch (register budget)
    const double2 z = make_double2(0.0, 0.0);
    const int L = len - 1;
    const int G = L >> 2;
    const int rem = L - 4 * G;
    double2 r[4] = {z, z, z, z}, lo[3] = {z, z, z};
    double2 v0 = z;
    double2 xs[B1];
#pragma unroll
    for (int k = 0; k < B1; ++k) {
        xs[k] = z;
        if (k < len) xs[k] = __ldg(x + sja[32 * k + lane]);
    }
#pragma unroll
    for (int k = 0; k < W4; ++k) {
        if (k == B1) {  // second batch (rows wider than 28)
#pragma unroll
            for (int t = 0; t < W4 - B1; ++t) {
                xs[t] = z;
                if (B1 + t < len) xs[t] = __ldg(x + sja[32 * (B1 + t) + lane]);
            }
        }
        const double2 p = prod_fma<SWAP>(saa[32 * k + lane], xs[k < B1 ? k : k - B1]);
        if (k == 0) {
            v0 = p;
            continue;
        }
        const int g = (k - 1) >> 2, q = (k - 1) & 3;
        if (g < G) {
            r[q] = (g == 0) ? p : cadd(r[q], p);
        } else if (q < 3 && g == G) {
            lo[q] = p;
        }
    }
    double2 s = make_double2(-0.0, -0.0);
    if (G > 0) s = cadd(cadd(r[0], r[1]), cadd(r[2], r[3]));
    if (rem > 0) s = cadd(s, lo[0]);
    if (rem > 1) s = cadd(s, lo[1]);
    if (rem > 2) s = cadd(s, lo[2]);
    if (len <= 0) return z;
    if (len == 1) return v0;
    return cadd(v0, s);
}

template <bool SWAP>
__device__ __forceinline__ double2 row_fast_dispatch(int W, const double2* __restrict__ x, const double2* saa,
                                                     const int32_t* sja, int lane, int len) {
    switch ((W + 3) >> 2) {
        case 0:
        case 1: return row_fast<4, SWAP>(x, saa, sja, lane, len);
        case 2: return row_fast<8, SWAP>(x, saa, sja, lane, len);
        case 3: return row_fast<12, SWAP>(x, saa, sja, lane, len);
        case 4: return row_fast<16, SWAP>(x, saa, sja, lane, len);
        case 5: return row_fast<20, SWAP>(x, saa, sja, lane, len);
        case 6: return row_fast<24, SWAP>(x, saa, sja, lane, len);
        case 7: return row_fast<28, SWAP>(x, saa, sja, lane, len);
        case 8: return row_fast<32, SWAP>(x, saa, sja, lane, len);
        default: return row_fast<36, SWAP>(x, saa, sja, lane, len);
    }
}

// Persistent pipelined SpMV over the CTA's 4096-row blocks (blk = blockIdx.x,
// +gridDim.x, ...).  For each row the consumer thread calls
// ctx = body.prefetch(row) before the row's products (so the epilogue
// operands are in flight during the row computation), then
// body.row(row, value, ctx).  Bodies with reductions (Body::kReduce) get
// window_done(blk, slices) after every window of A.win slices and
// block_done(blk) after the block's last row, each behind a named barrier
// over the consumer warps; plain bodies never synchronise the consumers.
// The producer warp exits once it has issued every chunk.  `smem` holds
// kBarBytes + ns*stage_bytes bytes.
template <bool SWAP, class Body>
__device__ __forceinline__ void sell_pipeline(const SellView& A, const double2* __restrict__ x, Body& body,
                                              unsigned char* smem) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    // tag[st] = CTA-local index of the chunk the producer last armed stage st
    // for.  A consumer waits for its own tag before the parity wait on
    // full[st]: the parity wait cannot tell use u from use u+2, and a
    // consumer warp can reach use u+1 of a stage before use u has landed.
    volatile uint32_t* tag = reinterpret_cast<volatile uint32_t*>(empty + kMaxStages);
    // wid[st] = width (entries per row) of the slice in stage st (cm == 0),
    // written before the stage's arrive: visible after the full-barrier wait
    uint32_t* wid = reinterpret_cast<uint32_t*>(empty + kMaxStages) + kMaxStages;
    unsigned char* ring = smem + kBarBytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ns = A.ns, nch = A.nch;
    const int cols = 1 + 4 * A.cm;
    constexpr int kSlicesPerBlock = kBlock / kSlice;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            tag[i] = 0xffffffffu;
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == kConsumerWarps) {  // producer warp: lane l owns ring stage l
        // Chunk i of the CTA's sequence uses stage i % ns, so lane l issues
        // chunks l, l + ns, l + 2ns, ... in order; each lane polls its own
        // empty barrier without blocking, so the lanes progress independently
        // and one warp instruction issues up to 32 bulk copies.
        const uint64_t pol = l2_evict_first_policy();
        const bool owner = lane < ns;
        uint32_t i = (uint32_t)lane, u = 0;
        int64_t off0 = 0, off1 = 0, s = 0;
        int c = 0, w = 0;
        bool active = false;
        auto locate = [&]() {  // coordinates + offsets of chunk i (loads issued early)
            const uint32_t seq = i / (uint32_t)nch;
            c = (int)(i % (uint32_t)nch);
            const int64_t blk = blockIdx.x + (int64_t)(seq / kSlicesPerBlock) * gridDim.x;
            s = blk * kSlicesPerBlock + (seq % kSlicesPerBlock);
            active = blk < A.nblocks && s < A.nslices;
            if (active) {
                off0 = __ldg(A.slice_off + s);
                off1 = __ldg(A.slice_off + s + 1);
            }
        };
        if (owner) locate();
        while (__any_sync(0xffffffffu, owner && active)) {
            if (owner && active && (u == 0 || mbar_test(&empty[lane], (u - 1) & 1))) {
                w = (int)((off1 - off0) / kSlice);
                tag[lane] = i;
                unsigned char* stage = ring + (size_t)lane * A.stage_bytes;
                if (A.cm == 0) {  // whole slice + its row lengths
                    wid[lane] = (uint32_t)w;
                    const uint32_t cnt = (uint32_t)w * kSlice;
                    mbar_arrive_expect_tx(&full[lane], cnt * 20u + kSlice);
                    if (cnt) {
                        bulk_g2s(stage, A.aa + off0, cnt * 16u, &full[lane], pol);
                        bulk_g2s(stage + A.ja_off, A.ja + off0, cnt * 4u, &full[lane], pol);
                    }
                    bulk_g2s(stage + A.rl_off, A.rowlen + s * kSlice, kSlice, &full[lane], pol);
                } else {
                    const int c0 = c == 0 ? 0 : 1 + 4 * A.cm * c;
                    const int c1 = min(w, cols + 4 * A.cm * c);
                    const uint32_t cnt = c1 > c0 ? (uint32_t)(c1 - c0) * kSlice : 0u;
                    mbar_arrive_expect_tx(&full[lane], cnt * 20u);
                    if (cnt) {
                        const int64_t off = off0 + (int64_t)c0 * kSlice;
                        bulk_g2s(stage, A.aa + off, cnt * 16u, &full[lane], pol);
                        bulk_g2s(stage + A.ja_off, A.ja + off, cnt * 4u, &full[lane], pol);
                    }
                }
                i += (uint32_t)ns;
                ++u;
                locate();
            }
        }
        return;
    }
    const bool fast = A.cm == 0 && A.fma;
    uint32_t sbase = 0;  // CTA-local index of the block's first slice
    for (int64_t blk = blockIdx.x; blk < A.nblocks; blk += gridDim.x) {
        const int64_t s_lo = blk * kSlicesPerBlock;
        const int64_t s_hi = (s_lo + kSlicesPerBlock < A.nslices) ? s_lo + kSlicesPerBlock : A.nslices;
        const int nsl = (int)(s_hi - s_lo);
        // windows of A.win slices; after each (but the last) the body may
        // reduce everything that lies entirely in the rows done so far
        const int win = Body::kReduce ? A.win : nsl;
        for (int w0 = 0; w0 < nsl; w0 += win) {
        const int w1 = min(nsl, w0 + win);
        for (int j = w0 + warp; j < w1; j += kConsumerWarps) {
            const int64_t row = (s_lo + j) * kSlice + lane;
            if (fast) {
                const uint32_t i = sbase + (uint32_t)j;
                const uint32_t q = __umulhi(i, A.ns_magic);
                const int st = (int)(i - q * (uint32_t)ns);
                while (tag[st] != i) {
                }
                mbar_wait(&full[st], q & 1);
                const unsigned char* stage = ring + (size_t)st * A.stage_bytes;
                const int W = (int)wid[st];
                const int len = stage[A.rl_off + lane];
                const bool mine = row < A.n_rows && len != 255;
                typename Body::RowCtx ctx;
                if (mine) ctx = body.prefetch(row);
                const double2 val = row_fast_dispatch<SWAP>(W, x, reinterpret_cast<const double2*>(stage),
                                                            reinterpret_cast<const int32_t*>(stage + A.ja_off),
                                                            lane, mine ? len : 0);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (mine) body.row(row, val, ctx);
                continue;
            }
            const int len = A.rowlen[row];
            const bool mine = row < A.n_rows && len != 255;
            typename Body::RowCtx ctx;
            if (mine) ctx = body.prefetch(row);
            RowAcc acc;
            acc.init(mine ? len : 0);
            for (int c = 0; c < nch; ++c) {
                const uint32_t i = (sbase + (uint32_t)j) * (uint32_t)nch + (uint32_t)c;
                const int st = (int)(i % ns);
                while (tag[st] != i) {
                }
                mbar_wait(&full[st], (i / ns) & 1);
                const unsigned char* stage = ring + (size_t)st * A.stage_bytes;
                if (A.cm == 0) {
                    if (mine)
                        acc.full_row(A, x, reinterpret_cast<const double2*>(stage),
                                     reinterpret_cast<const int32_t*>(stage + A.ja_off), lane);
                } else {
                    const int c0 = c == 0 ? 0 : 1 + 4 * A.cm * c;
                    if (mine && len > c0)
                        acc.chunk(A, x, reinterpret_cast<const double2*>(stage),
                                  reinterpret_cast<const int32_t*>(stage + A.ja_off), lane, c, c0);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            }
            if (mine) body.row(row, acc.result(), ctx);
        }
        if (Body::kReduce && w1 < nsl) {
            named_sync(1, kConsumers);
            body.window_done(blk, w1);
        }
        }
        sbase += (uint32_t)nsl;
        if (A.long_blk_ptr) {
            const int lb = A.long_blk_ptr[blk], le = A.long_blk_ptr[blk + 1];
            for (int li = lb + (int)threadIdx.x; li < le; li += kConsumers) {
                const int64_t row = (int64_t)A.long_row[li];
                typename Body::RowCtx ctx = body.prefetch(row);
                body.row(row, long_row_sum(A, x, li), ctx);
            }
        }
        if (Body::kReduce) {
            named_sync(1, kConsumers);
            body.block_done(blk);
        }
    }
}

// Kernel-side dispatch on numpy's elision swap (a launch-uniform flag).
template <class Body>
__device__ __forceinline__ void sell_run(const SellView& A, const double2* __restrict__ x, Body& body,
                                         unsigned char* smem) {
    if (A.swap) sell_pipeline<true>(A, x, body, smem);
    else sell_pipeline<false>(A, x, body, smem);
}

}  // namespace zk
