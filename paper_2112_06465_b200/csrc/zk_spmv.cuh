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
#include "zk_blockred.cuh"

namespace zk {

// 8 warps per CTA (2 per SM sub-partition, so up to 255 registers/thread):
// plain SpMV = 7 consumer warps + the TMA producer; fused reductions = 6
// consumer warps + producer + reducer (a 9th warp would cap registers at 168).
#ifndef ZK_RED_CW
#define ZK_RED_CW 6
#endif
#ifndef ZK_B1
#define ZK_B1 28
#endif
#ifndef ZK_PLAIN_CW
#define ZK_PLAIN_CW 7
#endif
constexpr int kPipeThreads = 32 * (ZK_PLAIN_CW + 1);
constexpr int kRedPipeThreads = 32 * (ZK_RED_CW + 2);
template <bool RED> struct PipeWarps {
    static constexpr int consumers = RED ? ZK_RED_CW : ZK_PLAIN_CW;
    static constexpr int producer = consumers;
    static constexpr int reducer = consumers + 1;
};
constexpr int kMaxStages = 32;
constexpr int kBarBytes = 2 * kMaxStages * 8 + 2 * kMaxStages * 4;  // full, empty mbarriers + stage tags, widths
constexpr int kSmemLimit = 227 * 1024;
constexpr int kFullCols = 33;  // widest row handled by the whole-row prefetch path
// Reduction stash: a ring of RedSmem::kSlots slice slots (32 rows each) of
// per-row reduction terms between the consumer warps and the reducer warp.
// Stash slots and reducer leaf batch per body (RedSmem::kSlots, kBatchRows;
// slots a power of two and above the batch's slices, or the consumers and
// the reducer deadlock).  Bodies with two complex terms (K4) keep a 16-slot
// stash and 256-row batches -- the smaller stash gives their TMA ring a
// stage -- the others take 32 slots and 512-row batches (fewer reducer
// passes).  Measured on C4, per phase and overall (batch rows / slots):
// 256/16 1.49, 512/32 1.515, 768/32 1.515, 1024/64 1.47, 128/32 1.30 solves/s;
// K4 919 us at 256/16 vs 923-941 at 512/32 and 932 at 384/16.
constexpr int kNodeSlots = 136;  // >= plan nodes (<= 129) per accumulator


struct SellView {
    int64_t n_rows, n_cols, nslices, nblocks;
    const double2* __restrict__ aa;
    const int32_t* __restrict__ ja;
    const int64_t* __restrict__ slice_off;
    const int32_t* __restrict__ slice_cmax;  // largest column of each slice (x leading edge)
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
    int32_t sv_off;       // byte offset of the staged vector rows (cm == 0): nsv x 32 double2
    int32_t nsv;          // vectors staged with each slice (the row epilogue's operands)
    const double2* sv[2]; // their base pointers (row-indexed, n_rows long)
    int32_t ns;           // ring stages for this launch
    uint32_t ns_magic;    // floor(2^32 / ns) + 1: i / ns = umulhi(i, ns_magic) for i < 2^27
    // plain (reduction-free) pipelines may cut the rows into smaller
    // pipeline blocks of `spb` slices (nvb of them), so a small matrix still
    // spreads over every SM; fused-reduction pipelines keep 4096-row blocks
    int32_t spb;
    int64_t nvb;
    bool prefetch;        // L2 bulk prefetch of each slice's new x rows (one more TMA op per slice)
    bool swap;            // numpy elided the gathered temporary: prod = F1(x[ja], aa)
    bool fma;
    int32_t narrow_w;     // plain launches: 8 / 16 = narrow kernels of that width class, 0 = the ring
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

// ---- long rows (> 65 entries, side CSR): one WARP per row ----------------------
// numpy's CDOUBLE_pairwise_sum over the products [s, s+L) of a long row: the
// recursion halves a range (split at (L - L%8)/2) until it holds <= 64
// elements, a leaf sums with four lane accumulators over full groups of
// four, (l0+l1)+(l2+l3), then its leftovers.  The warp walks the recursion in
// lockstep (every lane the same explicit stack, so control flow is uniform);
// each subtree of <= kLongChunk elements (<= 32 leaves) is a CHUNK whose
// leaves are summed one per lane in parallel and combined in the recursion's
// order through shuffles.  Every lane ends with the row value.
constexpr int64_t kLongChunk = 896;  // leaves are >= 28 elements: <= 32 leaves per chunk

__device__ __forceinline__ double2 long_prod(const SellView& A, const double2* __restrict__ x, int64_t idx) {
    return spmv_prod(A, A.long_aa[idx], __ldg(x + A.long_ja[idx]));
}

__device__ __forceinline__ int64_t pw_split(int64_t L) { return (L - L % 8) / 2; }

// One numpy leaf (L <= 64) of products [s, s+L), summed by one thread.
__device__ __forceinline__ double2 long_leaf(const SellView& A, const double2* __restrict__ x, int64_t s, int64_t L) {
    if (L < 4) {
        double2 acc = make_double2(-0.0, -0.0);
        for (int64_t k = 0; k < L; ++k) acc = cadd(acc, long_prod(A, x, s + k));
        return acc;
    }
    double2 r0 = long_prod(A, x, s), r1 = long_prod(A, x, s + 1), r2 = long_prod(A, x, s + 2), r3 = long_prod(A, x, s + 3);
    const int64_t G = L / 4;
    for (int64_t g = 1; g < G; ++g) {
        const double2 p0 = long_prod(A, x, s + 4 * g), p1 = long_prod(A, x, s + 4 * g + 1);
        const double2 p2 = long_prod(A, x, s + 4 * g + 2), p3 = long_prod(A, x, s + 4 * g + 3);
        r0 = cadd(r0, p0);
        r1 = cadd(r1, p1);
        r2 = cadd(r2, p2);
        r3 = cadd(r3, p3);
    }
    double2 acc = cadd(cadd(r0, r1), cadd(r2, r3));
    for (int64_t k = 4 * G; k < L; ++k) acc = cadd(acc, long_prod(A, x, s + k));
    return acc;
}

// A chunk [s, s+L) (L <= kLongChunk): lane i sums leaf i, then the chunk's
// tree is combined in recursion order (all lanes, shuffles).
static __device__ __noinline__ double2 long_chunk(const SellView A, const double2* __restrict__ x, int64_t s, int64_t L) {
    const int lane = threadIdx.x & 31;
    if (L <= 64) {  // a single leaf: lane 0 sums it
        double2 v = make_double2(0.0, 0.0);
        if (lane == 0) v = long_leaf(A, x, s, L);
        return make_double2(__shfl_sync(0xffffffffu, v.x, 0), __shfl_sync(0xffffffffu, v.y, 0));
    }
    // pass 1: enumerate leaves in order; lane i keeps leaf i
    int64_t st[8], ln[8];
    int8_t ph[8];
    int sp = 1, nleaf = 0;
    int64_t my_s = 0, my_l = 0;
    st[0] = s;
    ln[0] = L;
    ph[0] = 0;
    while (sp > 0) {
        const int64_t cs = st[sp - 1], cl = ln[sp - 1];
        if (cl <= 64) {
            if (nleaf == lane) {
                my_s = cs;
                my_l = cl;
            }
            ++nleaf;
            --sp;
            continue;
        }
        const int64_t h = pw_split(cl);
        if (ph[sp - 1] == 0) {
            ph[sp - 1] = 1;
            st[sp] = cs; ln[sp] = h; ph[sp] = 0; ++sp;
        } else if (ph[sp - 1] == 1) {
            ph[sp - 1] = 2;
            st[sp] = cs + h; ln[sp] = cl - h; ph[sp] = 0; ++sp;
        } else {
            --sp;
        }
    }
    const double2 leaf = lane < nleaf ? long_leaf(A, x, my_s, my_l) : make_double2(0.0, 0.0);
    // pass 2: post-order combine, leaf values fetched from their lanes
    double2 vals[8];
    int vp = 0, li = 0;
    sp = 1;
    st[0] = s;
    ln[0] = L;
    ph[0] = 0;
    while (sp > 0) {
        const int64_t cs = st[sp - 1], cl = ln[sp - 1];
        if (cl <= 64) {
            vals[vp++] = make_double2(__shfl_sync(0xffffffffu, leaf.x, li), __shfl_sync(0xffffffffu, leaf.y, li));
            ++li;
            --sp;
            continue;
        }
        const int64_t h = pw_split(cl);
        if (ph[sp - 1] == 0) {
            ph[sp - 1] = 1;
            st[sp] = cs; ln[sp] = h; ph[sp] = 0; ++sp;
        } else if (ph[sp - 1] == 1) {
            ph[sp - 1] = 2;
            st[sp] = cs + h; ln[sp] = cl - h; ph[sp] = 0; ++sp;
        } else {
            const double2 b = vals[--vp];
            const double2 a = vals[--vp];
            vals[vp++] = cadd(a, b);
            --sp;
        }
    }
    return vals[0];
}

// Row value of long row li: v0 + PW(v1 .. v_{L-1}); whole warp, uniform li.
static __device__ __noinline__ double2 long_row_warp(const SellView A, const double2* __restrict__ x, int li) {
    const int64_t lo = A.long_ia[li], L = A.long_ia[li + 1] - lo;
    const double2 v0 = long_prod(A, x, lo);
    const int64_t s = lo + 1, n = L - 1;
    // top of the recursion above the chunks (uniform explicit stack)
    int64_t st[48], ln[48];
    int8_t ph[48];
    double2 vals[48];
    int sp = 1, vp = 0;
    st[0] = s;
    ln[0] = n;
    ph[0] = 0;
    while (sp > 0) {
        const int64_t cs = st[sp - 1], cl = ln[sp - 1];
        if (cl <= kLongChunk) {
            vals[vp++] = long_chunk(A, x, cs, cl);
            --sp;
            continue;
        }
        const int64_t h = pw_split(cl);
        if (ph[sp - 1] == 0) {
            ph[sp - 1] = 1;
            st[sp] = cs; ln[sp] = h; ph[sp] = 0; ++sp;
        } else if (ph[sp - 1] == 1) {
            ph[sp - 1] = 2;
            st[sp] = cs + h; ln[sp] = cl - h; ph[sp] = 0; ++sp;
        } else {
            const double2 b = vals[--vp];
            const double2 a = vals[--vp];
            vals[vp++] = cadd(a, b);
            --sp;
        }
    }
    return cadd(v0, vals[0]);
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

struct RowSum {
    double2 v0, r[4], lo[3];
    int G, rem, len;
    __device__ __forceinline__ void init(int n) {
        const double2 z = make_double2(0.0, 0.0);
        len = n;
        const int L = n - 1;
        G = L >> 2;
        rem = L - 4 * G;
        v0 = z;
#pragma unroll
        for (int q = 0; q < 4; ++q) r[q] = z;
#pragma unroll
        for (int q = 0; q < 3; ++q) lo[q] = z;
    }
    __device__ __forceinline__ void add(int k, double2 p) {  // k: compile-time after unrolling
        if (k == 0) {
            v0 = p;
            return;
        }
        const int g = (k - 1) >> 2, q = (k - 1) & 3;
        if (g < G) {
            r[q] = (g == 0) ? p : cadd(r[q], p);
        } else if (q < 3 && g == G) {
            lo[q] = p;
        }
    }
    __device__ __forceinline__ double2 result() const {
        double2 s = make_double2(-0.0, -0.0);
        if (G > 0) s = cadd(cadd(r[0], r[1]), cadd(r[2], r[3]));
        if (rem > 0) s = cadd(s, lo[0]);
        if (rem > 1) s = cadd(s, lo[1]);
        if (rem > 2) s = cadd(s, lo[2]);
        if (len <= 0) return make_double2(0.0, 0.0);
        if (len == 1) return v0;
        return cadd(v0, s);
    }
};

// Columns [K0, K1) of one vector: gathers first, then the products in order.
template <int K0, int K1, bool SWAP>
__device__ __forceinline__ void row_seg(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                        int lane, RowSum& acc) {
    double2 xs[K1 - K0];
#pragma unroll
    for (int k = K0; k < K1; ++k) {
        xs[k - K0] = make_double2(0.0, 0.0);
        if (k < acc.len) xs[k - K0] = __ldg(x + sja[32 * k + lane]);
    }
#pragma unroll
    for (int k = K0; k < K1; ++k) acc.add(k, prod_fma<SWAP>(saa[32 * k + lane], xs[k - K0]));
}

// ---- uniform slices: every row of the warp has exactly W entries --------
// (the common case for stencil and FE matrices).  L, G and the leftover
// count are compile-time constants, so the numpy order is straight-line
// code with no predication at all.
template <int K0, int K1, int W, bool SWAP>
__device__ __forceinline__ void uni_seg(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                        int lane, double2& v0, double2 (&r)[4], double2 (&lo)[3]) {
    constexpr int L = W - 1, G = L >> 2;
    double2 xs[K1 - K0];
#pragma unroll
    for (int k = K0; k < K1; ++k) xs[k - K0] = __ldg(x + sja[32 * k + lane]);
#pragma unroll
    for (int k = K0; k < K1; ++k) {
        const double2 p = prod_fma<SWAP>(saa[32 * k + lane], xs[k - K0]);
        if (k == 0) {
            v0 = p;
        } else {
            const int g = (k - 1) >> 2, q = (k - 1) & 3;
            if (g < G) r[q] = (g == 0) ? p : cadd(r[q], p);
            else lo[q] = p;
        }
    }
}

template <int K0, int W, bool SWAP>
__device__ __forceinline__ void uni_segs(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                         int lane, double2& v0, double2 (&r)[4], double2 (&lo)[3]) {
    constexpr int K1 = (K0 + ZK_B1 < W) ? K0 + ZK_B1 : W;
    uni_seg<K0, K1, W, SWAP>(x, saa, sja, lane, v0, r, lo);
    if constexpr (K1 < W) uni_segs<K1, W, SWAP>(x, saa, sja, lane, v0, r, lo);
}

template <int W, bool SWAP>
__device__ __forceinline__ double2 row_uniform(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                               int lane) {
    constexpr int L = W - 1, G = L >> 2, REM = L - 4 * G;
    double2 v0, r[4], lo[3];
    uni_segs<0, W, SWAP>(x, saa, sja, lane, v0, r, lo);
    if constexpr (W == 1) {
        return v0;
    } else {
        double2 s = make_double2(-0.0, -0.0);
        if constexpr (G > 0) s = cadd(cadd(r[0], r[1]), cadd(r[2], r[3]));
#pragma unroll
        for (int j = 0; j < REM; ++j) s = cadd(s, lo[j]);
        return cadd(v0, s);
    }
}

template <bool SWAP>
__device__ __forceinline__ double2 row_uniform_dispatch(int W, const double2* __restrict__ x, const double2* saa,
                                                        const int32_t* sja, int lane) {
    switch (W) {
#define ZK_UNI(w) \
    case w: return row_uniform<w, SWAP>(x, saa, sja, lane);
        ZK_UNI(1) ZK_UNI(2) ZK_UNI(3) ZK_UNI(4) ZK_UNI(5) ZK_UNI(6) ZK_UNI(7) ZK_UNI(8)
        ZK_UNI(9) ZK_UNI(10) ZK_UNI(11) ZK_UNI(12) ZK_UNI(13) ZK_UNI(14) ZK_UNI(15) ZK_UNI(16)
        ZK_UNI(17) ZK_UNI(18) ZK_UNI(19) ZK_UNI(20) ZK_UNI(21) ZK_UNI(22) ZK_UNI(23) ZK_UNI(24)
        ZK_UNI(25) ZK_UNI(26) ZK_UNI(27) ZK_UNI(28) ZK_UNI(29) ZK_UNI(30) ZK_UNI(31) ZK_UNI(32)
#undef ZK_UNI
        default: return make_double2(0.0, 0.0);
    }
}

// Columns [K0, W4) in batches of ZK_B1 gathers.
template <int K0, int W4, bool SWAP>
__device__ __forceinline__ void row_segs(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                         int lane, RowSum& acc) {
    constexpr int K1 = (K0 + ZK_B1 < W4) ? K0 + ZK_B1 : W4;
    row_seg<K0, K1, SWAP>(x, saa, sja, lane, acc);
    if constexpr (K1 < W4) row_segs<K1, W4, SWAP>(x, saa, sja, lane, acc);
}

// NX = 1: out[0] = row of A x0.  NX = 2: out[1] = row of A x1 as well, the
// second vector's row summed after the first (one register set for the
// gathers: the two sets in flight at once spill at 255 registers).
template <int NX>
struct RowVals {
    double2 v[NX];
};

template <int W4, bool SWAP>
__device__ __forceinline__ double2 row_one(const double2* __restrict__ x, const double2* saa, const int32_t* sja,
                                           int lane, int len) {
    RowSum acc;
    acc.init(len);
    row_segs<0, W4, SWAP>(x, saa, sja, lane, acc);
    return acc.result();
}

template <int W4, bool SWAP, int NX>
__device__ __forceinline__ RowVals<NX> row_fast(const double2* __restrict__ x0, const double2* __restrict__ x1,
                                                const double2* saa, const int32_t* sja, int lane, int len) {
    RowVals<NX> out;
    if constexpr (NX == 1) {
        out.v[0] = row_one<W4, SWAP>(x0, saa, sja, lane, len);
    } else {
        // one code copy, run once per vector (the two rows' gather sets in
        // flight together do not fit in 255 registers)
#pragma unroll 1
        for (int v = 0; v < 2; ++v) {
            const double2 r = row_one<W4, SWAP>(v == 0 ? x0 : x1, saa, sja, lane, len);
            if (v == 0) out.v[0] = r;
            else out.v[1] = r;
        }
    }
    return out;
}

template <bool SWAP, int NX>
__device__ __forceinline__ RowVals<NX> row_fast_dispatch(int W, const double2* __restrict__ x0,
                                                         const double2* __restrict__ x1, const double2* saa,
                                                         const int32_t* sja, int lane, int len, bool pad) {
    // pad: row beyond n_rows (its result is not used)
    if (W >= 1 && W <= 32 && __all_sync(0xffffffffu, pad || len == W)) {
        RowVals<NX> out;
#pragma unroll 1
        for (int v = 0; v < NX; ++v) {
            const double2 r = row_uniform_dispatch<SWAP>(W, v == 0 ? x0 : x1, saa, sja, lane);
            if (v == 0) out.v[0] = r;
            else out.v[NX - 1] = r;
        }
        return out;
    }
    switch ((W + 3) >> 2) {
        case 0:
        case 1: return row_fast<4, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 2: return row_fast<8, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 3: return row_fast<12, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 4: return row_fast<16, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 5: return row_fast<20, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 6: return row_fast<24, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 7: return row_fast<28, SWAP, NX>(x0, x1, saa, sja, lane, len);
        case 8: return row_fast<32, SWAP, NX>(x0, x1, saa, sja, lane, len);
        default: return row_fast<36, SWAP, NX>(x0, x1, saa, sja, lane, len);
    }
}

// ---- narrow matrices: one thread per row, per-warp TMA double buffer ------
// Slices at most 8 (C1/C5's 7-point rows) or 16 (C3's P1 elements) wide and
// no long rows.  With short rows the ring's consumers (7 warps per SM) have
// too few gathers in flight (C5 SpMV 648 us, 0.68 of HBM).  Here a persistent
// warp walks slices s, s + nw, ...: the next slice's values arrive by one
// bulk copy into the warp's other stage and its columns and row lengths by
// loads into registers while the current slice's gathers are in flight, so
// only the gathers' latency is exposed (C5: 421 us; one warp per slice with
// direct loads and no prefetch measured 509 us).  Rows sum in numpy's order
// (RowSum, the fast path's order).
constexpr int kNarrowThreads = 256;
constexpr int kNarrowWarps = kNarrowThreads / 32;
#ifndef ZK_NARROW_MINB
#define ZK_NARROW_MINB 2  // width 8: CTAs per SM (108 registers, no spills; 3 CTAs spill at 80)
#endif
#ifndef ZK_NARROW2_MINB
#define ZK_NARROW2_MINB 2  // width 8, two vectors: 128 registers, no spills (1 CTA at 144: 857 vs 589 us on C5)
#endif
#ifndef ZK_NARROW16_WARPS
#define ZK_NARROW16_WARPS 12  // width 16, one vector: warps per CTA (148 registers: 12 fit one SM)
#endif
template <int WM>
struct NarrowCfg {
    static constexpr int kStage = WM * kSlice * 16;  // values of one slice
    // warps per CTA: 8, except width 16 with one vector (one CTA per SM)
    static constexpr int warps(int nx) { return (WM > 8 && nx == 1) ? ZK_NARROW16_WARPS : kNarrowWarps; }
    static constexpr int kBars = 256;  // two mbarriers per warp, up to 16 warps
    static constexpr int smem(int nx) { return kBars + warps(nx) * 2 * kStage; }
    static constexpr int kSmem = smem(1) > smem(2) ? smem(1) : smem(2);  // attribute for either
    static constexpr int kMinB = WM <= 8 ? ZK_NARROW_MINB : 1;    // one vector
    static constexpr int kMinB2 = WM <= 8 ? ZK_NARROW2_MINB : 1;  // two vectors
};

// NX = 2: rows of A x0 and A x1 from one pass over the matrix (both gather
// sets in flight, the two sums one after the other).
template <int WM, int NX, class Body>
__device__ __forceinline__ void narrow_tma_run(const SellView& A, const double2* __restrict__ x0,
                                               const double2* __restrict__ x1, Body& body, unsigned char* smem) {
    static_assert(Body::kSV == 0 && Body::kNC == 0 && Body::kNR == 0, "plain bodies only");
    constexpr int kStage = NarrowCfg<WM>::kStage;
    constexpr int kW = NarrowCfg<WM>::warps(NX);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + 2 * warp;
    static_assert(kW * 2 * 8 <= NarrowCfg<WM>::kBars, "mbarrier area");
    unsigned char* buf = smem + NarrowCfg<WM>::kBars + (size_t)warp * 2 * kStage;
    const int64_t ns = A.nslices, nw = (int64_t)gridDim.x * kW;
    int64_t s = (int64_t)blockIdx.x * kW + warp;
    if (s >= ns) return;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncwarp();
    const uint64_t pol = l2_evict_first_policy();
    const double2 z = make_double2(0.0, 0.0);
    // offsets of the current and the next slice
    int64_t o0 = A.slice_off[s], e0 = A.slice_off[s + 1];
    int64_t s1 = s + nw;
    int64_t o1 = s1 < ns ? A.slice_off[s1] : 0, e1 = s1 < ns ? A.slice_off[s1 + 1] : 0;
    if (lane == 0) {
        mbar_arrive_expect_tx(&bar[0], (uint32_t)(e0 - o0) * 16u);
        if (e0 > o0) bulk_g2s(buf, A.aa + o0, (uint32_t)(e0 - o0) * 16u, &bar[0], pol);
    }
    int32_t jc[WM];
    int lc;
    {
        const int W = (int)((e0 - o0) / kSlice);
#pragma unroll
        for (int q = 0; q < WM; ++q) jc[q] = q < W ? __ldcs(A.ja + o0 + 32 * q + lane) : 0;
        lc = s * kSlice + lane < A.n_rows ? (int)A.rowlen[s * kSlice + lane] : 0;
    }
    for (uint32_t k = 0; s < ns; s = s1, s1 += nw, ++k) {
        const int st = (int)(k & 1);
        double2 xs[NX][WM];
#pragma unroll
        for (int q = 0; q < WM; ++q) xs[0][q] = q < lc ? __ldg(x0 + jc[q]) : z;
        if constexpr (NX == 2) {
#pragma unroll
            for (int q = 0; q < WM; ++q) xs[NX - 1][q] = q < lc ? __ldg(x1 + jc[q]) : z;
        }
        // the next slice: values by TMA into the other stage, columns and
        // lengths into registers; offsets of the one after
        const int64_t s2 = s1 + nw;
        const int64_t o2 = s2 < ns ? A.slice_off[s2] : 0, e2 = s2 < ns ? A.slice_off[s2 + 1] : 0;
        int32_t jn[WM];
        int ln = 0;
        if (s1 < ns) {
            if (lane == 0) {
                mbar_arrive_expect_tx(&bar[st ^ 1], (uint32_t)(e1 - o1) * 16u);
                if (e1 > o1) bulk_g2s(buf + (st ^ 1) * kStage, A.aa + o1, (uint32_t)(e1 - o1) * 16u, &bar[st ^ 1], pol);
            }
            const int W1 = (int)((e1 - o1) / kSlice);
#pragma unroll
            for (int q = 0; q < WM; ++q) jn[q] = q < W1 ? __ldcs(A.ja + o1 + 32 * q + lane) : 0;
            ln = s1 * kSlice + lane < A.n_rows ? (int)A.rowlen[s1 * kSlice + lane] : 0;
        } else {
#pragma unroll
            for (int q = 0; q < WM; ++q) jn[q] = 0;
        }
        // the current slice
        mbar_wait(&bar[st], (k >> 1) & 1);
        const double2* sa = reinterpret_cast<const double2*>(buf + st * kStage) + lane;
        const int W = (int)((e0 - o0) / kSlice);
        double2 v[NX];
#pragma unroll
        for (int u = 0; u < NX; ++u) {
            RowSum acc;
            acc.init(lc);
#pragma unroll
            for (int q = 0; q < WM; ++q) acc.add(q, spmv_prod(A, q < W ? sa[32 * q] : z, xs[u][q]));
            v[u] = acc.result();
        }
        const int64_t row = s * kSlice + lane;
        if (row < A.n_rows) {
            double2 sv[1], tc[1];
            double tr[1];
            body.row(row, v, sv, tc, tr);
        }
        __syncwarp();  // every lane has read stage st before it is refilled
        o0 = o1;
        e0 = e1;
        o1 = o2;
        e1 = e2;
        lc = ln;
#pragma unroll
        for (int q = 0; q < WM; ++q) jc[q] = jn[q];
    }
}

// Persistent grid of a narrow launch (NX vectors).
int num_sms();  // zk_internal.h (cached device attribute)

__host__ __forceinline__ unsigned narrow_grid(const SellView& v, int nx = 1) {
    const int sms = num_sms();
    const int minb = v.narrow_w <= 8 ? (nx == 1 ? NarrowCfg<8>::kMinB : NarrowCfg<8>::kMinB2)
                                     : (nx == 1 ? NarrowCfg<16>::kMinB : NarrowCfg<16>::kMinB2);
    const int64_t want = (int64_t)sms * minb;
    const int w = v.narrow_w <= 8 ? NarrowCfg<8>::warps(nx) : NarrowCfg<16>::warps(nx);
    const int64_t need = (v.nslices + w - 1) / w;
    return (unsigned)(need < want ? (need > 0 ? need : 1) : want);
}
__host__ __forceinline__ size_t narrow_smem(const SellView& v, int nx = 1) {
    return v.narrow_w <= 8 ? NarrowCfg<8>::smem(nx) : NarrowCfg<16>::smem(nx);
}

// Launch kernel template KERN<8> or KERN<16> by the view's narrow width.
#define ZK_NARROW_LAUNCH(KERN, V, NX, STREAM, ...)                                                         \
    do {                                                                                                  \
        if ((V).narrow_w <= 8)                                                                            \
            KERN<8><<<narrow_grid((V), (NX)), 32 * NarrowCfg<8>::warps(NX), narrow_smem((V), (NX)), (STREAM)>>>(__VA_ARGS__); \
        else                                                                                              \
            KERN<16><<<narrow_grid((V), (NX)), 32 * NarrowCfg<16>::warps(NX), narrow_smem((V), (NX)), (STREAM)>>>(__VA_ARGS__); \
    } while (0)
// Dynamic shared memory attributes of both instantiations.
#define ZK_NARROW_ATTR(KERN)                                                                                     \
    do {                                                                                                        \
        ZK_CUDA(cudaFuncSetAttribute(KERN<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, NarrowCfg<8>::kSmem));   \
        ZK_CUDA(cudaFuncSetAttribute(KERN<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, NarrowCfg<16>::kSmem)); \
    } while (0)

// Index of long row `row` in the side CSR (binary search in its block's range).
__device__ __forceinline__ int long_index(const SellView& A, int64_t blk, int64_t row) {
    int lo = A.long_blk_ptr[blk], hi = A.long_blk_ptr[blk + 1] - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)A.long_row[mid] < row) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}


// The long rows of one slice (lanes in `lm`), one after the other, each by
// the whole warp; the owning lane takes the row value.
template <int NX>
static __device__ __noinline__ void long_rows_slice(const SellView A, const double2* __restrict__ x0,
                                                    const double2* __restrict__ x1, unsigned lm, int64_t row,
                                                    RowVals<NX>& val) {
    const int lane = threadIdx.x & 31;
    for (; lm; lm &= lm - 1) {
        const int src = __ffs(lm) - 1;
        const int64_t lrow = __shfl_sync(0xffffffffu, row, src);
        const int li = long_index(A, lrow / kBlock, lrow);
        const double2 r0 = long_row_warp(A, x0, li);
        if (lane == src) val.v[0] = r0;
        if constexpr (NX == 2) {
            const double2 r1 = long_row_warp(A, x1, li);
            if (lane == src) val.v[1] = r1;
        }
    }
}

// Generic slice path (rows wider than kFullCols split over chunks, or the
// non-FMA fingerprint): RowAcc per vector, chunk by chunk.  Out of line so
// its registers do not weigh on the fast path.
template <int NX>
__device__ __noinline__ RowVals<NX> generic_slice(const SellView A, const double2* __restrict__ x0,
                                                  const double2* __restrict__ x1, uint64_t* full, uint64_t* empty,
                                                  volatile uint32_t* tag, const unsigned char* ring, uint32_t sq,
                                                  int lane, int len) {
    RowAcc acc[NX];
#pragma unroll
    for (int v = 0; v < NX; ++v) acc[v].init(len);
    const int ns = A.ns, nch = A.nch;
    for (int c = 0; c < nch; ++c) {
        const uint32_t i = sq * (uint32_t)nch + (uint32_t)c;
        const int st = (int)(i % ns);
        while (tag[st] != i) {
        }
        mbar_wait(&full[st], (i / ns) & 1);
        const unsigned char* stage = ring + (size_t)st * A.stage_bytes;
        const double2* saa = reinterpret_cast<const double2*>(stage);
        const int32_t* sja = reinterpret_cast<const int32_t*>(stage + A.ja_off);
#pragma unroll
        for (int v = 0; v < NX; ++v) {
            const double2* xv = v == 0 ? x0 : x1;
            if (A.cm == 0) {
                if (len > 0) acc[v].full_row(A, xv, saa, sja, lane);
            } else {
                const int c0 = c == 0 ? 0 : 1 + 4 * A.cm * c;
                if (len > c0) acc[v].chunk(A, xv, saa, sja, lane, c, c0);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    RowVals<NX> out;
#pragma unroll
    for (int v = 0; v < NX; ++v) out.v[v] = acc[v].result();
    return out;
}

// ---- fused reductions: consumer warps -> stash ring -> reducer warp --------
// Per row the body returns NC complex and NR real reduction terms; the
// consumer warp that owns a slice writes them into stash slot
// (CTA slice sequence number) % kSlots and arrives on that slot's
// `sfull` barrier.  The reducer warp takes the slices of each 4096-row block
// in order, sums every pairwise leaf of the block's plans as soon as all its
// rows are in (leaf_upto table), releases slots no pending leaf still needs
// (`sfree`), and after the last leaf combines the tree, stores the block
// partials and counts the arrival.  The reducer of the CTA retiring the last
// block folds all partials in order (vecops.py:159-161) and hands the totals
// to body.finish().  Consumers therefore never wait for a reduction.
struct RedCfg {
    PlanPtrs pc, pr;       // complex / real plans (vecops.py DEFAULT_PLAN, 4096)
    double* partials;      // nblocks x (2 NC + NR) doubles
    unsigned int* counter; // block arrivals (reset by body.finish)
    int defer;             // row-sharded solve: leave the fold to the cross-rank finish kernel
    double* slots;         // non-null: streaming fold (zk_blockred.cuh) instead of arrivals + last-CTA fold
};

constexpr int kPlanCache = 2560;  // bytes of shared memory per cached plan (full-block plans: ~2.0 / 1.3 KB)

template <int NC, int NR>
struct RedSmem {
    static constexpr int kSlots = NC >= 2 ? 16 : 32;
    static constexpr int kBatchRows = NC >= 2 ? 256 : 512;  // the reducer sums leaves in batches of ~this many rows
    static_assert((kSlots & (kSlots - 1)) == 0, "stash slots: power of two");
    // Deadlock freedom: the reducer may hold a whole leaf batch, plus one
    // partially covered leaf (<= 64 complex / 128 real rows), plus up to a
    // slice of misalignment, while the consumers need the slice being
    // waited on -- all of it must fit in the stash at once.
    static_assert(kSlots * kSlice >= kBatchRows + 128 + 2 * kSlice, "stash too small for the reducer's leaf batch");
    static constexpr uint32_t kMask = (uint32_t)(kSlots * kSlice - 1);
    static constexpr size_t kBars = 2 * kSlots * 8;
    static constexpr size_t kStashC = (size_t)kSlots * kSlice * NC * 16;
    static constexpr size_t kStashR = (size_t)kSlots * kSlice * NR * 8;
    static constexpr size_t kNodesC = (size_t)kNodeSlots * NC * 16;
    static constexpr size_t kNodesR = (size_t)kNodeSlots * NR * 8;
    static constexpr size_t kPlans = (size_t)kPlanCache * ((NC > 0) + (NR > 0));
    static constexpr int kFoldPer = 8;  // fold_progress staging: 32 x 8 doubles (in the stash, free by then)
    static constexpr size_t kFold = 64;
    static constexpr size_t kBytes = (NC + NR) ? kBars + kStashC + kStashR + kNodesC + kNodesR + kPlans + kFold : 0;
    unsigned char* base;
    __device__ uint64_t* sfull() const { return reinterpret_cast<uint64_t*>(base); }
    __device__ uint64_t* sfree() const { return reinterpret_cast<uint64_t*>(base) + kSlots; }
    __device__ double2* stc() const { return reinterpret_cast<double2*>(base + kBars); }
    __device__ double* str() const { return reinterpret_cast<double*>(base + kBars + kStashC); }
    __device__ double2* ndc() const { return reinterpret_cast<double2*>(base + kBars + kStashC + kStashR); }
    __device__ double* ndr() const { return reinterpret_cast<double*>(base + kBars + kStashC + kStashR + kNodesC); }
    __device__ char* planc() const { return reinterpret_cast<char*>(base + kBars + kStashC + kStashR + kNodesC + kNodesR); }
    __device__ char* planr() const { return planc() + (NC > 0 ? kPlanCache : 0); }
    __device__ FoldState* fstate() const { return reinterpret_cast<FoldState*>(planc() + kPlans); }
    __device__ double* fbuf() const { return reinterpret_cast<double*>(base + kBars); }
};

// Copies a plan blob into shared memory (whole warp); returns the pointer to
// use (the global copy when it does not fit).
__device__ __forceinline__ const char* cache_plan(const char* g, char* s) {
    const PlanHeader* h = reinterpret_cast<const PlanHeader*>(g);
    const int bytes = h->ops_off + 16 * h->nops;
    if (bytes > kPlanCache) return g;
    const int4* src = reinterpret_cast<const int4*>(g);
    int4* dst = reinterpret_cast<int4*>(s);
    for (int i = threadIdx.x & 31; i < (bytes + 15) / 16; i += 32) dst[i] = src[i];
    __syncwarp();
    return s;
}

// Leaves [lo, hi) of `plan` over the stash (segment element e = block row
// 1 + e at stash row (rowbase + e) & mask).  One (leaf, lane) item per
// warp lane; the item's <= 16 elements are loaded before the in-order adds.
template <typename V, int NACC>
__device__ __forceinline__ void red_leaves(const char* plan, const V* stash, uint32_t rowbase, V* nodes, int lo,
                                           int hi, uint32_t mask) {
    constexpr int LANES = VT<V>::lanes;
    constexpr int GMAX = (LANES == 4 ? 64 : 128) / LANES;  // 16
    const PlanHeader* h = reinterpret_cast<const PlanHeader*>(plan);
    const int lane = threadIdx.x & 31;
    if (h->seq) {  // L < lanes: one sequential leaf from -0.0
        if (lane == 0) {
            V sacc[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) sacc[a] = VT<V>::negzero();
            for (int k = 0; k < h->L; ++k) {
                const uint32_t r = (rowbase + (uint32_t)k) & mask;
#pragma unroll
                for (int a = 0; a < NACC; ++a) sacc[a] = VT<V>::add(sacc[a], stash[r * NACC + a]);
            }
#pragma unroll
            for (int a = 0; a < NACC; ++a) nodes[a] = sacc[a];
        }
        return;
    }
    const int2* leaves = reinterpret_cast<const int2*>(plan + h->leaves_off);
    const int q = lane & (LANES - 1);
    for (int it0 = lo * LANES; it0 < hi * LANES; it0 += 32) {
        const int itm = it0 + lane;
        const bool valid = itm < hi * LANES;
        const int leaf = itm / LANES;
        const int2 lf = valid ? leaves[leaf] : make_int2(0, 0);
        const int G = lf.y / LANES;
        const int rem = lf.y - G * LANES;
        const uint32_t r0 = rowbase + (uint32_t)(lf.x + q);
        V vals[GMAX][NACC];
#pragma unroll
        for (int g = 0; g < GMAX; ++g) {
            if (g < G) {
                const uint32_t r = (r0 + (uint32_t)(LANES * g)) & mask;
#pragma unroll
                for (int a = 0; a < NACC; ++a) vals[g][a] = stash[r * NACC + a];
            }
        }
        V acc[NACC];
#pragma unroll
        for (int a = 0; a < NACC; ++a) acc[a] = vals[0][a];
#pragma unroll
        for (int g = 1; g < GMAX; ++g) {
            if (g < G) {
#pragma unroll
                for (int a = 0; a < NACC; ++a) acc[a] = VT<V>::add(acc[a], vals[g][a]);
            }
        }
        // lane tree: (l0+l1)+(l2+l3) [+ ((l4+l5)+(l6+l7)) for real]
#pragma unroll
        for (int d = 1; d < LANES; d <<= 1) {
#pragma unroll
            for (int a = 0; a < NACC; ++a) {
                V o = VT<V>::shfl_down(acc[a], d);
                if ((q & (2 * d - 1)) == 0) acc[a] = VT<V>::add(acc[a], o);
            }
        }
        // leftovers (q < rem), added in order by the leaf's lane 0
        V left[NACC];
        const uint32_t rl = (r0 + (uint32_t)(LANES * G)) & mask;
#pragma unroll
        for (int a = 0; a < NACC; ++a) left[a] = (valid && q < rem) ? stash[rl * NACC + a] : VT<V>::zero();
        const int grp = lane & ~(LANES - 1);
#pragma unroll
        for (int j = 0; j < LANES - 1; ++j) {
#pragma unroll
            for (int a = 0; a < NACC; ++a) {
                V o = VT<V>::shfl(left[a], grp + j);
                if (j < rem) acc[a] = VT<V>::add(acc[a], o);
            }
        }
        if (valid && q == 0) {
#pragma unroll
            for (int a = 0; a < NACC; ++a) nodes[leaf * NACC + a] = acc[a];
        }
    }
}

// Internal nodes in the plan's round order (one warp, __syncwarp per round).
template <typename V, int NACC>
__device__ __forceinline__ void red_tree(const char* plan, V* nodes, V (&pw)[NACC]) {
    const PlanHeader* h = reinterpret_cast<const PlanHeader*>(plan);
    const int lane = threadIdx.x & 31;
    if (h->L <= 0) return;
    __syncwarp();
    if (!h->seq) {
        const int4* ops = reinterpret_cast<const int4*>(plan + h->ops_off);
        for (int r = 0; r < h->nrounds; ++r) {
            const int lo = h->round_off[r], hi = h->round_off[r + 1];
            for (int o = lo + lane; o < hi; o += 32) {
                const int4 opn = ops[o];
#pragma unroll
                for (int a = 0; a < NACC; ++a)
                    nodes[opn.x * NACC + a] = VT<V>::add(nodes[opn.y * NACC + a], nodes[opn.z * NACC + a]);
            }
            __syncwarp();
        }
    }
#pragma unroll
    for (int a = 0; a < NACC; ++a) pw[a] = nodes[h->root * NACC + a];
}

template <int NC, int NR, class Body>
__device__ __noinline__ void reducer_warp(const SellView A, Body body, const RedCfg R, RedSmem<NC, NR> sm) {
    constexpr int NP = 2 * NC + NR;
    constexpr int kBatchC = RedSmem<NC, NR>::kBatchRows / 64, kBatchR = RedSmem<NC, NR>::kBatchRows / 128;
    const int lane = threadIdx.x & 31;
    const char* pc_full = NC ? cache_plan(R.pc.full, sm.planc()) : nullptr;
    const char* pr_full = NR ? cache_plan(R.pr.full, sm.planr()) : nullptr;
    const bool stream = R.slots != nullptr;
    uint32_t m = 0;  // CTA slice sequence number of the block's first slice
    for (int64_t blk = blockIdx.x; blk < A.nblocks; blk += gridDim.x) {
        const int64_t base = blk * kBlock;
        const int64_t nrows = (A.n_rows - base < kBlock) ? A.n_rows - base : kBlock;
        const int nsl = (int)((nrows + kSlice - 1) / kSlice);
        const char* pcp = nullptr;
        const char* prp = nullptr;
        if (NC) pcp = nrows == kBlock ? pc_full : R.pc.tail;
        if (NR) prp = nrows == kBlock ? pr_full : R.pr.tail;
        const PlanHeader* hc = reinterpret_cast<const PlanHeader*>(pcp);
        const PlanHeader* hr = reinterpret_cast<const PlanHeader*>(prp);
        const int nlc = NC ? hc->nleaves : 0, nlr = NR ? hr->nleaves : 0;
        const uint32_t rowbase = m * kSlice + 1;  // stash row of segment element 0 (block row 1)
        int lc = 0, lr = 0, rel = 0;
        double2 v0c[NC > 0 ? NC : 1];
        double v0r[NR > 0 ? NR : 1];
        for (int j = 0; j < nsl; ++j) {
            const uint32_t sq = m + (uint32_t)j;
            mbar_wait(&sm.sfull()[sq % RedSmem<NC, NR>::kSlots], (sq / RedSmem<NC, NR>::kSlots) & 1);
            const bool lastj = j + 1 == nsl;
            if (j == 0) {
                const int k0 = (int)((m * kSlice) & RedSmem<NC, NR>::kMask);
#pragma unroll
                for (int a = 0; a < NC; ++a) v0c[a] = sm.stc()[k0 * NC + a];
#pragma unroll
                for (int a = 0; a < NR; ++a) v0r[a] = sm.str()[k0 * NR + a];
            }
            int need = (int)nrows;  // first block row a pending leaf still reads
            bool worked = false;
            if constexpr (NC > 0) {
                const int hi = lastj ? nlc : min((int)hc->leaf_upto[j + 1], nlc);
                if (hi - lc >= kBatchC || (lastj && hi > lc)) {
                    red_leaves<double2, NC>(pcp, sm.stc(), rowbase, sm.ndc(), lc, hi, RedSmem<NC, NR>::kMask);
                    lc = hi;
                    worked = true;
                }
                if (lc < nlc) need = min(need, 1 + reinterpret_cast<const int2*>(pcp + hc->leaves_off)[lc].x);
            }
            if constexpr (NR > 0) {
                const int hi = lastj ? nlr : min((int)hr->leaf_upto[j + 1], nlr);
                if (hi - lr >= kBatchR || (lastj && hi > lr)) {
                    red_leaves<double, NR>(prp, sm.str(), rowbase, sm.ndr(), lr, hi, RedSmem<NC, NR>::kMask);
                    lr = hi;
                    worked = true;
                }
                if (lr < nlr) need = min(need, 1 + reinterpret_cast<const int2*>(prp + hr->leaves_off)[lr].x);
            }
            const int upto = lastj ? nsl : min(j + 1, need / kSlice);
            if (upto > rel) {
                if (worked) __syncwarp();  // every lane is done reading the released rows
                if (lane == 0)
                    for (int k = rel; k < upto; ++k) mbar_arrive(&sm.sfree()[(m + (uint32_t)k) % RedSmem<NC, NR>::kSlots]);
                rel = upto;
            }
        }
        m += (uint32_t)nsl;
        double2 pwc[NC > 0 ? NC : 1];
        double pwr[NR > 0 ? NR : 1];
        if constexpr (NC > 0) red_tree<double2, NC>(pcp, sm.ndc(), pwc);
        if constexpr (NR > 0) red_tree<double, NR>(prp, sm.ndr(), pwr);
        if (stream) {
            if (lane == 0) {
                double* S = R.slots + blk * NP;
#pragma unroll
                for (int a = 0; a < NC; ++a) {
                    const double2 t = hc->L > 0 ? cadd(v0c[a], pwc[a]) : v0c[a];
                    slot_store(S + 2 * a, t.x);
                    slot_store(S + 2 * a + 1, t.y);
                }
#pragma unroll
                for (int a = 0; a < NR; ++a) slot_store(S + 2 * NC + a, hr->L > 0 ? __dadd_rn(v0r[a], pwr[a]) : v0r[a]);
            }
            continue;
        }
        unsigned int last = 0;
        if (lane == 0) {
            double* P = R.partials + blk * NP;
#pragma unroll
            for (int a = 0; a < NC; ++a) {
                const double2 t = hc->L > 0 ? cadd(v0c[a], pwc[a]) : v0c[a];
                P[2 * a] = t.x;
                P[2 * a + 1] = t.y;
            }
#pragma unroll
            for (int a = 0; a < NR; ++a) P[2 * NC + a] = hr->L > 0 ? __dadd_rn(v0r[a], pwr[a]) : v0r[a];
            __threadfence();
            last = (atomicAdd(R.counter, 1u) == (unsigned)A.nblocks - 1) ? 1u : 0u;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        __syncwarp();
        if (last && R.defer) {  // this rank's partials are complete; the ranks fold together
            if (lane == 0) *R.counter = 0;
        } else if (last) {
            __threadfence();
            double tot[NP];
            // the stash is free now (every slice of this CTA was reduced): fold scratch
            static_assert(RedSmem<NC, NR>::kStashC + RedSmem<NC, NR>::kStashR >= 2 * kFoldStage * 8, "fold scratch");
            warp_fold<double>(R.partials, NP, A.nblocks, reinterpret_cast<double*>(sm.stc()), tot);
            if (lane == 0) body.finish(tot);
        }
    }
    // streaming fold: the last CTA -- one block fewer than the first CTAs
    // when the blocks do not divide evenly -- folds the partials in block
    // order as they land once its own blocks are done (its stash is free:
    // staging), so the fold overlaps the other CTAs' last blocks
    if (stream && blockIdx.x == gridDim.x - 1) {
        if (lane == 0) sm.fstate()->pos = 0;
        if (lane < NP) sm.fstate()->tot[lane] = -0.0;
        __syncwarp();
        fold_progress<NP, RedSmem<NC, NR>::kFoldPer>(R.slots, (long long)A.nblocks * NP, sm.fstate(), sm.fbuf(), true);
        if (lane == 0) body.finish(sm.fstate()->tot);
    }
}

// Persistent pipelined SpMV over the CTA's 4096-row blocks (blk = blockIdx.x,
// +gridDim.x, ...).  For each row the consumer thread calls
// body.row(row, values, svals, tc, tr), which stores the row's outputs and
// returns its Body::kNC complex / Body::kNR real reduction terms (see
// reducer_warp; plain bodies have none, PipeWarps gives the warp roles).
// svals are the row's entries of the Body::kSV vectors A.sv[] (the
// epilogue's operands), which the producer stages with the slice by TMA, so
// they cost the consumer neither registers nor load latency.  NX = 2 multiplies the matrix with two vectors in
// one pass over it.  `smem` holds kBarBytes + ns*stage_bytes + RedSmem bytes.
template <bool SWAP, int NX, class Body>
__device__ __forceinline__ void sell_pipeline(const SellView& A, const double2* __restrict__ x0,
                                              const double2* __restrict__ x1, Body& body, const RedCfg& R,
                                              unsigned char* smem) {
    constexpr int NC = Body::kNC, NR = Body::kNR;
    constexpr bool kRed = (NC + NR) > 0;
    constexpr int kCW = PipeWarps<kRed>::consumers;
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
    RedSmem<NC, NR> sm{ring + (size_t)A.ns * A.stage_bytes};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ns = A.ns, nch = A.nch;
    const int cols = 1 + 4 * A.cm;
    // pipeline block: the 4096-row reduction block for fused reductions,
    // A.spb slices otherwise
    const int kSlicesPerBlock = kRed ? kBlock / kSlice : A.spb;
    const int64_t nblk = kRed ? A.nblocks : A.nvb;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            tag[i] = 0xffffffffu;
        }
        if (kRed) {
            for (int i = 0; i < RedSmem<NC, NR>::kSlots; ++i) {
                mbar_init(&sm.sfull()[i], 1);
                mbar_init(&sm.sfree()[i], 1);
            }
        }
        mbar_fence_init();
    }
    __syncthreads();
    if constexpr (kRed) {
        if (warp == PipeWarps<kRed>::reducer) {
            reducer_warp<NC, NR>(A, body, R, sm);
            return;
        }
    }
    if (warp == PipeWarps<kRed>::producer) {  // producer warp: lane l owns ring stage l
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
        int32_t cm_hi = -1, cm_lo = 0;  // x columns to prefetch for chunk i
        auto locate = [&]() {  // coordinates + offsets of chunk i (loads issued early)
            const uint32_t seq = i / (uint32_t)nch;
            c = (int)(i % (uint32_t)nch);
            const int64_t blk = blockIdx.x + (int64_t)(seq / kSlicesPerBlock) * gridDim.x;
            s = blk * kSlicesPerBlock + (seq % kSlicesPerBlock);
            active = blk < nblk && s < A.nslices;
            if (active) {
                off0 = __ldg(A.slice_off + s);
                off1 = __ldg(A.slice_off + s + 1);
                // leading edge of the x window: columns above the previous
                // slice's largest (a block's first slice: the 4096 below its own)
                cm_hi = __ldg(A.slice_cmax + s);
                cm_lo = (s % kSlicesPerBlock != 0) ? __ldg(A.slice_cmax + s - 1) + 1
                                                   : cm_hi - (kSlicesPerBlock * kSlice - 1);
                if (cm_lo < 0) cm_lo = 0;
            }
        };
        if (owner) locate();
        while (__any_sync(0xffffffffu, owner && active)) {
            if (owner && active && (u == 0 || mbar_test(&empty[lane], (u - 1) & 1))) {
                w = (int)((off1 - off0) / kSlice);
                tag[lane] = i;
                unsigned char* stage = ring + (size_t)lane * A.stage_bytes;
                if (A.cm == 0) {  // whole slice + its row lengths + the staged vector rows
                    wid[lane] = (uint32_t)w;
                    const uint32_t cnt = (uint32_t)w * kSlice;
                    const int64_t r0 = s * kSlice;
                    const uint32_t vrows = (uint32_t)min((int64_t)kSlice, A.n_rows - r0);
                    mbar_arrive_expect_tx(&full[lane], cnt * 20u + kSlice + (uint32_t)A.nsv * vrows * 16u);
                    if (cnt) {
                        bulk_g2s(stage, A.aa + off0, cnt * 16u, &full[lane], pol);
                        bulk_g2s(stage + A.ja_off, A.ja + off0, cnt * 4u, &full[lane], pol);
                    }
                    bulk_g2s(stage + A.rl_off, A.rowlen + r0, kSlice, &full[lane], pol);
                    for (int v = 0; v < A.nsv; ++v)
                        bulk_g2s(stage + A.sv_off + v * kSlice * 16, A.sv[v] + r0, vrows * 16u, &full[lane], pol);
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
                if (c == 0 && cm_hi >= cm_lo && A.prefetch) {  // x rows this slice is first to touch -> L2
                    const uint32_t nb = (uint32_t)min(cm_hi - cm_lo + 1, 4096) * 16u;
                    bulk_prefetch_l2(x0 + cm_lo, nb);
                    if (x1) bulk_prefetch_l2(x1 + cm_lo, nb);
                }
                i += (uint32_t)ns;
                ++u;
                locate();
            }
        }
        return;
    }
    // ---- consumer warps: warp w takes slices w, w+kCW, ... of each block ----
    const bool fast = A.cm == 0 && A.fma;
    uint32_t sbase = 0;  // CTA-local index of the block's first slice
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t s_lo = blk * kSlicesPerBlock;
        const int64_t s_hi = (s_lo + kSlicesPerBlock < A.nslices) ? s_lo + kSlicesPerBlock : A.nslices;
        const int nsl = (int)(s_hi - s_lo);
        for (int j = warp; j < nsl; j += kCW) {
            const int64_t row = (s_lo + j) * kSlice + lane;
            const uint32_t sq = sbase + (uint32_t)j;  // CTA slice sequence number
            const bool mine = row < A.n_rows;
            constexpr int SV = Body::kSV;
            double2 svals[SV > 0 ? SV : 1];  // the row's epilogue operands (staged with the slice)
            RowVals<NX> val;
            int len;
            if (fast) {
                const uint32_t q = __umulhi(sq, A.ns_magic);
                const int st = (int)(sq - q * (uint32_t)ns);
                while (tag[st] != sq) {
                }
                mbar_wait(&full[st], q & 1);
                const unsigned char* stage = ring + (size_t)st * A.stage_bytes;
                const int W = (int)wid[st];
                len = stage[A.rl_off + lane];
                val = row_fast_dispatch<SWAP, NX>(W, x0, x1, reinterpret_cast<const double2*>(stage),
                                                  reinterpret_cast<const int32_t*>(stage + A.ja_off), lane,
                                                  (mine && len != 255) ? len : 0, !mine);
#pragma unroll
                for (int v = 0; v < SV; ++v)
                    svals[v] = reinterpret_cast<const double2*>(stage + A.sv_off)[v * kSlice + lane];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            } else {
                len = A.rowlen[row];
                val = generic_slice<NX>(A, x0, x1, full, empty, tag, ring, sq, lane, (mine && len != 255) ? len : 0);
#pragma unroll
                for (int v = 0; v < SV; ++v) svals[v] = mine ? A.sv[v][row] : make_double2(0.0, 0.0);
            }
            // long rows (side CSR): the whole warp sums each in turn, out of
            // line and only for matrices that have any (keeps the hot loop's
            // registers and schedule)
            if (A.long_blk_ptr != nullptr) {
                const unsigned lm = __ballot_sync(0xffffffffu, mine && len == 255);
                if (lm) long_rows_slice<NX>(A, x0, x1, lm, row, val);
            }
            double2 tc[NC > 0 ? NC : 1];
            double tr[NR > 0 ? NR : 1];
            if (mine) body.row(row, val.v, svals, tc, tr);
            if (kRed) {
                if (sq >= (uint32_t)RedSmem<NC, NR>::kSlots) mbar_wait(&sm.sfree()[sq % RedSmem<NC, NR>::kSlots], ((sq / RedSmem<NC, NR>::kSlots) - 1) & 1);
                const int k = (int)((sq * kSlice + lane) & RedSmem<NC, NR>::kMask);
                if (mine) {
#pragma unroll
                    for (int a = 0; a < NC; ++a) sm.stc()[k * NC + a] = tc[a];
#pragma unroll
                    for (int a = 0; a < NR; ++a) sm.str()[k * NR + a] = tr[a];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.sfull()[sq % RedSmem<NC, NR>::kSlots]);
            }
        }
        sbase += (uint32_t)nsl;
    }
}

// Kernel-side dispatch on numpy's elision swap (a launch-uniform flag).
template <int NX, class Body>
__device__ __forceinline__ void sell_run(const SellView& A, const double2* __restrict__ x0,
                                         const double2* __restrict__ x1, Body& body, const RedCfg& R,
                                         unsigned char* smem) {
    if (A.swap) sell_pipeline<true, NX>(A, x0, x1, body, R, smem);
    else sell_pipeline<false, NX>(A, x0, x1, body, R, smem);
}

}  // namespace zk
