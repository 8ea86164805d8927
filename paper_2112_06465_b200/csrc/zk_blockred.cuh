// zk_blockred.cuh -- split block reduction for persistent kernels.
//
// Same arithmetic as block_reduce (zk_reduce.cuh) -- numpy's pairwise order
// inside the block, Python's left fold across blocks -- but organised so a
// block costs two barriers instead of a dozen: every participating thread
// runs the leaf phase (leaf_phase), one warp then combines the leaves in the
// plan's round order with __syncwarp only (warp_tree) while the other warps
// already start on the next block (the caller double-buffers the nodes), and
// the same warp stores the partial and counts the arrival (warp_finish).
// The warp that sees the last arrival folds every partial (warp_fold).
#pragma once
#include "zk_reduce.cuh"

namespace zk {

// Leaf phase over threads [0, nthr); no barrier inside.  The block's first
// element (v[0]) is handled by the caller.
template <typename V, int NACC, class Op>
__device__ __forceinline__ void leaf_phase(const char* plan, int64_t seg0, const Op& op, V* nodes, int nthr,
                                           int leaf_lo = 0, int leaf_hi = 1 << 30) {
    using Item = typename Op::Item;
    constexpr int LANES = VT<V>::lanes;
    constexpr int U = Op::U;
    const PlanHeader* h = plan_hdr(plan);
    const int L = h->L;
    if (L <= 0 || (int)threadIdx.x >= nthr) return;
    if (leaf_hi > h->nleaves) leaf_hi = h->nleaves;
    if (leaf_lo >= leaf_hi) return;
    if (h->seq) {
        if (threadIdx.x == 0) {
            V s[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) s[a] = VT<V>::negzero();
            for (int k = 0; k < L; ++k) {
                V v[NACC];
                Item it = op.load(seg0 + k);
                op.apply(seg0 + k, it, v);
#pragma unroll
                for (int a = 0; a < NACC; ++a) s[a] = VT<V>::add(s[a], v[a]);
            }
#pragma unroll
            for (int a = 0; a < NACC; ++a) nodes[a] = s[a];
        }
        return;
    }
    const int2* leaves = reinterpret_cast<const int2*>(plan + h->leaves_off);
    const int nitems = leaf_hi * LANES;
    const int lane = threadIdx.x & 31;
    const int q = lane & (LANES - 1);
    for (int it0 = leaf_lo * LANES + (threadIdx.x & ~31); it0 < nitems; it0 += nthr) {
        const int itm = it0 + lane;
        const bool valid = itm < nitems;
        const int leaf = itm / LANES;
        const int2 lf = valid ? __ldg(leaves + leaf) : make_int2(0, 0);
        const int G = lf.y / LANES;
        const int rem = lf.y - G * LANES;
        const int64_t e0 = seg0 + lf.x + q;
        const int64_t el = seg0 + lf.x + (int64_t)LANES * G + q;
        const bool has_left = valid && q < rem;
        Item left_item;
        if (has_left) left_item = op.load(el);
        V acc[NACC];
#pragma unroll
        for (int a = 0; a < NACC; ++a) acc[a] = VT<V>::zero();
        if (valid) {
            for (int g0 = 0; g0 < G; g0 += U) {
                Item items[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (g0 + u < G) items[u] = op.load(e0 + (int64_t)LANES * (g0 + u));
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (g0 + u < G) {
                        V v[NACC];
                        op.apply(e0 + (int64_t)LANES * (g0 + u), items[u], v);
#pragma unroll
                        for (int a = 0; a < NACC; ++a) acc[a] = (g0 + u == 0) ? v[a] : VT<V>::add(acc[a], v[a]);
                    }
                }
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
        // leftover elements, owned by lanes q < rem, added in order by lane 0
        V left[NACC];
        if (has_left) {
            op.apply(el, left_item, left);
        } else {
#pragma unroll
            for (int a = 0; a < NACC; ++a) left[a] = VT<V>::zero();
        }
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

// Leaf phase run by a single warp over leaves [leaf_lo, leaf_hi) (the
// reducer warp of the SpMV pipelines); same item mapping and order as
// leaf_phase with the warp's lane as the thread index.
template <typename V, int NACC, class Op>
__device__ __forceinline__ void warp_leaves(const char* plan, int64_t seg0, const Op& op, V* nodes, int leaf_lo,
                                            int leaf_hi) {
    constexpr int LANES = VT<V>::lanes;
    const PlanHeader* h = plan_hdr(plan);
    const int L = h->L;
    const int lane = threadIdx.x & 31;
    if (L <= 0) return;
    if (leaf_hi > h->nleaves) leaf_hi = h->nleaves;
    if (leaf_lo >= leaf_hi) return;
    if (h->seq) {
        if (lane == 0) {
            V s[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) s[a] = VT<V>::negzero();
            for (int k = 0; k < L; ++k) {
                V v[NACC];
                typename Op::Item it = op.load(seg0 + k);
                op.apply(seg0 + k, it, v);
#pragma unroll
                for (int a = 0; a < NACC; ++a) s[a] = VT<V>::add(s[a], v[a]);
            }
#pragma unroll
            for (int a = 0; a < NACC; ++a) nodes[a] = s[a];
        }
        return;
    }
    const int2* leaves = reinterpret_cast<const int2*>(plan + h->leaves_off);
    const int nitems = leaf_hi * LANES;
    const int q = lane & (LANES - 1);
    for (int it0 = leaf_lo * LANES; it0 < nitems; it0 += 32) {
        const int itm = it0 + lane;
        const bool valid = itm < nitems;
        const int leaf = itm / LANES;
        const int2 lf = valid ? __ldg(leaves + leaf) : make_int2(0, 0);
        const int G = lf.y / LANES;
        const int rem = lf.y - G * LANES;
        const int64_t e0 = seg0 + lf.x + q;
        V acc[NACC];
#pragma unroll
        for (int a = 0; a < NACC; ++a) acc[a] = VT<V>::zero();
        if (valid) {
            for (int g = 0; g < G; ++g) {
                V v[NACC];
                op.apply(e0 + (int64_t)LANES * g, typename Op::Item{}, v);
#pragma unroll
                for (int a = 0; a < NACC; ++a) acc[a] = (g == 0) ? v[a] : VT<V>::add(acc[a], v[a]);
            }
        }
#pragma unroll
        for (int d = 1; d < LANES; d <<= 1) {
#pragma unroll
            for (int a = 0; a < NACC; ++a) {
                V o = VT<V>::shfl_down(acc[a], d);
                if ((q & (2 * d - 1)) == 0) acc[a] = VT<V>::add(acc[a], o);
            }
        }
        V left[NACC];
        if (valid && q < rem) {
            op.apply(seg0 + lf.x + (int64_t)LANES * G + q, typename Op::Item{}, left);
        } else {
#pragma unroll
            for (int a = 0; a < NACC; ++a) left[a] = VT<V>::zero();
        }
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

// One full warp combines the leaves (after a barrier made them visible).
// Every lane returns PW of the segment in `pw` (untouched when L == 0).
template <typename V, int NACC>
__device__ __forceinline__ void warp_tree(const char* plan, V* nodes, V (&pw)[NACC]) {
    const PlanHeader* h = plan_hdr(plan);
    const int lane = threadIdx.x & 31;
    if (h->L <= 0) return;
    if (!h->seq) {
        const int4* ops = reinterpret_cast<const int4*>(plan + h->ops_off);
        for (int r = 0; r < h->nrounds; ++r) {
            const int lo = h->round_off[r], hi = h->round_off[r + 1];
            for (int o = lo + lane; o < hi; o += 32) {
                const int4 opn = __ldg(ops + o);
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

// Lane 0 of the finishing warp stores partial = v0 + PW (v0 alone when the
// segment is empty) and counts the arrival.  Warp-uniform result: true when
// this was the last of `total` arrivals.
template <typename V, int NACC>
__device__ __forceinline__ bool warp_finish(const char* plan, const V (&v0)[NACC], const V (&pw)[NACC], V* partials,
                                            int64_t blk, unsigned int* counter, unsigned int total) {
    const int lane = threadIdx.x & 31;
    unsigned int last = 0;
    if (lane == 0) {
        const bool has = plan_hdr(plan)->L > 0;
#pragma unroll
        for (int a = 0; a < NACC; ++a) partials[blk * NACC + a] = has ? VT<V>::add(v0[a], pw[a]) : v0[a];
        __threadfence();
        last = (atomicAdd(counter, 1u) == total - 1) ? 1u : 0u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) __threadfence();
    return last != 0;
}

// Ordered fold core.  partials holds nb rows of nchains doubles; lane c
// (< nchains) adds column c to `tot` in row order (__dadd_rn: the Python
// left fold, one rounding per add).  The serial add chain is the critical
// path, so nothing else may sit on it: the warp stages kFoldStage doubles
// at a time into a double-buffered smem window (scratch: 2*kFoldStage
// doubles) with the next window's __ldcg loads issued before the current
// window is folded, and each chain lane reads 16 values into registers
// ahead of its 16 dependent adds (an LDS per add left the smem latency on
// the chain: ~19 cycles per partial, measured).
constexpr int kFoldStage = 256;

__device__ __forceinline__ void fold_stream(const double* partials, int nchains, int64_t nb, double* scratch,
                                            double& tot) {
    constexpr int PER = kFoldStage / 32;
    const int lane = threadIdx.x & 31;
    const int64_t total = nb * nchains;
    double r[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int64_t i = (int64_t)k * 32 + lane;
        r[k] = i < total ? __ldcg(partials + i) : 0.0;
    }
    int stage = 0;
    for (int64_t e0 = 0; e0 < total; e0 += kFoldStage, stage ^= 1) {
        double* buf = scratch + stage * kFoldStage;
#pragma unroll
        for (int k = 0; k < PER; ++k) buf[k * 32 + lane] = r[k];
        __syncwarp();
        const int64_t e1 = (total - e0 < kFoldStage) ? total : e0 + kFoldStage;
        if (e1 < total) {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int64_t i = e1 + (int64_t)k * 32 + lane;
                r[k] = i < total ? __ldcg(partials + i) : 0.0;
            }
        }
        if (lane < nchains) {
            int j = (int)(((int64_t)lane - e0 % nchains + nchains) % nchains);  // first index of chain in window
            const int n = (int)(e1 - e0);
            for (; j + 15 * nchains < n; j += 16 * nchains) {
                double v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = buf[j + k * nchains];
#pragma unroll
                for (int k = 0; k < 16; ++k) tot = __dadd_rn(tot, v[k]);
            }
            for (; j < n; j += nchains) tot = __dadd_rn(tot, buf[j]);
        }
    }
    __syncwarp();
}

// Ordered fold of chains continued across calls: lane c (< nchains) adds
// partials[b*nchains + c] for b < nb to its running total `tot` (first
// call: first = true starts the chain; -0.0 + p == p for every p, so
// starting from -0.0 is the left fold that starts at partials[c]).
__device__ __forceinline__ void warp_fold_cont(const double* partials, int nchains, int64_t nb, double* scratch,
                                               double& tot, bool first) {
    if (first) tot = -0.0;
    fold_stream(partials, nchains, nb, scratch, tot);
}

// Ordered fold by one warp (vecops.py:159-161): lane c (< nacc*NC) folds the
// real component chain c.  scratch: 2*kFoldStage doubles.  Result (nacc
// values) valid in lane 0.
template <typename V>
__device__ __forceinline__ void warp_fold(const V* partials, int nacc, int64_t nb, V* scratch, V* result) {
    constexpr int NC = sizeof(V) / sizeof(double);
    const int lane = threadIdx.x & 31;
    const int nchains = nacc * NC;
    double tot = -0.0;
    fold_stream(reinterpret_cast<const double*>(partials), nchains, nb, reinterpret_cast<double*>(scratch), tot);
    double* r = reinterpret_cast<double*>(result);
    for (int c = 0; c < nchains; ++c) {
        const double v = __shfl_sync(0xffffffffu, tot, c);
        if (lane == 0) r[c] = v;
    }
}

// ---- streaming ordered fold ---------------------------------------------------
// Block partials published into slots that hold kSlotEmpty (a signalling
// NaN: arithmetic never produces one, NaN results are quiet) until their
// value lands; one warp folds them in block order while the pass is still
// running and re-marks each consumed slot empty for the next pass.  No
// fence or atomic per block: each slot is its own flag.
constexpr unsigned long long kSlotEmpty = 0x7FF47FF47FF47FF4ull;
constexpr int kPollPer = 16;  // slots per lane in flight per poll round

__device__ __forceinline__ void slot_store(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double slot_load(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// tot += buf[j0 + m*NCH] for m < cnt in order, the smem loads of the next
// 16 issued ahead of the current 16 dependent adds (the chain stays pure
// DADD, ~14 cycles per add on B200).
template <int NCH>
__device__ __forceinline__ double chain_fold(double tot, const double* buf, int j0, int cnt) {
    const double* q = buf + j0;
    int m = 0;
    if (cnt >= 16) {
        double w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = q[k * NCH];
        for (; m + 32 <= cnt; m += 16) {
            double u[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) u[k] = q[(m + 16 + k) * NCH];
#pragma unroll
            for (int k = 0; k < 16; ++k) tot = __dadd_rn(tot, w[k]);
#pragma unroll
            for (int k = 0; k < 16; ++k) w[k] = u[k];
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) tot = __dadd_rn(tot, w[k]);
        m += 16;
    }
    for (; m < cnt; ++m) tot = __dadd_rn(tot, q[m * NCH]);
    return tot;
}

// Fold nrows*NCH slots in row order, lane c < NCH carrying chain c (column
// c); result[0..NCH) valid in lane 0.  Whole warp.  Per round the warp
// polls 32*kPollPer slots with all loads in flight, waits for the missing
// ones, re-marks them empty and stages them in smem; the next round's loads
// are issued before this round is folded, so the poll's L2 round trip
// overlaps the add chain (the chain starts from -0.0: -0.0 + p == p, the
// left fold starting at the first partial).
template <int NCH>
__device__ __forceinline__ void stream_fold(double* slots, int64_t nrows, double* result) {
    constexpr int W = 32 * kPollPer;
    __shared__ double sbuf[2 * W];
    const int lane = threadIdx.x & 31;
    const int64_t total = nrows * NCH;
    const double empty = __longlong_as_double((long long)kSlotEmpty);
    double tot = -0.0;
    double v[kPollPer];
#pragma unroll
    for (int k = 0; k < kPollPer; ++k) {
        const int64_t i = k * 32 + lane;
        v[k] = i < total ? slot_load(slots + i) : 0.0;
    }
    int stage = 0;
    for (int64_t e0 = 0; e0 < total; e0 += W, stage ^= 1) {
        double* buf = sbuf + stage * W;
#pragma unroll
        for (int k = 0; k < kPollPer; ++k) {
            const int64_t i = e0 + k * 32 + lane;
            if (i < total) {
                while ((unsigned long long)__double_as_longlong(v[k]) == kSlotEmpty) {
                    __nanosleep(32);
                    v[k] = slot_load(slots + i);
                }
                slot_store(slots + i, empty);
            }
            buf[k * 32 + lane] = v[k];
        }
        __syncwarp();
        const int64_t e1 = e0 + W;
        if (e1 < total) {
#pragma unroll
            for (int k = 0; k < kPollPer; ++k) {
                const int64_t i = e1 + k * 32 + lane;
                v[k] = i < total ? slot_load(slots + i) : 0.0;
            }
        }
        if (lane < NCH) {
            const int nw = (int)(total - e0 < W ? total - e0 : W);
            const int j0 = (int)(((int64_t)lane - e0 % NCH + NCH) % NCH);
            const int cnt = nw > j0 ? (nw - j0 + NCH - 1) / NCH : 0;
            tot = chain_fold<NCH>(tot, buf, j0, cnt);
        }
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const double t = __shfl_sync(0xffffffffu, tot, c);
        if (lane == 0) result[c] = t;
    }
}

// Incremental form of stream_fold for a folder warp that also has other
// work (the SpMV reducer): folds the contiguous ready prefix of the slots
// from fs->pos on, in whole rows of NCH, and returns when it meets a slot
// that has not landed (blocking = false) or when all `total` slots are
// folded (blocking = true).  State lives in shared memory between calls;
// buf: 32*PER doubles of staging.  Whole warp.
struct FoldState {
    long long pos;  // next slot to fold (a multiple of NCH)
    double tot[4];  // running chains
};

template <int NCH, int PER>
__device__ __noinline__ void fold_progress(double* slots, long long total, FoldState* fs, double* buf, bool blocking) {
    constexpr int W = 32 * PER;
    const int lane = threadIdx.x & 31;
    const double empty = __longlong_as_double((long long)kSlotEmpty);
    long long pos = fs->pos;
    double tot = lane < NCH ? fs->tot[lane] : 0.0;
    while (pos < total) {
        double v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const long long i = pos + k * 32 + lane;
            v[k] = i < total ? slot_load(slots + i) : 0.0;
        }
        int first_missing = W;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const long long i = pos + k * 32 + lane;
            const unsigned miss = __ballot_sync(0xffffffffu, i < total && (unsigned long long)__double_as_longlong(v[k]) == kSlotEmpty);
            if (miss && first_missing == W) first_missing = k * 32 + __ffs(miss) - 1;
        }
        long long navail = total - pos < first_missing ? total - pos : first_missing;
        navail -= navail % NCH;
        if (navail == 0) {
            if (!blocking) break;
            __nanosleep(64);
            continue;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int j = k * 32 + lane;
            if (j < navail) {
                slot_store(slots + pos + j, empty);
                buf[j] = v[k];
            }
        }
        __syncwarp();
        if (lane < NCH) tot = chain_fold<NCH>(tot, buf, lane, (int)(navail / NCH));
        __syncwarp();
        pos += navail;
    }
    if (lane < NCH) fs->tot[lane] = tot;
    if (lane == 0) fs->pos = pos;
    __syncwarp();
}

}  // namespace zk
