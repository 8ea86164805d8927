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

// Ordered fold of chains continued across calls: lane c (< nchains) adds
// partials[b*nchains + c] for b < nb to its running total `tot` (first
// call: first = true starts the chain at partials[c]).  Whole warp.
__device__ __forceinline__ void warp_fold_cont(const double* partials, int nchains, int64_t nb, double* scratch,
                                               int chunk, double& tot, bool first) {
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = 0; c0 < nb; c0 += chunk) {
        const int64_t cn = (nb - c0 < chunk) ? nb - c0 : chunk;
        for (int64_t i = lane; i < cn * nchains; i += 32) scratch[i] = __ldcg(partials + c0 * nchains + i);
        __syncwarp();
        if (lane < nchains) {
            int64_t b = 0;
            if (first && c0 == 0) {
                tot = scratch[lane];
                b = 1;
            }
#pragma unroll 16
            for (; b < cn; ++b) tot = __dadd_rn(tot, scratch[b * nchains + lane]);
        }
        __syncwarp();
    }
}

// Ordered fold by one warp (vecops.py:159-161): lane c (< nacc*NC) folds the
// real component chain c; partials are staged through `scratch` (chunk*nacc
// values).  Result (nacc values) valid in lane 0.
template <typename V>
__device__ __forceinline__ void warp_fold(const V* partials, int nacc, int64_t nb, V* scratch, int chunk, V* result) {
    constexpr int NC = sizeof(V) / sizeof(double);
    const int lane = threadIdx.x & 31;
    const int nchains = nacc * NC;
    const int a = lane / NC, comp = lane % NC;
    const double* sd = reinterpret_cast<const double*>(scratch);
    double tot = 0.0;
    for (int64_t c0 = 0; c0 < nb; c0 += chunk) {
        const int64_t cn = (nb - c0 < chunk) ? nb - c0 : chunk;
        const int64_t nv = cn * nacc;
        for (int64_t i = lane; i < nv; i += 32) scratch[i] = __ldcg(partials + c0 * nacc + i);
        __syncwarp();
        if (lane < nchains) {
            int64_t b = 0;
            if (c0 == 0) {
                tot = sd[a * NC + comp];
                b = 1;
            }
#pragma unroll 16
            for (; b < cn; ++b) tot = __dadd_rn(tot, sd[(b * nacc + a) * NC + comp]);
        }
        __syncwarp();
    }
    double* r = reinterpret_cast<double*>(result);
    for (int c = 0; c < nchains; ++c) {
        const double v = __shfl_sync(0xffffffffu, tot, c);
        if (lane == 0) r[c] = v;
    }
}

}  // namespace zk
