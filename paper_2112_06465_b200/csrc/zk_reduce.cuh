// zk_reduce.cuh -- per-block numpy-order reductions and the ordered fold.
//
// One CTA (or the consumer warps of one CTA) owns one reduction block
// (block_size consecutive elements, the ReductionPlan granularity of
// vecops.py:89-109).  The block partial is v[0] + PW(v[1:]) in numpy's exact
// pairwise order (zk_plan.h).  Each (leaf, lane) pair of the plan is one work
// item; the lane's elements are leaf_start + lanes*g + q, exactly the
// elements numpy's lane accumulator q visits, so the accumulation order is
// bit-identical.
//
// Element work is an `Op` with two steps so loads can run ahead of the
// in-order accumulation:  `Item load(e)` issues the global loads for element
// e, `apply(e, item, v)` performs the fused elementwise update for e (each
// element is visited exactly once) and returns its reduction term(s).  A
// lane prefetches Op::U elements before applying them in order, which keeps
// U x (bytes per element) in flight per thread -- the block pass is an HBM
// stream, and without this it is latency-bound.
//
// Block partials are folded left to right (vecops.py:159-161) by the CTA
// that finishes last (threadfence + arrival counter), staged through shared
// memory so the serial chain runs at DADD latency.
#pragma once
#include "zk_common.cuh"
#include "zk_pipe.cuh"
#include "zk_plan.h"

namespace zk {

template <typename V> struct VT;
template <> struct VT<double2> {
    static constexpr int lanes = 4;
    static __device__ __forceinline__ double2 add(double2 a, double2 b) { return cadd(a, b); }
    static __device__ __forceinline__ double2 negzero() { return make_double2(-0.0, -0.0); }
    static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
    static __device__ __forceinline__ double2 shfl(double2 v, int src) {
        return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
    }
    static __device__ __forceinline__ double2 shfl_down(double2 v, int d) {
        return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
    }
};
template <> struct VT<double> {
    static constexpr int lanes = 8;
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double negzero() { return -0.0; }
    static __device__ __forceinline__ double zero() { return 0.0; }
    static __device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
    static __device__ __forceinline__ double shfl_down(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
};

struct PlanPtrs {
    const char* full;  // plan for full blocks (L = block_size - 1)
    const char* tail;  // plan for the last, partial block (may equal full)
};

__device__ __forceinline__ const PlanHeader* plan_hdr(const char* p) { return reinterpret_cast<const PlanHeader*>(p); }

// Block pass over segment base `seg0` (global index of v[1]).  On return
// (after a barrier) nodes[root*NACC + a] holds PW of the segment.
template <typename V, int NACC, class Op, class Sync>
__device__ __forceinline__ void block_pass(const char* plan, int64_t seg0, const Op& op, V* nodes, Sync sync) {
    using Item = typename Op::Item;
    constexpr int LANES = VT<V>::lanes;
    constexpr int U = Op::U;
    const PlanHeader* h = plan_hdr(plan);
    const int L = h->L;
    const int nthr = sync.nthreads();
    if (L > 0 && (int)threadIdx.x < nthr) {
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
        } else {
            const int2* leaves = reinterpret_cast<const int2*>(plan + h->leaves_off);
            const int nitems = h->nleaves * LANES;
            const int lane = threadIdx.x & 31;
            const int q = lane & (LANES - 1);
            for (int it0 = (threadIdx.x & ~31); it0 < nitems; it0 += nthr) {
                const int itm = it0 + lane;
                const bool valid = itm < nitems;
                const int leaf = itm / LANES;
                const int2 lf = valid ? leaves[leaf] : make_int2(0, 0);
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
    }
    sync();
    if (L > 0 && !h->seq) {
        const int4* ops = reinterpret_cast<const int4*>(plan + h->ops_off);
        for (int r = 0; r < h->nrounds; ++r) {
            const int lo = h->round_off[r], hi = h->round_off[r + 1];
            for (int o = lo + (int)threadIdx.x; o < hi; o += nthr) {
                int4 opn = ops[o];
#pragma unroll
                for (int a = 0; a < NACC; ++a)
                    nodes[opn.x * NACC + a] = VT<V>::add(nodes[opn.y * NACC + a], nodes[opn.z * NACC + a]);
            }
            sync();
        }
    }
}

// Full segment reduction for block `blk` of a vector of length n.  Thread 0
// returns the block partials in `out`; op.apply runs exactly once per element.
template <typename V, int NACC, class Op, class Sync = CtaSync>
__device__ __forceinline__ void block_reduce(PlanPtrs plans, int64_t n, int64_t block_size, int64_t blk, const Op& op,
                                             V* nodes, V (&out)[NACC], Sync sync = Sync()) {
    const int64_t base = blk * block_size;
    const bool full = base + block_size <= n;
    const char* plan = full ? plans.full : plans.tail;
    V v0[NACC];
    if (threadIdx.x == 0) {
        typename Op::Item it = op.load(base);
        op.apply(base, it, v0);
    }
    block_pass<V, NACC>(plan, base + 1, op, nodes, sync);
    if (threadIdx.x == 0) {
        const PlanHeader* h = plan_hdr(plan);
#pragma unroll
        for (int a = 0; a < NACC; ++a)
            out[a] = (h->L > 0) ? VT<V>::add(v0[a], nodes[h->root * NACC + a]) : v0[a];
    }
    sync();  // nodes may be reused by the caller's next pass
}

// Arrival counter over `total` arrivals (one per block): true in every
// participating thread of the CTA making the last arrival.  Thread 0 must
// have written this block's partials before the call.
template <class Sync = CtaSync>
__device__ __forceinline__ bool arrive_last(unsigned int* counter, unsigned int total, unsigned int* flag_smem,
                                            Sync sync = Sync()) {
    __threadfence();
    sync();
    if (threadIdx.x == 0) {
        unsigned int prev = atomicAdd(counter, 1u);
        *flag_smem = (prev == total - 1) ? 1u : 0u;
    }
    sync();
    const bool last = *flag_smem != 0;
    if (last) __threadfence();
    return last;
}

// Left fold of nacc interleaved partial streams (partials[b*nacc + a]),
// vecops.py:159-161: total = p[0]; total = total + p[b] for b = 1..nb-1.
// Componentwise Python adds are independent chains, so each real component
// of each accumulator folds on its own warp.  `scratch` holds at least
// chunk*nacc values; `res_smem` >= 16 doubles.  Result valid in thread 0.
template <typename V, class Sync = CtaSync>
__device__ void ordered_fold(const V* partials, int nacc, int64_t nb, V* scratch, int64_t chunk, V* result,
                             double* res_smem, Sync sync = Sync()) {
    constexpr int NC = sizeof(V) / sizeof(double);
    const int nthr = sync.nthreads();
    const int nchains = nacc * NC;
    const int warp = threadIdx.x >> 5;
    const bool chain = (threadIdx.x & 31) == 0 && warp < nchains;
    const int a = warp / NC, comp = warp % NC;
    double tot = 0.0;
    const double* sd = reinterpret_cast<const double*>(scratch);
    for (int64_t c0 = 0; c0 < nb; c0 += chunk) {
        const int64_t cn = (nb - c0 < chunk) ? nb - c0 : chunk;
        const int64_t nv = cn * nacc;
        if ((int)threadIdx.x < nthr)
            for (int64_t i = threadIdx.x; i < nv; i += nthr) scratch[i] = __ldcg(partials + c0 * nacc + i);
        sync();
        if (chain) {
            int64_t b = 0;
            if (c0 == 0) {
                tot = sd[(0 * nacc + a) * NC + comp];
                b = 1;
            }
#pragma unroll 16
            for (; b < cn; ++b) tot = __dadd_rn(tot, sd[(b * nacc + a) * NC + comp]);
        }
        sync();
    }
    if (chain) res_smem[warp] = tot;
    sync();
    if (threadIdx.x == 0) {
        double* r = reinterpret_cast<double*>(result);
        for (int c = 0; c < nchains; ++c) r[c] = res_smem[c];
    }
    sync();
}

}  // namespace zk
