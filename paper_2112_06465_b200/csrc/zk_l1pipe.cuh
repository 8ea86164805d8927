// zk_l1pipe.cuh -- TMA-fed level-1 block reductions (sm_100a).
//
// The reductions of vecops.zdot / znorm2 (vecops.py:156-200) and the fused
// elementwise+reduction phases of the solvers are HBM streams whose result
// must be summed in numpy's pairwise order.  A thread-per-(leaf, lane)
// kernel that loads its own operands keeps only what fits in its registers
// in flight and stalls at every block boundary (warps active ~20%, 0.59-0.72
// of HBM, profiles/r01_ncu_summary.txt).  This engine decouples the bytes in
// flight from the summation order:
//
//   * a persistent CTA per SM streams its 4096-element blocks STAGE by
//     STAGE: a stage is a subtree of numpy's pairwise recursion with at most
//     32 (leaf, lane) items (the plan's stage table, zk_plan.cpp), <= 512
//     elements of each input vector;
//   * the producer warp's lanes own the ring slots and move every input
//     vector's stage range into shared memory with 1-D TMA bulk copies
//     (cp.async.bulk, L2 evict-first): up to ~200 KB in flight per SM
//     without a register;
//   * consumer warps take whole stages: lane = (leaf, lane accumulator q),
//     reading its elements leaf_start + q + LANES*g from shared memory in
//     numpy's order, applying the op's fused elementwise update (outputs go
//     straight to HBM) and accumulating the term; lane tree and leftovers by
//     shuffles; leaf sums into a double-buffered node array;
//   * a tree warp combines the block's leaves in the plan's round order as
//     soon as its last stage is consumed (while the consumers stream the next
//     block), adds the reduceat head v[0] and publishes the block partial --
//     into a streaming-fold slot (1 GPU) or into the partials array
//     (row-sharded solve: folded across ranks later);
//   * CTA 0's fold warp folds the slots in block order WHILE the pass runs
//     (stream_fold, zk_blockred.cuh: the serial add chain overlaps the
//     stream) and hands the totals to Fin::finish.
//
// The arithmetic is the plan's -- identical to leaf_phase/warp_tree -- so
// results are bitwise those of the reference, whatever the launch geometry.
#pragma once
#include "zk_blockred.cuh"

namespace zk {

constexpr int kL1Consumers = 10;
constexpr int kL1Threads = 32 * (kL1Consumers + 3);  // producer + consumers + tree warp + fold warp
constexpr int kL1StaticSmem = 2 * 32 * kPollPer * 8;  // stream_fold's staging (static shared memory)
constexpr int kL1MaxIn = 6;
constexpr int kL1Nodes = 136;  // >= plan nodes of a 4096 block (<= 129)

// Launch description of one engine pass.
struct L1View {
    int64_t n, nblocks;
    PlanPtrs plans;               // 4096-element blocks: full / tail plans (kind matches the op's V)
    const double2* in[kL1MaxIn];  // staged input vectors (nullptr: not staged, reads input alias[v])
    int8_t alias[kL1MaxIn];       // for a null in[v]: the input whose staged copy it reads (same vector)
    int32_t nin;                  // staged (non-null) inputs
    int32_t ns;                   // ring slots
    int32_t slot_bytes;           // nin * smax * 16
    int32_t fine;                 // stage table: 0 (<= 32 items) or 1 (<= 16 items, half-size slots)
    int32_t smax;                 // elements per staged vector in a slot (kStageMaxElems[Fine])
    double* slots;                // streaming fold slots (nblocks * NP), or nullptr
    double* partials;             // stored partials (nblocks * NP) when slots == nullptr
};

// Engine geometry for a DEFAULT_PLAN pass over n elements (zk_blas1.cu):
// staged inputs in[0..nin_op) (null = alias), fold slots or stored partials,
// reduction terms of vbytes (0: 16 complex / 8 real).  False when it does
// not fit the engine.
bool l1_view(zk_context* c, int64_t n, int32_t kind, const double2* const* in, const int8_t* alias, int nin_op,
             double* slots, double* partials, L1View& P, size_t& smem, unsigned& grid, int vbytes = 0,
             int fine = -1);

template <typename V>
struct L1Smem {
    // [full mbarriers ns][empty mbarriers ns][blkdone 2][nodefree 2][tags ns]
    // [nodes 2 x kL1Nodes V][v0 2 V][plans: full, tail][ring]
    static constexpr int kMaxSlots = 32;
    static constexpr int kPlanBytes = 4096;
    static constexpr size_t kBars = (2 * kMaxSlots + 4) * 8;
    static constexpr size_t kTags = kMaxSlots * 4;
    static constexpr size_t kNodes = 2 * kL1Nodes * sizeof(V);
    static constexpr size_t kV0 = 2 * sizeof(V) > 16 ? 2 * sizeof(V) : 16;
    static constexpr size_t kHead = (kBars + kTags + kNodes + kV0 + 2 * kPlanBytes + 127) / 128 * 128;
};

// Shared-memory head (everything but the ring) for reduction terms of vbytes.
inline size_t l1_head_bytes(int vbytes) {
    using S = L1Smem<double>;
    const size_t v0 = 2 * (size_t)vbytes > 16 ? 2 * (size_t)vbytes : 16;
    return (S::kBars + S::kTags + 2 * (size_t)kL1Nodes * vbytes + v0 + 2 * S::kPlanBytes + 127) / 128 * 128;
}

// Copies a plan blob (header..stage table) into shared memory; whole warp.
__device__ __forceinline__ const char* l1_cache_plan(const char* g, char* s) {
    const PlanHeader* h = reinterpret_cast<const PlanHeader*>(g);
    const int bytes = h->stages_off[1] + 16 * h->nstages[1];
    if (bytes > L1Smem<double>::kPlanBytes) return g;
    const int4* src = reinterpret_cast<const int4*>(g);
    int4* dst = reinterpret_cast<int4*>(s);
    for (int i = threadIdx.x & 31; i < (bytes + 15) / 16; i += 32) dst[i] = src[i];
    return s;
}

// Internal nodes in the plan's round order by one warp (the plan may live in
// shared memory: generic loads, not __ldg as warp_tree uses).
template <typename V>
__device__ __forceinline__ V l1_tree(const char* plan, V* nodes) {
    const PlanHeader* h = plan_hdr(plan);
    const int lane = threadIdx.x & 31;
    if (!h->seq) {
        const int4* ops = reinterpret_cast<const int4*>(plan + h->ops_off);
        for (int r = 0; r < h->nrounds; ++r) {
            const int lo = h->round_off[r], hi = h->round_off[r + 1];
            for (int o = lo + lane; o < hi; o += 32) {
                const int4 opn = ops[o];
                nodes[opn.x] = VT<V>::add(nodes[opn.y], nodes[opn.z]);
            }
            __syncwarp();
        }
    }
    return nodes[h->root];
}

// Op interface:  V (double2 complex / double real term), NIN (staged inputs),
//   __device__ V apply(int64_t e, const double2 (&v)[NIN]) const
// -- the fused elementwise update of global element e (writes its outputs)
// returning its reduction term.  Fin: static kNP; __device__ finish(const double*).
template <class Op, class Fin>
__device__ __forceinline__ void l1_pipeline(const L1View& P, const Op& op, Fin& fin, unsigned char* smem) {
    using V = typename Op::V;
    constexpr int NIN = Op::NIN;
    constexpr int LANES = VT<V>::lanes;
    constexpr int NP = (int)(sizeof(V) / sizeof(double));
    using SM = L1Smem<V>;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + SM::kMaxSlots;
    uint64_t* blkdone = empty + SM::kMaxSlots;
    uint64_t* nodefree = blkdone + 2;
    volatile uint32_t* tag = reinterpret_cast<volatile uint32_t*>(smem + SM::kBars);
    V* nodes = reinterpret_cast<V*>(smem + SM::kBars + SM::kTags);
    V* v0s = reinterpret_cast<V*>(smem + SM::kBars + SM::kTags + SM::kNodes);
    char* pl_full = reinterpret_cast<char*>(smem + SM::kBars + SM::kTags + SM::kNodes + SM::kV0);
    char* pl_tail = pl_full + SM::kPlanBytes;
    unsigned char* ring = smem + SM::kHead;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ns = P.ns;

    const PlanHeader* hf = plan_hdr(P.plans.full);
    const int fine = P.fine;
    const int nst_full = hf->nstages[fine];
    const int64_t tail_blk = P.nblocks - 1;
    const bool has_tail = P.plans.tail != P.plans.full;
    // CTA-local block k -> global block blockIdx.x + k * gridDim.x
    const int64_t nblk_cta = (P.nblocks - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const bool own_tail = has_tail && ((tail_blk - blockIdx.x) % gridDim.x == 0);
    const int64_t total_stages =
        own_tail ? (nblk_cta - 1) * nst_full + plan_hdr(P.plans.tail)->nstages[fine] : nblk_cta * nst_full;
    const int nst_tail_blk = own_tail ? plan_hdr(P.plans.tail)->nstages[fine] : nst_full;

    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            tag[i] = 0xffffffffu;
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&blkdone[b], (uint32_t)nst_full);
            mbar_init(&nodefree[b], 1);
        }
        mbar_fence_init();
    }
    if (warp == kL1Consumers + 1) {  // tree warp caches the plans
        l1_cache_plan(P.plans.full, pl_full);
        if (has_tail) l1_cache_plan(P.plans.tail, pl_tail);
    }
    __syncthreads();
    const char* cfull = (hf->stages_off[1] + 16 * hf->nstages[1] <= SM::kPlanBytes) ? pl_full : P.plans.full;
    const char* ctail = P.plans.full;
    if (has_tail) {
        const PlanHeader* ht = plan_hdr(P.plans.tail);
        ctail = (ht->stages_off[1] + 16 * ht->nstages[1] <= SM::kPlanBytes) ? pl_tail : P.plans.tail;
    } else {
        ctail = cfull;
    }

    // stage q of this CTA -> (CTA block k, global block, plan, stage index)
    auto locate = [&](int64_t q, int64_t& k, int64_t& blk, const char*& plan, int& s) {
        k = q / nst_full;
        s = (int)(q - k * nst_full);
        blk = blockIdx.x + k * gridDim.x;
        plan = (has_tail && blk == tail_blk) ? ctail : cfull;
    };

    if (warp == 0) {  // ---- producer: lane l owns ring slot l ----
        const uint64_t pol = l2_evict_first_policy();
        const bool owner = lane < ns;
        int64_t q = lane;
        uint32_t u = 0;
        while (__any_sync(0xffffffffu, owner && q < total_stages)) {
            if (owner && q < total_stages && (u == 0 || mbar_test(&empty[lane], (u - 1) & 1))) {
                int64_t k, blk;
                const char* plan;
                int s;
                locate(q, k, blk, plan, s);
                const int4 st = reinterpret_cast<const int4*>(plan + plan_hdr(plan)->stages_off[fine])[s];
                const int64_t e0 = blk * kBlock + st.x;
                const uint32_t bytes = (uint32_t)(st.y - st.x) * 16u;
                tag[lane] = (uint32_t)q;
                mbar_arrive_expect_tx(&full[lane], bytes * (uint32_t)P.nin);
                unsigned char* dst = ring + (size_t)lane * P.slot_bytes;
                int slot_in = 0;
#pragma unroll
                for (int v = 0; v < NIN; ++v) {
                    if (P.in[v]) {
                        bulk_g2s(dst + (size_t)slot_in * P.smax * 16, P.in[v] + e0, bytes, &full[lane], pol);
                        ++slot_in;
                    }
                }
                q += ns;
                ++u;
            }
        }
        return;
    }

    if (warp <= kL1Consumers) {  // ---- consumers: warp w takes stages w-1, w-1+CW, ... ----
        // staged position of each op input (inputs not staged alias another)
        int pos[NIN];
        {
            int c = 0;
#pragma unroll
            for (int v = 0; v < NIN; ++v) pos[v] = P.in[v] ? c++ : -1;
#pragma unroll
            for (int v = 0; v < NIN; ++v)
                if (pos[v] < 0) pos[v] = pos[P.alias[v]] >= 0 ? pos[P.alias[v]] : 0;
        }
        for (int64_t q = warp - 1; q < total_stages; q += kL1Consumers) {
            int64_t k, blk;
            const char* plan;
            int s;
            locate(q, k, blk, plan, s);
            const PlanHeader* h = plan_hdr(plan);
            const int4 st = reinterpret_cast<const int4*>(plan + h->stages_off[fine])[s];
            const int slot = (int)(q % ns);
            while (tag[slot] != (uint32_t)q) {
            }
            mbar_wait(&full[slot], (uint32_t)((q / ns) & 1));
            const double2* sbase = reinterpret_cast<const double2*>(ring + (size_t)slot * P.slot_bytes);
            const int64_t base = blk * kBlock;
            const int buf = (int)(k & 1);
            if (k >= 2) mbar_wait(&nodefree[buf], (uint32_t)(((k >> 1) - 1) & 1));
            V* nd = nodes + buf * kL1Nodes;
            auto elem = [&](int be, double2 (&vals)[NIN]) {  // block element be (staged)
                const int li = be - st.x;
#pragma unroll
                for (int v = 0; v < NIN; ++v) vals[v] = sbase[pos[v] * P.smax + li];
            };
            if (s == 0 && lane == 0) {  // reduceat head v[0]
                double2 vals[NIN];
                elem(0, vals);
                v0s[buf] = op.apply(base, vals);
            }
            if (h->seq) {  // L < LANES: one sequential leaf from -0.0
                if (lane == 0 && h->L > 0) {
                    V acc = VT<V>::negzero();
                    for (int e = 1; e <= h->L; ++e) {
                        double2 vals[NIN];
                        elem(e, vals);
                        acc = VT<V>::add(acc, op.apply(base + e, vals));
                    }
                    nd[0] = acc;
                }
            } else {
                const int2* leaves = reinterpret_cast<const int2*>(plan + h->leaves_off);
                const int leaf = st.z + lane / LANES;
                const int qq = lane & (LANES - 1);
                const bool valid = leaf < st.w;
                const int2 lf = valid ? leaves[leaf] : make_int2(0, 0);
                const int G = lf.y / LANES;
                const int rem = lf.y - G * LANES;
                const int be0 = 1 + lf.x + qq;  // block element of group 0
                V acc = VT<V>::zero();
                if (valid) {
                    // U groups' operands read from shared memory ahead of their
                    // in-order accumulation (the add chain stays the plan's)
                    constexpr int U = NIN <= 2 ? 4 : 2;
                    int g = 0;
                    for (; g + U <= G; g += U) {
                        double2 vals[U][NIN];
#pragma unroll
                        for (int u = 0; u < U; ++u) elem(be0 + LANES * (g + u), vals[u]);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const V t = op.apply(base + be0 + LANES * (g + u), vals[u]);
                            acc = (g + u == 0) ? t : VT<V>::add(acc, t);
                        }
                    }
                    for (; g < G; ++g) {
                        double2 vals[NIN];
                        elem(be0 + LANES * g, vals);
                        const V t = op.apply(base + be0 + LANES * g, vals);
                        acc = (g == 0) ? t : VT<V>::add(acc, t);
                    }
                }
#pragma unroll
                for (int d = 1; d < LANES; d <<= 1) {
                    const V o = VT<V>::shfl_down(acc, d);
                    if ((qq & (2 * d - 1)) == 0) acc = VT<V>::add(acc, o);
                }
                V left = VT<V>::zero();
                if (valid && qq < rem) {
                    double2 vals[NIN];
                    elem(be0 + LANES * G, vals);
                    left = op.apply(base + be0 + LANES * G, vals);
                }
                const int grp = lane & ~(LANES - 1);
#pragma unroll
                for (int j = 0; j < LANES - 1; ++j) {
                    const V o = VT<V>::shfl(left, grp + j);
                    if (j < rem) acc = VT<V>::add(acc, o);
                }
                if (valid && qq == 0) nd[leaf] = acc;
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[slot]);
                // the tail block may have fewer stages than the barrier's count
                const int nst_blk = (has_tail && blk == tail_blk) ? nst_tail_blk : nst_full;
                if (s == nst_blk - 1 && nst_blk < nst_full) {
                    for (int r = 0; r < nst_full - nst_blk; ++r) mbar_arrive(&blkdone[buf]);
                }
                mbar_arrive(&blkdone[buf]);
            }
        }
        return;
    }

    if (warp == kL1Consumers + 2) {  // ---- fold warp (CTA 0): the ordered left fold, as partials land ----
        if (P.slots != nullptr && blockIdx.x == 0) {
            double t[NP];
            stream_fold<NP>(P.slots, P.nblocks, t);
            if (lane == 0) fin.finish(t);
        }
        return;
    }

    // ---- tree warp: combine each block, publish its partial ----
    for (int64_t k = 0; k < nblk_cta; ++k) {
        const int buf = (int)(k & 1);
        mbar_wait(&blkdone[buf], (uint32_t)((k >> 1) & 1));
        const int64_t blk = blockIdx.x + k * gridDim.x;
        const char* plan = (has_tail && blk == tail_blk) ? ctail : cfull;
        V* nd = nodes + buf * kL1Nodes;
        const bool has = plan_hdr(plan)->L > 0;
        const V pw = has ? l1_tree<V>(plan, nd) : VT<V>::zero();
        if (lane == 0) {
            const V p = has ? VT<V>::add(v0s[buf], pw) : v0s[buf];
            const double* pd = reinterpret_cast<const double*>(&p);
#pragma unroll
            for (int c = 0; c < NP; ++c) {
                if (P.slots) slot_store(P.slots + blk * NP + c, pd[c]);
                else P.partials[blk * NP + c] = pd[c];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&nodefree[buf]);
    }
}

}  // namespace zk
