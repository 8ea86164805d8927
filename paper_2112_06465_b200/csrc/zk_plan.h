// zk_plan.h -- numpy pairwise-summation plans.
//
// A reduceat segment of a reduction block is v[0] + PW(v[1:L+1]) (numpy
// reduceat copies the first element, then adds the pairwise sum of the rest;
// vecops.py:156-162, sparse.py:231).  PW recursively halves the range until a
// leaf holds <= 64 complex (CDOUBLE_pairwise_sum) or <= 128 real
// (DOUBLE_pairwise_sum) elements; a leaf is summed by 4 (complex) or 8 (real)
// interleaved lane accumulators, combined as (l0+l1)+(l2+l3) (resp. the
// 8-lane tree), then the leftover elements sequentially.  Ranges shorter
// than the lane count are summed sequentially from -0.0.
//
// A Plan flattens that recursion for one segment length L so a CTA can run
// it in parallel: every (leaf, lane) pair becomes one thread work item, and
// the internal nodes are grouped into rounds whose operands are all ready.
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace zk {

enum PlanKind : int32_t { kComplex = 0, kReal = 1 };

struct PlanHeader {
    int32_t L;          // segment length (block length - 1)
    int32_t kind;       // kComplex / kReal
    int32_t lanes;      // 4 or 8
    int32_t seq;        // 1: L < lanes -> one sequential leaf summed from -0.0
    int32_t nleaves;
    int32_t nnodes;     // leaves + internal nodes
    int32_t root;       // node index of the root (valid when L > 0)
    int32_t nrounds;
    int32_t round_off[40];  // ops of round r: [round_off[r], round_off[r+1])
    int32_t leaves_off;     // int2 (start, len) array, byte offset from header
    int32_t ops_off;        // int4 (dst, a, b, 0) array, byte offset from header
    int32_t nops;
    // Stage table (int4 {b_lo, b_hi, l_lo, l_hi} at stages_off): the segment
    // cut into subtrees of the pairwise recursion with at most 32 (leaf,
    // lane) items each -- 8 complex / 4 real leaves, <= 512 elements --
    // stage s holding block elements [b_lo, b_hi) (stage 0 also element 0,
    // the reduceat head) and leaves [l_lo, l_hi).  The TMA-fed level-1
    // engine (zk_l1pipe.cuh) streams a block stage by stage.
    // [0]: stages of <= kStageItems items; [1]: <= kStageItems / 2 (finer
    // stages for ops that stage many vectors: more ring slots in flight)
    int32_t nstages[2];
    int32_t stages_off[2];
    // leaf_upto[j]: number of leaves whose elements all lie in rows [0, 32*j)
    // of the 4096-row block (element e of the segment is block row 1+e); lets
    // the SpMV kernels reduce leaves as soon as the rows under them are done.
    int16_t leaf_upto[130];
};

constexpr int kStageItems = 32;     // (leaf, lane) items per stage: one warp
constexpr int kStageMaxElems = 520; // >= 1 + 8 * 64 (complex) and 1 + 4 * 128 (real)
constexpr int kStageMaxElemsFine = 264;  // >= 1 + 4 * 64 and 1 + 2 * 128

// Builds the plan for segment length L into `out` (host memory); returns the
// number of bytes used.  `out` may be null to query the size.
size_t build_plan(int32_t L, int32_t kind, void* out);

}  // namespace zk
