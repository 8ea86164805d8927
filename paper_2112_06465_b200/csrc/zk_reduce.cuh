// zk_reduce.cuh -- shared types of the numpy-order block reductions.
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
// Block partials are folded left to right (vecops.py:159-161) by one warp,
// staged through shared memory so the serial chain runs at DADD latency
// (zk_blockred.cuh: leaf_phase, warp_tree, warp_finish, warp_fold).
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

// Two complex reductions summed side by side in the same (complex) order,
// e.g. <t, t> and <t, s> of BiCGStab's omega (krylov.py:282-286).
struct cplx2 {
    double2 a, b;
};
template <> struct VT<cplx2> {
    static constexpr int lanes = 4;
    static __device__ __forceinline__ cplx2 add(cplx2 x, cplx2 y) { return {cadd(x.a, y.a), cadd(x.b, y.b)}; }
    static __device__ __forceinline__ cplx2 negzero() {
        return {make_double2(-0.0, -0.0), make_double2(-0.0, -0.0)};
    }
    static __device__ __forceinline__ cplx2 zero() { return {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}; }
    static __device__ __forceinline__ cplx2 shfl(cplx2 v, int src) {
        return {VT<double2>::shfl(v.a, src), VT<double2>::shfl(v.b, src)};
    }
    static __device__ __forceinline__ cplx2 shfl_down(cplx2 v, int d) {
        return {VT<double2>::shfl_down(v.a, d), VT<double2>::shfl_down(v.b, d)};
    }
};

struct PlanPtrs {
    const char* full;  // plan for full blocks (L = block_size - 1)
    const char* tail;  // plan for the last, partial block (may equal full)
};

__device__ __forceinline__ const PlanHeader* plan_hdr(const char* p) { return reinterpret_cast<const PlanHeader*>(p); }

}  // namespace zk
