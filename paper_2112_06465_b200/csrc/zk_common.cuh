// zk_common.cuh -- shared device arithmetic for libzk (sm_100a).
//
// Every floating-point operation on the result path is spelled with an _rn
// intrinsic so the compiler cannot contract or reorder it (the library is
// also built with -fmad=false as a second guard).  The formulas are the
// reference's, not approximations of them:
//
//   f1()        numpy complex multiply (SURVEY Appendix A "F1"):
//               re = fma(a.re, b.re, -(a.im*b.im)), im = fma(a.re, b.im, a.im*b.re)
//               or, with the plain fingerprint, every product rounded.
//   cmul_py()   CPython / Cplx multiply (cnum.py:113-115): plain, no FMA.
//   cdiv_py()   Cplx Smith division with true divisions (cnum.py:118-134).
//   small_py()  krylov.py:209-210  abs(value) < 1e-300.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace zk {

constexpr int kBlock = 4096;       // DEFAULT_PLAN block size (vecops.py:98)
constexpr int kThreads = 256;      // CTA size of the block-pass kernels
constexpr int kSlice = 32;         // SELL slice height (rows per warp)
constexpr int kShortMax = 65;      // rows up to 1 + 64 nnz fit one pairwise leaf
constexpr double kBreakdownEps = 1e-300;

__device__ __forceinline__ double2 cz(double re, double im) { return make_double2(re, im); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// numpy complex multiply a*b.
__device__ __forceinline__ double2 f1(double2 a, double2 b, bool fma) {
    if (fma) {
        return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                            __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
    }
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double2 conjz(double2 a) { return make_double2(a.x, -a.y); }

// |z|^2 as znorm2 forms it: (re*re) + (im*im), two separately rounded products.
__device__ __forceinline__ double abs2_np(double2 a) {
    return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

__device__ __forceinline__ double2 cmul_py(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double2 cdiv_py(double2 a, double2 b) {
    double c = b.x, d = b.y;
    if (fabs(c) >= fabs(d)) {
        double r = __ddiv_rn(d, c);
        double den = __dadd_rn(c, __dmul_rn(d, r));
        return make_double2(__ddiv_rn(__dadd_rn(a.x, __dmul_rn(a.y, r)), den),
                            __ddiv_rn(__dsub_rn(a.y, __dmul_rn(a.x, r)), den));
    }
    double r = __ddiv_rn(c, d);
    double den = __dadd_rn(__dmul_rn(c, r), d);
    return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(a.x, r), a.y), den),
                        __ddiv_rn(__dsub_rn(__dmul_rn(a.y, r), a.x), den));
}

// abs(Cplx) is math.hypot; only its comparison with 1e-300 matters.  When
// max(|re|,|im|) >= 1e-300 the modulus is >= 1e-300 exactly; below that the
// scaled hypot decides (its <=1ulp error can only matter within one ulp of
// the threshold).
__device__ __forceinline__ bool small_py(double2 v) {
    double a = fabs(v.x), b = fabs(v.y);
    double m = fmax(a, b);
    if (!(m < kBreakdownEps)) return false;  // also false for NaN (hypot(nan) < eps is False)
    return hypot(a, b) < kBreakdownEps;
}

__device__ __forceinline__ bool small_py(double v) { return !(fabs(v) >= kBreakdownEps) && fabs(v) < kBreakdownEps; }

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

// Device-side predication of a graph-captured kernel: the solver drivers
// capture a whole loop body once, and each kernel decides from the solver's
// state words whether it runs (p[0] = done, p[1] = the solver's flag).
//   kAlways: always;  kLive: unless done;  kLiveNoFlag: unless done or flag;
//   kLiveFlag: only when not done and flag is set.
struct Gate {
    const int32_t* p;
    int32_t mode;
    enum : int32_t { kAlways = 0, kLive = 1, kLiveNoFlag = 2, kLiveFlag = 3 };
    __device__ __forceinline__ bool skip() const {
        if (p == nullptr || mode == kAlways) return false;
        const int32_t done = p[0], flag = p[1];
        if (done) return true;
        if (mode == kLiveNoFlag) return flag != 0;
        if (mode == kLiveFlag) return flag == 0;
        return false;
    }
};

}  // namespace zk
