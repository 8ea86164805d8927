// zk_spmv.cuh -- SELL-32 complex128 SpMV row engine (device side).
//
// Layout (built once per matrix by zk_csr_create, zk_spmv.cu):
//   rows are cut into 32-row slices; slice s stores its rows column-major,
//   element k of slice-row r at aa[slice_off[s] + 32*k + r] (double2) and
//   ja[...] (int32), padded to the slice's longest row.  A warp owns a slice
//   and a thread owns a row, so every aa/ja load instruction of the warp is
//   one contiguous 512 B / 128 B transaction, and for stencil matrices the
//   x gathers of a warp (x[j_r + k] over 32 consecutive rows) are contiguous
//   too.  Rows longer than 65 entries ("long rows", absent from stencil and
//   FE matrices) are kept in a side CSR and summed by one thread with the
//   full pairwise recursion.
//
// Arithmetic (sparse.py:217-232 + numpy): the product of
// entry k is F1(aa_k, x[ja_k]) -- or F1(x[ja_k], aa_k) once numpy's
// temporary elision kicks in (nnz*16 >= 256 KiB) -- and a row with L
// entries sums as v0 + PW(v1..v_{L-1}); for L-1 <= 64 that is one pairwise
// leaf: four lane accumulators over full groups of four, (l0+l1)+(l2+l3),
// then the leftovers in order.  One thread evaluates exactly that sequence
// in registers, so results do not depend on the launch geometry (rows are
// independent: test_sparse.py:157-165).
#pragma once
#include "zk_common.cuh"

namespace zk {

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
    bool swap;  // numpy elided the gathered temporary: prod = F1(x[ja], aa)
    bool fma;
};

__device__ __forceinline__ double2 sell_prod(const SellView& A, const double2* __restrict__ x, int64_t idx) {
    double2 a = __ldg(A.aa + idx);
    int j = __ldg(A.ja + idx);
    double2 xv = __ldg(x + j);
    return A.swap ? f1(xv, a, A.fma) : f1(a, xv, A.fma);
}

// Row sum for a short row whose element k sits at base + 32*k.
__device__ __forceinline__ double2 sell_row(const SellView& A, const double2* __restrict__ x, int64_t base, int len) {
    if (len == 0) return make_double2(0.0, 0.0);
    double2 v0 = sell_prod(A, x, base);
    const int L = len - 1;
    if (L == 0) return v0;
    double2 s;
    if (L < 4) {
        s = make_double2(-0.0, -0.0);
        for (int k = 1; k <= L; ++k) s = cadd(s, sell_prod(A, x, base + 32 * (int64_t)k));
    } else {
        double2 r0 = sell_prod(A, x, base + 32);
        double2 r1 = sell_prod(A, x, base + 64);
        double2 r2 = sell_prod(A, x, base + 96);
        double2 r3 = sell_prod(A, x, base + 128);
        const int G = L >> 2;
        for (int g = 1; g < G; ++g) {
            const int64_t idx = base + 32 * (int64_t)(1 + 4 * g);
            double2 p0 = sell_prod(A, x, idx);
            double2 p1 = sell_prod(A, x, idx + 32);
            double2 p2 = sell_prod(A, x, idx + 64);
            double2 p3 = sell_prod(A, x, idx + 96);
            r0 = cadd(r0, p0);
            r1 = cadd(r1, p1);
            r2 = cadd(r2, p2);
            r3 = cadd(r3, p3);
        }
        s = cadd(cadd(r0, r1), cadd(r2, r3));
        for (int k = 1 + 4 * G; k <= L; ++k) s = cadd(s, sell_prod(A, x, base + 32 * (int64_t)k));
    }
    return cadd(v0, s);
}

__device__ __forceinline__ double2 long_prod(const SellView& A, const double2* __restrict__ x, int64_t idx) {
    double2 a = A.long_aa[idx];
    double2 xv = __ldg(x + A.long_ja[idx]);
    return A.swap ? f1(xv, a, A.fma) : f1(a, xv, A.fma);
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

// All rows of 4096-row block `blk`; epi(row, value) is called once per row
// by the thread that computed it.  No barrier inside.
template <class Epi>
__device__ __forceinline__ void spmv_block(const SellView& A, const double2* __restrict__ x, int64_t blk, Epi& epi) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int64_t s_lo = blk * (kBlock / kSlice);
    int64_t s_hi = s_lo + kBlock / kSlice;
    if (s_hi > A.nslices) s_hi = A.nslices;
    for (int64_t s = s_lo + warp; s < s_hi; s += nwarps) {
        const int64_t row = s * kSlice + lane;
        const int len = A.rowlen[row];
        if (row < A.n_rows && len != 255) {
            double2 v = sell_row(A, x, A.slice_off[s] + lane, len);
            epi(row, v);
        }
    }
    if (A.long_blk_ptr) {
        const int lb = A.long_blk_ptr[blk], le = A.long_blk_ptr[blk + 1];
        for (int li = lb + (int)threadIdx.x; li < le; li += blockDim.x) epi((int64_t)A.long_row[li], long_row_sum(A, x, li));
    }
}

}  // namespace zk
