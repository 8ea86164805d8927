// zk_spmv.cu -- CSR -> SELL-32 conversion and the plain SpMV kernel.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "zk_internal.h"
#include "zk_spmv.cuh"

namespace zk {

// Ring geometry for a launch that also needs `extra` bytes of dynamic
// shared memory after the ring (epilogue stash, reduction nodes).
SellView sell_view(const zk_csr* A, const zk_context* c, size_t extra, int nsv) {
    SellView v;
    v.narrow_w = 0;
    v.sv[0] = v.sv[1] = nullptr;
    v.n_rows = A->n_rows;
    v.n_cols = A->n_cols;
    v.nslices = A->nslices;
    v.nblocks = A->nblocks;
    v.aa = A->aa;
    v.ja = A->ja;
    v.slice_off = A->slice_off;
    v.slice_cmax = A->slice_cmax;
    v.rowlen = A->rowlen;
    v.long_row = A->long_row;
    v.long_blk_ptr = A->n_long ? A->long_blk_ptr : nullptr;
    v.long_ia = A->long_ia;
    v.long_ja = A->long_ja;
    v.long_aa = A->long_aa;
    // Ring chunk = (1 + 4 cm) columns of a slice (two pairwise groups, or one
    // when shared memory is tight), independent of the row width.
    const int w = A->wmax > 0 ? A->wmax : 1;
    // Stay within the 196 KB shared-memory carve-out so that L1 keeps >= 60 KB
    // for the x gathers (a 228 KB carve-out leaves 28 KB and the gathers'
    // L1 hit rate collapses); ZK_SMEM_KB overrides (experiments only).
    const char* env_kb = std::getenv("ZK_SMEM_KB");
    const long limit = env_kb ? std::atol(env_kb) * 1024 : 196 * 1024;
    const long avail = std::min<long>(limit, kSmemLimit) - 1024 - kBarBytes - (long)extra;
    const char* env_cm = std::getenv("ZK_CM");      // tuning overrides (experiments only)
    const char* env_ns = std::getenv("ZK_NS");
    const int cm_hi = env_cm ? std::atoi(env_cm) : 2;
    const int cm_lo = env_cm ? cm_hi : 1;
    if ((!env_cm || cm_hi == 0) && w <= kFullCols) {  // whole slice per stage, whole-row prefetch
        // stage = [aa: wpad x 32 double2][ja: wpad x 32 int32][32 row lengths],
        // wpad = w rounded up to 4 (the fast row path reads whole groups)
        const int wpad = (w + 3) & ~3;
        v.cm = 0;
        v.nch = 1;
        v.ja_off = wpad * kSlice * 16;
        v.rl_off = v.ja_off + wpad * kSlice * 4;
        v.sv_off = v.rl_off + kSlice;
        v.nsv = nsv;
        v.stage_bytes = (v.sv_off + nsv * kSlice * 16 + 127) / 128 * 128;
        // as many stages as the carve-out holds: C4 SpMV 724 us at 10 stages, 713 at 11
        // (with the x prefetch on; a cap of 10 measured better before it)
        const long ns = avail / v.stage_bytes;
        v.ns = (int)(ns > kMaxStages ? kMaxStages : (ns < 1 ? 1 : ns));
        if (env_ns && std::atoi(env_ns) > 0) {  // experiments: any depth the shared memory holds
            const long want = std::atoi(env_ns);
            v.ns = (int)std::min<long>(std::min<long>(want, kMaxStages), ns < 1 ? 1 : ns);
        }
        v.swap = (A->nnz_elide * 16 >= c->elide_bytes);
        v.fma = c->fma != 0;
        v.ns_magic = (uint32_t)((1ull << 32) / (uint64_t)v.ns + 1);
        v.spb = kBlock / kSlice;
        v.nvb = A->nblocks;
        {
            // the x L2 bulk prefetch (one more TMA op per slice): C4 SpMV 731 -> 724 us
            // (three A/B pairs, +0.7% solves/s); it cost C5 1.7% when C5's 7-wide rows
            // still ran on the ring (they take the narrow kernels now).  ZK_PREFETCH=0: off
            const char* e = std::getenv("ZK_PREFETCH");
            v.prefetch = !(e && e[0] == '0');
        }
        return v;
    }
    for (int cm = cm_hi; cm >= cm_lo; --cm) {
        const int cols = 1 + 4 * cm;
        v.cm = cm;
        v.nch = w <= cols ? 1 : 1 + (w - cols + 4 * cm - 1) / (4 * cm);
        v.ja_off = cols * kSlice * 16;
        v.rl_off = 0;
        v.sv_off = 0;
        v.nsv = nsv;
        v.stage_bytes = (cols * kSlice * 20 + 127) / 128 * 128;
        const long ns = avail / v.stage_bytes;
        v.ns = (int)(ns > kMaxStages ? kMaxStages : (ns < 1 ? 1 : ns));
        if (v.ns >= 20) break;
    }
    if (env_ns && std::atoi(env_ns) > 0 && std::atoi(env_ns) < v.ns) v.ns = std::atoi(env_ns);
    v.swap = (A->nnz_elide * 16 >= c->elide_bytes);
    v.fma = c->fma != 0;
    v.ns_magic = (uint32_t)((1ull << 32) / (uint64_t)v.ns + 1);
    v.spb = kBlock / kSlice;
    v.nvb = A->nblocks;
    v.prefetch = true;
    return v;
}

size_t pipe_smem_bytes(const SellView& v, size_t extra) {
    return (size_t)kBarBytes + (size_t)v.ns * v.stage_bytes + extra;
}

unsigned pipe_grid(const zk_csr* A) {
    int64_t g = A->nblocks < num_sms() ? A->nblocks : num_sms();
    return (unsigned)(g > 0 ? g : 1);
}

// Plain (reduction-free) SpMV launches: pipeline blocks of v.spb slices --
// 16 (512 rows) for large matrices, fewer when the matrix has fewer blocks
// than two per SM, so every SM streams -- and its grid.
unsigned plain_grid(const zk_csr* A, SellView& v) {
    const int64_t want = 2 * (int64_t)num_sms();
    // 16 slices (512 rows) per pipeline block: a finer last wave than the
    // 4096-row reduction block (C4 SpMV 712 -> 704 us; 32 slices: 707)
    int64_t spb = 16;
    if (A->nslices < want * spb) {
        spb = (A->nslices + want - 1) / want;
        if (spb < 4) spb = 4;
    }
    if (const char* e = std::getenv("ZK_SPB")) {  // experiments: pipeline block size in slices
        const int64_t f = std::atoll(e);
        if (f >= 1 && f < spb) spb = f;
    }
    v.spb = (int32_t)spb;
    v.nvb = (A->nslices + spb - 1) / spb;
    {
        // A/B switch (experiments only): "0" the ring only, "8" no width-16 class
        const char* e = std::getenv("ZK_NARROW");
        const int cap = (e && e[0] == '0') ? 0 : (e && e[0] == '8') ? 8 : 16;
        v.narrow_w = (A->n_long == 0 && A->wmax <= cap) ? (A->wmax <= 8 ? 8 : 16) : 0;
    }
    const int64_t g = v.nvb < num_sms() ? v.nvb : num_sms();
    return (unsigned)(g > 0 ? g : 1);
}

namespace {

// Scatter CSR rows into the SELL layout (thread per short row) and the side
// CSR (thread per long row).  Setup only.
// Column indices are range-checked here, on the device (the C ABI must not
// trust them; a host loop over 200M+ entries would dominate an upload).
__global__ void k_sell_scatter(int64_t n_rows, int64_t n_cols, const int64_t* __restrict__ ia,
                               const int64_t* __restrict__ ja, const double2* __restrict__ aa,
                               const int64_t* __restrict__ slice_off, const uint8_t* __restrict__ rowlen,
                               double2* __restrict__ saa, int32_t* __restrict__ sja, int32_t* __restrict__ cmax,
                               unsigned int* bad) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n_rows) return;
    const int len = rowlen[row];
    if (len == 255) return;
    const int64_t base = slice_off[row / kSlice] + (row % kSlice);
    const int64_t lo = ia[row];
    bool ok = true;
    for (int k = 0; k < len; ++k) {
        const int64_t j = ja[lo + k];
        ok &= (j >= 0) & (j < n_cols);
        saa[base + 32 * (int64_t)k] = aa[lo + k];
        sja[base + 32 * (int64_t)k] = ok ? (int32_t)j : 0;
    }
    if (!ok) atomicOr(bad, 1u);
    if (len > 0 && ok) atomicMax(cmax + row / kSlice, (int32_t)ja[lo + len - 1]);  // columns ascend
}

__global__ void k_long_scatter(int32_t n_long, int64_t n_cols, const int32_t* __restrict__ long_row,
                               const int64_t* __restrict__ ia, const int64_t* __restrict__ ja,
                               const double2* __restrict__ aa, const int64_t* __restrict__ long_ia,
                               int32_t* __restrict__ lja, double2* __restrict__ laa, int32_t* __restrict__ cmax,
                               unsigned int* bad) {
    const int li = blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= n_long) return;
    const int64_t lo = ia[long_row[li]], len = long_ia[li + 1] - long_ia[li];
    bool ok = true;
    for (int64_t k = 0; k < len; ++k) {
        const int64_t j = ja[lo + k];
        ok &= (j >= 0) & (j < n_cols);
        lja[long_ia[li] + k] = ok ? (int32_t)j : 0;
        laa[long_ia[li] + k] = aa[lo + k];
    }
    if (!ok) atomicOr(bad, 1u);
    if (len > 0 && ok) atomicMax(cmax + long_row[li] / kSlice, (int32_t)ja[lo + len - 1]);
}

// ---- streamed upload: host CSR -> SELL-32 with the H2D copies pipelined ------
// Row lengths, slice widths and the monotonicity check of the row pointers
// on the device (one thread per row; slice width = widest short row).
__global__ void k_rowinfo(int64_t n_rows, const int64_t* __restrict__ ia, uint8_t* __restrict__ rowlen,
                          int64_t* __restrict__ swidth, unsigned long long* info) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int64_t len = 0;
    if (row < n_rows) {
        len = ia[row + 1] - ia[row];
        if (len < 0) atomicOr(info + 0, 1ull);  // row pointers decrease
        if (len > kShortMax) atomicAdd(info + 1, 1ull);
        rowlen[row] = len > kShortMax ? 255 : (uint8_t)(len < 0 ? 0 : len);
    }
    int64_t w = (row < n_rows && len >= 0 && len <= kShortMax) ? len : 0;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) w = max(w, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)w, d));
    if (lane == 0 && row - lane < n_rows) {
        swidth[row / kSlice] = (int64_t)kSlice * w;
        atomicMax(info + 2, (unsigned long long)w);
    }
}

// Scatter rows [r0, r1) whose entries sit in the staging buffers (entry k of
// the matrix at index k - nz0).
__global__ void k_sell_scatter_chunk(int64_t r0, int64_t r1, int64_t n_cols, const int64_t* __restrict__ ia,
                                     int64_t nz0, const int64_t* __restrict__ ja, const double2* __restrict__ aa,
                                     const int64_t* __restrict__ slice_off, const uint8_t* __restrict__ rowlen,
                                     double2* __restrict__ saa, int32_t* __restrict__ sja, int32_t* __restrict__ cmax,
                                     unsigned int* bad) {
    const int64_t row = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= r1) return;
    const int len = rowlen[row];
    const int64_t base = slice_off[row / kSlice] + (row % kSlice);
    const int64_t lo = ia[row] - nz0;
    bool ok = true;
    for (int k = 0; k < len; ++k) {
        const int64_t j = ja[lo + k];
        ok &= (j >= 0) & (j < n_cols);
        saa[base + 32 * (int64_t)k] = aa[lo + k];
        sja[base + 32 * (int64_t)k] = ok ? (int32_t)j : 0;
    }
    if (!ok) atomicOr(bad, 1u);
    if (len > 0 && ok) atomicMax(cmax + row / kSlice, (int32_t)ja[lo + len - 1]);
}

struct PlainSpmv {
    static constexpr int kNC = 0, kNR = 0, kSV = 0;  // no reductions, no staged operands
    double2* __restrict__ y;
    __device__ __forceinline__ void row(int64_t r, const double2 (&v)[1], const double2 (&)[1], double2 (&)[1],
                                        double (&)[1]) {
        y[r] = v[0];
    }
    __device__ __forceinline__ void finish(const double*) {}
};

template <int WM>
__global__ void __launch_bounds__(32 * NarrowCfg<WM>::warps(1), NarrowCfg<WM>::kMinB)
    k_spmv_narrow(SellView A, const double2* __restrict__ x, double2* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    PlainSpmv body{y};
    narrow_tma_run<WM, 1>(A, x, x, body, smem);
}

__global__ void __launch_bounds__(kPipeThreads, 1) k_spmv(SellView A, const double2* __restrict__ x,
                                                          double2* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    PlainSpmv body{y};
    const RedCfg R{};
    sell_run<1>(A, x, nullptr, body, R, smem);
}

// y = A x fused with <w, y> (DEFAULT_PLAN blocks over y): sparse.spmv then
// vecops.zdot(w, y), bit for bit, in one pass over the matrix.
struct SpmvDotBody {
    static constexpr int kNC = 1, kNR = 0, kSV = 1;  // staged: w
    double2* __restrict__ y;
    double2* result;
    unsigned int* counter;
    bool conj, fma;
    __device__ __forceinline__ void row(int64_t r, const double2 (&v)[1], const double2 (&w)[1], double2 (&tc)[1],
                                        double (&)[1]) {
        y[r] = v[0];
        tc[0] = f1(conj ? conjz(w[0]) : w[0], v[0], fma);
    }
    __device__ void finish(const double* t) {
        *result = make_double2(t[0], t[1]);
        *counter = 0;
    }
};

__global__ void __launch_bounds__(kRedPipeThreads, 1) k_spmv_dot(SellView A, const double2* __restrict__ x,
                                                                 SpmvDotBody body, RedCfg R) {
    extern __shared__ __align__(128) unsigned char smem[];
    sell_run<1>(A, x, nullptr, body, R, smem);
}

template <class T>
T* dalloc(zk_context* c, size_t count) {
    return static_cast<T*>(c->alloc.alloc(sizeof(T) * (count ? count : 1)));
}

// numpy's complex division 1 / d (CDOUBLE_divide, the Smith variant with a
// reciprocal scale, every operation rounded -- checked bitwise against
// np.divide(1.0, d) on 200k values spanning 1e-26..1e26), as build_jacobi
// forms the inverse diagonal (krylov.py:120).
__device__ __forceinline__ double2 np_recip(double2 d) {
    const double br = d.x, bi = d.y;
    if (fabs(br) >= fabs(bi)) {
        if (br == 0.0 && bi == 0.0) return make_double2(__ddiv_rn(1.0, fabs(br)), __ddiv_rn(0.0, fabs(bi)));
        const double rat = __ddiv_rn(bi, br);
        const double scl = __ddiv_rn(1.0, __dadd_rn(br, __dmul_rn(bi, rat)));
        return make_double2(__dmul_rn(__dadd_rn(1.0, __dmul_rn(0.0, rat)), scl),
                            __dmul_rn(__dsub_rn(0.0, __dmul_rn(1.0, rat)), scl));
    }
    const double rat = __ddiv_rn(br, bi);
    const double scl = __ddiv_rn(1.0, __dadd_rn(bi, __dmul_rn(br, rat)));
    return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(1.0, rat), 0.0), scl),
                        __dmul_rn(__dsub_rn(__dmul_rn(0.0, rat), 1.0), scl));
}

// build_jacobi on the device (krylov.py:106-120, CsrMatrix.diagonal
// sparse.py:125-134): the stored diagonal entry of each row i < min(n_rows,
// n_cols) (0 when absent), the first row whose entry is zero, and 1 / d.
__global__ void k_jacobi_build(int64_t n, SellView A, double2* __restrict__ minv, unsigned long long* zero_row) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double2 d = make_double2(0.0, 0.0);
    const int len = A.rowlen[i];
    if (len == 255) {
        int lo = A.long_blk_ptr[i / kBlock], hi = A.long_blk_ptr[i / kBlock + 1] - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int64_t)A.long_row[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        for (int64_t k = A.long_ia[lo]; k < A.long_ia[lo + 1]; ++k)
            if (A.long_ja[k] == i) d = A.long_aa[k];
    } else {
        const int64_t base = A.slice_off[i / kSlice] + (i % kSlice);
        for (int k = 0; k < len; ++k)
            if (A.ja[base + 32 * (int64_t)k] == i) d = A.aa[base + 32 * (int64_t)k];
    }
    if (d.x == 0.0 && d.y == 0.0) atomicMin(zero_row, (unsigned long long)i);
    minv[i] = np_recip(d);
}

}  // namespace

// Returns the first row with a zero diagonal entry, or -1 (minv filled either way).
int64_t jacobi_build_device(zk_context* c, const zk_csr* A, double2* minv) {
    const int64_t n = A->n_rows < A->n_cols ? A->n_rows : A->n_cols;
    if (n <= 0) return -1;
    unsigned long long* zr = reinterpret_cast<unsigned long long*>(c->counter + 2);
    const unsigned long long none = ~0ull;
    ZK_CUDA(cudaMemcpyAsync(zr, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
    const SellView v = sell_view(A, c, 0, 0);
    k_jacobi_build<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(n, v, minv, zr);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
    unsigned long long out = 0;
    ZK_CUDA(cudaMemcpyAsync(&out, zr, sizeof(out), cudaMemcpyDeviceToHost, c->stream));
    ZK_CUDA(cudaStreamSynchronize(c->stream));
    return out == none ? -1 : (int64_t)out;
}

void destroy_sell(zk_csr* A) {
    zk_context* c = A->ctx;
    void* ptrs[] = {A->aa, A->ja, A->slice_off, A->slice_cmax, A->rowlen, A->long_row, A->long_blk_ptr,
                    A->long_ia, A->long_ja, A->long_aa};
    for (void* p : ptrs)
        if (p) c->alloc.free(p);
    delete A;
}

// Builds the SELL matrix from device CSR arrays and the host copy of ia.
zk_csr* build_sell(zk_context* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia_h,
                   const int64_t* ia_d, const int64_t* ja_d, const double2* aa_d) {
    zk_csr* A = new zk_csr();
    std::memset(A, 0, sizeof(*A));
    A->ctx = c;
    A->n_rows = n_rows;
    A->n_cols = n_cols;
    A->nnz = nnz;
    A->nnz_elide = nnz;
    A->nslices = (n_rows + kSlice - 1) / kSlice;
    A->nblocks = (n_rows + kBlock - 1) / kBlock;
    const int64_t nrp = A->nslices * kSlice;
    std::vector<uint8_t> rowlen(nrp, 0);
    std::vector<int64_t> slice_off(A->nslices + 1, 0);
    std::vector<int32_t> long_row;
    std::vector<int32_t> long_blk_ptr(A->nblocks + 1, 0);
    std::vector<int64_t> long_ia(1, 0);
    for (int64_t s = 0; s < A->nslices; ++s) {
        int w = 0;
        for (int r = 0; r < kSlice; ++r) {
            const int64_t row = s * kSlice + r;
            if (row >= n_rows) break;
            const int64_t len = ia_h[row + 1] - ia_h[row];
            if (len > kShortMax) {
                rowlen[row] = 255;
                long_row.push_back((int32_t)row);
                long_ia.push_back(long_ia.back() + len);
                long_blk_ptr[row / kBlock + 1]++;
            } else {
                rowlen[row] = (uint8_t)len;
                w = std::max(w, (int)len);
            }
        }
        slice_off[s + 1] = slice_off[s] + (int64_t)kSlice * w;
    }
    for (int64_t b = 0; b < A->nblocks; ++b) long_blk_ptr[b + 1] += long_blk_ptr[b];
    for (int64_t s = 0; s < A->nslices; ++s)
        A->wmax = std::max<int32_t>(A->wmax, (int32_t)((slice_off[s + 1] - slice_off[s]) / kSlice));
    A->sell_elems = slice_off[A->nslices];
    A->n_long = (int32_t)long_row.size();
    cudaStream_t st = c->stream;
    A->aa = dalloc<double2>(c, A->sell_elems);
    A->ja = dalloc<int32_t>(c, A->sell_elems);
    A->slice_off = dalloc<int64_t>(c, A->nslices + 1);
    A->slice_cmax = dalloc<int32_t>(c, A->nslices);
    ZK_CUDA(cudaMemsetAsync(A->slice_cmax, 0xff, sizeof(int32_t) * (A->nslices ? A->nslices : 1), st));
    A->rowlen = dalloc<uint8_t>(c, nrp);
    ZK_CUDA(cudaMemsetAsync(A->aa, 0, sizeof(double2) * A->sell_elems, st));
    ZK_CUDA(cudaMemsetAsync(A->ja, 0, sizeof(int32_t) * A->sell_elems, st));
    ZK_CUDA(cudaMemcpyAsync(A->slice_off, slice_off.data(), sizeof(int64_t) * slice_off.size(),
                            cudaMemcpyHostToDevice, st));
    ZK_CUDA(cudaMemcpyAsync(A->rowlen, rowlen.data(), nrp, cudaMemcpyHostToDevice, st));
    if (n_rows > 0) {
        k_sell_scatter<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(n_rows, n_cols, ia_d, ja_d, aa_d,
                                                                         A->slice_off, A->rowlen, A->aa, A->ja,
                                                                         A->slice_cmax, c->counter + 1);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
    }
    if (A->n_long) {
        A->long_row = dalloc<int32_t>(c, A->n_long);
        A->long_blk_ptr = dalloc<int32_t>(c, A->nblocks + 1);
        A->long_ia = dalloc<int64_t>(c, A->n_long + 1);
        A->long_ja = dalloc<int32_t>(c, long_ia.back());
        A->long_aa = dalloc<double2>(c, long_ia.back());
        ZK_CUDA(cudaMemcpyAsync(A->long_row, long_row.data(), sizeof(int32_t) * A->n_long, cudaMemcpyHostToDevice, st));
        ZK_CUDA(cudaMemcpyAsync(A->long_blk_ptr, long_blk_ptr.data(), sizeof(int32_t) * long_blk_ptr.size(),
                                cudaMemcpyHostToDevice, st));
        ZK_CUDA(cudaMemcpyAsync(A->long_ia, long_ia.data(), sizeof(int64_t) * long_ia.size(), cudaMemcpyHostToDevice,
                                st));
        k_long_scatter<<<(A->n_long + 255) / 256, 256, 0, st>>>(A->n_long, n_cols, A->long_row, ia_d, ja_d, aa_d,
                                                               A->long_ia, A->long_ja, A->long_aa, A->slice_cmax,
                                                               c->counter + 1);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
    }
    // host vectors are freed on return: wait for the async copies
    unsigned int bad = 0;
    ZK_CUDA(cudaMemcpyAsync(&bad, c->counter + 1, sizeof(bad), cudaMemcpyDeviceToHost, st));
    ZK_CUDA(cudaStreamSynchronize(st));
    if (bad) {
        ZK_CUDA(cudaMemsetAsync(c->counter + 1, 0, sizeof(unsigned int), st));
        destroy_sell(A);
        throw ZkError{ZK_ERR_FORMAT, "column index out of range"};
    }
    return A;
}


// Host CSR -> device SELL-32 without host passes over the rows: ia goes up
// first and the row lengths, slice widths and offsets are computed on the
// device (CUB scan), then ja/aa stream up in chunks of ~kChunkNnz entries
// on a copy stream through two device staging buffers while the scatter of
// the previous chunk runs (int64 -> int32 narrowing and the column range
// check happen in the scatter).  Returns nullptr (nothing allocated that
// is not freed) when the matrix has rows longer than kShortMax -- their side
// CSR is built by build_sell -- after the row pointers were verified.
zk_csr* build_sell_streamed(zk_context* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia_h,
                            const int64_t* ja_h, const double2* aa_h) {
    constexpr int64_t kChunkNnz = int64_t(1) << 25;  // 32M entries: 768 MB per staging buffer
    cudaStream_t st = c->stream;
    if (!c->copy_stream) {
        ZK_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (auto& e : c->up_ev) ZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int64_t nslices = (n_rows + kSlice - 1) / kSlice;
    int64_t* ia_d = dalloc<int64_t>(c, n_rows + 1);
    uint8_t* rowlen = dalloc<uint8_t>(c, nslices * kSlice);
    int64_t* swidth = dalloc<int64_t>(c, nslices + 1);
    int64_t* slice_off = dalloc<int64_t>(c, nslices + 1);
    unsigned long long* info = dalloc<unsigned long long>(c, 4);
    ZK_CUDA(cudaMemsetAsync(info, 0, 4 * sizeof(unsigned long long), st));
    ZK_CUDA(cudaMemsetAsync(rowlen, 0, nslices * kSlice, st));
    ZK_CUDA(cudaMemsetAsync(swidth, 0, sizeof(int64_t) * (nslices + 1), st));
    ZK_CUDA(cudaMemcpyAsync(ia_d, ia_h, sizeof(int64_t) * (n_rows + 1), cudaMemcpyHostToDevice, st));
    k_rowinfo<<<(unsigned)((nslices * kSlice + 255) / 256), 256, 0, st>>>(n_rows, ia_d, rowlen, swidth, info);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
    size_t tmp_bytes = 0;
    ZK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, swidth, slice_off, nslices + 1, st));
    void* tmp = c->alloc.alloc(tmp_bytes ? tmp_bytes : 1);
    ZK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, swidth, slice_off, nslices + 1, st));
    unsigned long long h_info[4];
    int64_t total = 0;
    ZK_CUDA(cudaMemcpyAsync(h_info, info, sizeof(h_info), cudaMemcpyDeviceToHost, st));
    ZK_CUDA(cudaMemcpyAsync(&total, slice_off + nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ZK_CUDA(cudaStreamSynchronize(st));
    c->alloc.free(tmp);
    c->alloc.free(swidth);
    c->alloc.free(info);
    auto release = [&]() {
        c->alloc.free(ia_d);
        c->alloc.free(rowlen);
        c->alloc.free(slice_off);
    };
    if (h_info[0]) {
        release();
        throw ZkError{ZK_ERR_FORMAT, "row pointers are not nondecreasing"};
    }
    if (h_info[1]) {  // long rows: the host-side builder makes their side CSR
        release();
        return nullptr;
    }
    zk_csr* A = new zk_csr();
    std::memset(A, 0, sizeof(*A));
    A->ctx = c;
    A->n_rows = n_rows;
    A->n_cols = n_cols;
    A->nnz = nnz;
    A->nnz_elide = nnz;
    A->nslices = nslices;
    A->nblocks = (n_rows + kBlock - 1) / kBlock;
    A->wmax = (int32_t)h_info[2];
    A->sell_elems = total;
    A->slice_off = slice_off;
    A->rowlen = rowlen;
    A->aa = dalloc<double2>(c, total);
    A->ja = dalloc<int32_t>(c, total);
    A->slice_cmax = dalloc<int32_t>(c, nslices);
    ZK_CUDA(cudaMemsetAsync(A->slice_cmax, 0xff, sizeof(int32_t) * (nslices ? nslices : 1), st));
    ZK_CUDA(cudaMemsetAsync(A->aa, 0, sizeof(double2) * (total ? total : 1), st));
    ZK_CUDA(cudaMemsetAsync(A->ja, 0, sizeof(int32_t) * (total ? total : 1), st));
    // chunked H2D (copy stream) || scatter (compute stream), two staging buffers
    const int64_t cap = nnz < kChunkNnz ? nnz : kChunkNnz;
    int64_t* sja[2];
    double2* saa[2];
    for (int b = 0; b < 2; ++b) {
        sja[b] = dalloc<int64_t>(c, cap);
        saa[b] = dalloc<double2>(c, cap);
    }
    cudaEvent_t* ev_copy = c->up_ev;       // [0], [1]
    cudaEvent_t* ev_free = c->up_ev + 2;   // [2], [3]
    ZK_CUDA(cudaEventRecord(ev_free[0], st));  // staging free once the memsets above are ordered
    ZK_CUDA(cudaEventRecord(ev_free[1], st));
    int64_t r0 = 0, k = 0;
    while (r0 < n_rows) {
        // rows [r0, r1): as many as fit in one staging buffer (rows are <= 65 entries)
        const int64_t nz0 = ia_h[r0];
        const int64_t* lim = std::upper_bound(ia_h + r0 + 1, ia_h + n_rows + 1, nz0 + cap);
        int64_t r1 = (int64_t)(lim - ia_h) - 1;
        if (r1 <= r0) r1 = r0 + 1;
        const int64_t cnt = ia_h[r1] - nz0;
        const int b = (int)(k & 1);
        ZK_CUDA(cudaStreamWaitEvent(c->copy_stream, ev_free[b], 0));
        if (cnt > 0) {
            ZK_CUDA(cudaMemcpyAsync(sja[b], ja_h + nz0, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, c->copy_stream));
            ZK_CUDA(cudaMemcpyAsync(saa[b], aa_h + nz0, sizeof(double2) * cnt, cudaMemcpyHostToDevice, c->copy_stream));
        }
        ZK_CUDA(cudaEventRecord(ev_copy[b], c->copy_stream));
        ZK_CUDA(cudaStreamWaitEvent(st, ev_copy[b], 0));
        k_sell_scatter_chunk<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, st>>>(
            r0, r1, n_cols, ia_d, nz0, sja[b], saa[b], slice_off, rowlen, A->aa, A->ja, A->slice_cmax, c->counter + 1);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
        ZK_CUDA(cudaEventRecord(ev_free[b], st));
        r0 = r1;
        ++k;
    }
    unsigned int bad = 0;
    ZK_CUDA(cudaMemcpyAsync(&bad, c->counter + 1, sizeof(bad), cudaMemcpyDeviceToHost, st));
    ZK_CUDA(cudaStreamSynchronize(st));
    for (int b = 0; b < 2; ++b) {
        c->alloc.free(sja[b]);
        c->alloc.free(saa[b]);
    }
    c->alloc.free(ia_d);
    if (bad) {
        ZK_CUDA(cudaMemsetAsync(c->counter + 1, 0, sizeof(unsigned int), st));
        destroy_sell(A);
        throw ZkError{ZK_ERR_FORMAT, "column index out of range"};
    }
    return A;
}

void spmv_device(zk_context* c, const zk_csr* A, const double2* x, double2* y) {
    if (A->n_rows == 0) return;
    if (A->nnz == 0) {
        ZK_CUDA(cudaMemsetAsync(y, 0, sizeof(double2) * A->n_rows, c->stream));
        return;
    }
    SellView v = sell_view(A, c, 0, 0);
    const unsigned grid = plain_grid(A, v);
    if (v.narrow_w) {
        ZK_NARROW_ATTR(k_spmv_narrow);
        ZK_NARROW_LAUNCH(k_spmv_narrow, v, 1, c->stream, v, x, y);
        ZK_CUDA(cudaGetLastError());
        c->launches++;
        return;
    }
    const size_t smem = pipe_smem_bytes(v, 0);
    ZK_CUDA(cudaFuncSetAttribute(k_spmv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_spmv<<<grid, kPipeThreads, smem, c->stream>>>(v, x, y);
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

void spmv_dot_device(zk_context* c, const zk_csr* A, const double2* x, double2* y, const double2* w, bool conj,
                     double2* result) {
    const size_t extra = RedSmem<1, 0>::kBytes;
    SellView v = sell_view(A, c, extra, 1);
    v.sv[0] = w;
    const size_t smem = pipe_smem_bytes(v, extra);
    const int64_t nb = A->nblocks;
    double* partials = static_cast<double*>(c->scratch_partials(sizeof(double2) * (nb ? nb : 1)));
    const PlanPtrs p = c->plans_for(A->n_rows, kBlock, kComplex);
    ZK_CUDA(cudaFuncSetAttribute(k_spmv_dot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_spmv_dot<<<pipe_grid(A), kRedPipeThreads, smem, c->stream>>>(
        v, x, SpmvDotBody{y, result, c->counter, conj, c->fma != 0},
        RedCfg{p, p, partials, c->counter, 0, fold_slots(c, 2 * (nb ? nb : 1))});
    ZK_CUDA(cudaGetLastError());
    c->launches++;
}

}  // namespace zk
