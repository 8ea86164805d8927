// Microbenchmark of the ordered-fold building blocks on one warp:
// dependent __dadd_rn chain latency and stream_fold over ready slots.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2112_06465_b200/csrc -I../include fold_bench.cu
#include <cstdio>
#include "zk_blockred.cuh"
using namespace zk;

__global__ void k_chain(const double* v, int64_t n, double* out, long long* cyc) {
    double t = -0.0;
    long long c0 = clock64();
    for (int64_t i = 0; i < n; i += 16) {
        double w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = v[(i + k) & 1023];
#pragma unroll
        for (int k = 0; k < 16; ++k) t = __dadd_rn(t, w[k]);
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) { *out = t; *cyc = c1 - c0; }
}

template <int NCH>
__global__ void k_sfold(double* slots, int64_t nrows, double* out) {
    double r[NCH];
    stream_fold<NCH>(slots, nrows, r);
    if (threadIdx.x == 0) out[0] = r[0];
}

__global__ void k_fill(double* p, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v + (double)i;
}

int main() {
    double *v, *out, *slots; long long* cyc;
    cudaMalloc(&v, 1024 * 8); cudaMalloc(&out, 64); cudaMalloc(&cyc, 8); cudaMalloc(&slots, 8 * 100000);
    k_fill<<<4, 256>>>(v, 1024, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int64_t n = 1 << 20;
    k_chain<<<1, 32>>>(v, n, out, cyc);
    cudaEventRecord(e0); k_chain<<<1, 32>>>(v, n, out, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("chain: %.2f cycles/add, %.2f ns/add\n", (double)c / n, ms * 1e6 / n);
    for (int nch = 1; nch <= 2; ++nch) {
        int64_t rows = 24414;
        k_fill<<<64, 256>>>(slots, rows * nch, 1.0);
        cudaEventRecord(e0);
        if (nch == 1) k_sfold<1><<<1, 32>>>(slots, rows, out); else k_sfold<2><<<1, 32>>>(slots, rows, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("stream_fold<%d> %lld rows: %.1f us (%.2f ns/row)\n", nch, (long long)rows, ms * 1e3, ms * 1e6 / rows);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
