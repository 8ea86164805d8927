// zk_internal.h -- host-side objects behind the C ABI (include/zk.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/zk.h"
#include "zk_plan.h"
#include "zk_reduce.cuh"

namespace zk {

void set_error(const std::string& msg);

struct CudaError {
    cudaError_t err;
    std::string where;
};

#define ZK_CUDA(call)                                                             \
    do {                                                                          \
        cudaError_t _e = (call);                                                  \
        if (_e != cudaSuccess) throw ::zk::CudaError{_e, #call};                  \
    } while (0)

struct ZkError {
    int code;
    std::string msg;
};

// Size-class caching allocator over cudaMalloc (cudaFree synchronises the
// device, and the reference test-suite creates thousands of small vectors).
// Thread-safe: ctypes releases the GIL during calls, so a DeviceBuffer's
// finaliser may free on one thread while another call allocates.
class Allocator {
public:
    void* alloc(size_t bytes);
    void free(void* p);
    void release_cached();
    size_t bytes_in_use() const { return in_use_; }
    ~Allocator();

private:
    static size_t round(size_t b);
    std::map<size_t, std::vector<void*>> cache_;
    std::map<void*, size_t> live_;
    size_t in_use_ = 0;
    std::recursive_mutex mu_;
};

struct SolverPlan;   // zk_bicgstab.cu
struct KrylovPlan;   // zk_krylov.cu

}  // namespace zk

// SELL-32 device matrix (see zk_spmv.cu for the layout).
struct zk_csr {
    zk_context* ctx;
    int64_t n_rows, n_cols, nnz;
    int64_t nnz_elide;              // nnz numpy's temporary-elision rule sees (the unsharded matrix's)
    int64_t nslices, nblocks;       // 32-row slices, 4096-row blocks
    int64_t sell_elems;             // padded element count
    int32_t wmax;                   // widest slice (entries per row)
    double2* aa;                    // [sell_elems]
    int32_t* ja;                    // [sell_elems]
    int64_t* slice_off;             // [nslices + 1]
    int32_t* slice_cmax;            // [nslices] largest column index of the slice (-1: none)
    uint8_t* rowlen;                // [nslices * 32]; 255 = long row
    int32_t n_long;
    int32_t* long_row;              // [n_long]
    int32_t* long_blk_ptr;          // [nblocks + 1]
    int64_t* long_ia;               // [n_long + 1]
    int32_t* long_ja;
    double2* long_aa;
    zk::SolverPlan* solver[2];      // BiCGStab [identity, jacobi]
    zk::KrylovPlan* kplan[4];       // [BiCGSTAB(l) identity, jacobi, TFQMR identity, jacobi]
};

struct zk_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // matrix upload pipeline (zk_spmv.cu build_sell_streamed)
    cudaEvent_t up_ev[4] = {};
    zk::Allocator alloc;
    std::map<std::pair<int32_t, int32_t>, char*> plans;  // (L, kind) -> device plan
    int fma = 1;
    int64_t elide_bytes = 262144;
    // scratch for API reductions
    void* partials = nullptr;
    size_t partials_bytes = 0;
    unsigned int* counter = nullptr;
    double* d_result = nullptr;    // 4 doubles
    double* h_result = nullptr;    // pinned, 4 doubles
    char* bounce = nullptr;        // pinned 2 x 8 MB: chunked reads into pageable memory
    cudaEvent_t bounce_ev[2] = {};
    int64_t launches = 0;          // kernels launched by this context
    cudaEvent_t events[32] = {};   // zk_event_record slots
    bool profile = false;          // zk_profile_enable
    double prof_ms[32] = {};  // >= ZK_NPHASES
    int64_t prof_n[32] = {};
    std::mutex mu;

    char* plan(int32_t L, int32_t kind);
    const char* plan_host(int32_t L, int32_t kind);       // host copy of the same plan
    std::map<std::pair<int32_t, int32_t>, std::vector<char>> plans_h;
    zk::PlanPtrs plans_for(int64_t n, int64_t block, int32_t kind);
    void* scratch_partials(size_t bytes);
    // streaming-fold slots (zk_blas1.cu): kept filled with the empty marker
    double* slots = nullptr;
    int64_t slots_n = 0;
};

namespace zk {
int num_sms();
// count doubles of streaming-fold slots (zk_blockred.cuh), all at the empty
// marker between passes; grown on demand (zk_blas1.cu)
double* fold_slots(zk_context* c, int64_t count);
}
