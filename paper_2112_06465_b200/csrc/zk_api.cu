// zk_api.cu -- the C ABI (include/zk.h): context, memory, argument checks,
// error mapping.  No C++ exception crosses the boundary.
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "zk_internal.h"

namespace zk {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

size_t Allocator::round(size_t b) {
    if (b < 512) return 512;
    if (b < (1u << 20)) {  // power-of-two classes below 1 MiB
        size_t r = 512;
        while (r < b) r <<= 1;
        return r;
    }
    return (b + (2u << 20) - 1) / (2u << 20) * (2u << 20);  // 2 MiB granules
}

void* Allocator::alloc(size_t bytes) {
    std::lock_guard<std::recursive_mutex> lk(mu_);
    const size_t r = round(bytes);
    auto it = cache_.find(r);
    void* p = nullptr;
    if (it != cache_.end() && !it->second.empty()) {
        p = it->second.back();
        it->second.pop_back();
    } else {
        cudaError_t e = cudaMalloc(&p, r);
        if (e != cudaSuccess) {
            cudaGetLastError();
            release_cached();
            e = cudaMalloc(&p, r);
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw ZkError{ZK_ERR_NOMEM, "device allocation of " + std::to_string(r) + " bytes failed"};
            }
        }
    }
    live_[p] = r;
    in_use_ += r;
    return p;
}

void Allocator::free(void* p) {
    if (!p) return;
    std::lock_guard<std::recursive_mutex> lk(mu_);
    auto it = live_.find(p);
    if (it == live_.end()) throw ZkError{ZK_ERR_PARAMETER, "zk_free: pointer not owned by this context"};
    cache_[it->second].push_back(p);
    in_use_ -= it->second;
    live_.erase(it);
}

void Allocator::release_cached() {
    std::lock_guard<std::recursive_mutex> lk(mu_);
    for (auto& kv : cache_)
        for (void* p : kv.second) cudaFree(p);
    cache_.clear();
}

Allocator::~Allocator() {
    release_cached();
    for (auto& kv : live_) cudaFree(kv.first);
}

int plan_nnodes(zk_context* c, int32_t L, int32_t kind) {
    (void)c;
    if (L <= 0) return 1;
    std::vector<char> buf(build_plan(L, kind, nullptr));
    build_plan(L, kind, buf.data());
    return reinterpret_cast<const PlanHeader*>(buf.data())->nnodes;
}

// launchers (zk_blas1.cu, zk_spmv.cu, zk_bicgstab.cu)
void launch_zscal(zk_context* c, int64_t n, double2 a, double2* x);
void launch_zaxpy(zk_context* c, int64_t n, double2 a, const double2* x, double2* y);
void launch_zaxmy(zk_context* c, int64_t n, const double2* x, double2* y);
void launch_jacobi(zk_context* c, int64_t n, const double2* v, const double2* m, double2* out);
void zdot_device(zk_context* c, int64_t n, const double2* x, const double2* y, bool conj, int64_t block, int mode,
                 double2* result, Gate gate = Gate{nullptr, 0});
void znorm2_device(zk_context* c, int64_t n, const double2* x, int64_t block, int mode, double* result,
                   Gate gate = Gate{nullptr, 0});
zk_csr* build_sell_streamed(zk_context* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia_h,
                            const int64_t* ja_h, const double2* aa_h);
zk_csr* build_sell(zk_context* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia_h,
                   const int64_t* ia_d, const int64_t* ja_d, const double2* aa_d);
void spmv_device(zk_context* c, const zk_csr* A, const double2* x, double2* y);
struct DistSolver;
DistSolver* dist_create(zk_context* c, zk_csr* A, int64_t n_halo, int64_t nnz_global, bool jacobi, int64_t maxit,
                        int nranks, int64_t maxb);
void dist_destroy(DistSolver* D);
void* dist_vector(DistSolver* D, int which, int64_t* len);
void dist_reset(DistSolver* D, double tol, int64_t maxit, bool has_x0);
void dist_phase(DistSolver* D, int phase);
void dist_finish(DistSolver* D, int phase, const int64_t* rank_blocks);
void dist_pack(DistSolver* D, int which, const int64_t* idx, int64_t count, double2* out);
void dist_status(DistSolver* D, zk_solve_report* rep, int32_t* done);
void dist_history(DistSolver* D, double* host, int64_t count);
void spmv_dot_device(zk_context* c, const zk_csr* A, const double2* x, double2* y, const double2* w, bool conj,
                     double2* result);
int bicgstab_device(zk_context* c, zk_csr* A, const double2* b, const double2* minv, const double2* x0, double tol,
                    int64_t maxit, double2* x_out, double* history_host, zk_solve_report* rep);
void destroy_solver_plan(zk_context* c, SolverPlan* P);
void destroy_krylov_plan(zk_context* c, KrylovPlan* P);
int krylov_device(zk_context* c, zk_csr* A, int solver, int ell, const double2* b, const double2* minv,
                  const double2* x0, double tol, int64_t maxit, double2* x_out, double* history_host,
                  zk_solve_report* rep, int32_t* what_j);
void destroy_sell(zk_csr* A);
int64_t jacobi_build_device(zk_context* c, const zk_csr* A, double2* minv);

}  // namespace zk

using namespace zk;

char* zk_context::plan(int32_t L, int32_t kind) {
    auto key = std::make_pair(L, kind);
    auto it = plans.find(key);
    if (it != plans.end()) return it->second;
    size_t bytes = build_plan(L, kind, nullptr);
    std::vector<char> host(bytes);
    build_plan(L, kind, host.data());
    char* d = static_cast<char*>(alloc.alloc(bytes));
    ZK_CUDA(cudaMemcpyAsync(d, host.data(), bytes, cudaMemcpyHostToDevice, stream));
    ZK_CUDA(cudaStreamSynchronize(stream));
    plans[key] = d;
    return d;
}

const char* zk_context::plan_host(int32_t L, int32_t kind) {
    auto key = std::make_pair(L, kind);
    auto it = plans_h.find(key);
    if (it != plans_h.end()) return it->second.data();
    std::vector<char> host(build_plan(L, kind, nullptr));
    build_plan(L, kind, host.data());
    return plans_h.emplace(key, std::move(host)).first->second.data();
}

PlanPtrs zk_context::plans_for(int64_t n, int64_t block, int32_t kind) {
    PlanPtrs p;
    p.full = plan((int32_t)(block - 1), kind);
    int64_t nb = (n + block - 1) / block;
    int64_t tail = n - (nb - 1) * block;
    p.tail = (nb > 0 && tail != block) ? plan((int32_t)(tail - 1), kind) : p.full;
    return p;
}

void* zk_context::scratch_partials(size_t bytes) {
    if (bytes > partials_bytes) {
        if (partials) alloc.free(partials);
        partials = alloc.alloc(bytes);
        partials_bytes = bytes;
    }
    return partials;
}

namespace {

template <class F>
zk_status guarded(F&& f) {
    try {
        f();
        return ZK_OK;
    } catch (const ZkError& e) {
        set_error(e.msg);
        return e.code;
    } catch (const CudaError& e) {
        set_error(std::string("CUDA error ") + cudaGetErrorName(e.err) + " (" + cudaGetErrorString(e.err) + ") in " +
                  e.where);
        return ZK_ERR_CUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return ZK_ERR_CUDA;
    }
}

void need(bool cond, int code, const std::string& msg) {
    if (!cond) throw ZkError{code, msg};
}

void need_ctx(zk_context* c) { need(c != nullptr, ZK_ERR_PARAMETER, "null context"); }

void need_ptr(const void* p, int64_t n, const char* what) {
    need(n == 0 || p != nullptr, ZK_ERR_PARAMETER, std::string("null pointer for ") + what);
}

void check_plan(int64_t block, int mode) {
    need(mode == ZK_MODE_BLOCKED || mode == ZK_MODE_SEQUENTIAL, ZK_ERR_PARAMETER,
         "mode must be 'sequential' or 'blocked'");
    need(block >= 64 && block <= 65536 && (block & (block - 1)) == 0, ZK_ERR_PARAMETER,
         "block_size must be a power of two in [64, 65536], got " + std::to_string(block));
}

inline double2* D2(double* p) { return reinterpret_cast<double2*>(p); }
inline const double2* D2(const double* p) { return reinterpret_cast<const double2*>(p); }

}  // namespace

extern "C" {

const char* zk_last_error(void) { return g_err.c_str(); }
const char* zk_version(void) { return "zk 0.1 sm_100a"; }

zk_status zk_context_create(int device, zk_context** out) {
    return guarded([&] {
        need(out != nullptr, ZK_ERR_PARAMETER, "null output");
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw ZkError{ZK_ERR_NODEVICE, "no CUDA device available (libzk has no CPU fallback)"};
        }
        need(device >= 0 && device < ndev, ZK_ERR_PARAMETER, "device index out of range");
        ZK_CUDA(cudaSetDevice(device));
        zk_context* c = new zk_context();
        c->device = device;
        ZK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->counter = static_cast<unsigned int*>(c->alloc.alloc(sizeof(unsigned int) * 4));
        ZK_CUDA(cudaMemset(c->counter, 0, sizeof(unsigned int) * 4));
        c->d_result = static_cast<double*>(c->alloc.alloc(sizeof(double) * 4));
        ZK_CUDA(cudaMallocHost(&c->h_result, sizeof(double) * 4));
        num_sms();
        *out = c;
    });
}

zk_status zk_context_destroy(zk_context* c) {
    return guarded([&] {
        if (!c) return;
        cudaStreamSynchronize(c->stream);
        for (auto& e : c->events)
            if (e) cudaEventDestroy(e);
        if (c->h_result) cudaFreeHost(c->h_result);
        if (c->bounce) cudaFreeHost(c->bounce);
        for (auto& e : c->bounce_ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : c->up_ev)
            if (e) cudaEventDestroy(e);
        if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
        cudaStreamDestroy(c->stream);
        delete c;
    });
}

zk_status zk_set_arith(zk_context* c, int use_fma, int64_t elide_bytes) {
    return guarded([&] {
        need_ctx(c);
        need(elide_bytes > 0, ZK_ERR_PARAMETER, "elide_bytes must be positive");
        c->fma = use_fma ? 1 : 0;
        c->elide_bytes = elide_bytes;
    });
}

zk_status zk_malloc(zk_context* c, size_t bytes, void** dptr) {
    return guarded([&] {
        need_ctx(c);
        need(dptr != nullptr, ZK_ERR_PARAMETER, "null output");
        std::lock_guard<std::mutex> g(c->mu);
        *dptr = c->alloc.alloc(bytes);
    });
}

zk_status zk_free(zk_context* c, void* dptr) {
    return guarded([&] {
        need_ctx(c);
        std::lock_guard<std::mutex> g(c->mu);
        c->alloc.free(dptr);
    });
}

zk_status zk_host_alloc(size_t bytes, void** hptr) {
    return guarded([&] { ZK_CUDA(cudaMallocHost(hptr, bytes ? bytes : 1)); });
}

zk_status zk_host_free(void* hptr) {
    return guarded([&] { ZK_CUDA(cudaFreeHost(hptr)); });
}

zk_status zk_memcpy_h2d(zk_context* c, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        need_ctx(c);
        if (!bytes) return;
        ZK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    });
}

// Large reads into pageable host memory go through two pinned bounce chunks:
// the DMA of chunk k+1 runs while chunk k is copied out on the host (a
// pageable cudaMemcpy runs at ~4 GB/s here: 30 ms for a C4 solution).
static constexpr size_t kBounce = 8u << 20;

static bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

zk_status zk_memcpy_d2h(zk_context* c, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        need_ctx(c);
        if (!bytes) return;
        if (bytes < 2 * kBounce || host_pinned(dst)) {
            ZK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
            ZK_CUDA(cudaStreamSynchronize(c->stream));
            return;
        }
        if (!c->bounce) {
            ZK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->bounce), 2 * kBounce, cudaHostAllocDefault));
            for (auto& e : c->bounce_ev) ZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const size_t nch = (bytes + kBounce - 1) / kBounce;
        auto issue = [&](size_t k) {
            const size_t off = k * kBounce, len = std::min(kBounce, bytes - off);
            ZK_CUDA(cudaMemcpyAsync(c->bounce + (k & 1) * kBounce, static_cast<const char*>(src) + off, len,
                                    cudaMemcpyDeviceToHost, c->stream));
            ZK_CUDA(cudaEventRecord(c->bounce_ev[k & 1], c->stream));
        };
        issue(0);
        for (size_t k = 0; k < nch; ++k) {
            if (k + 1 < nch) issue(k + 1);  // stream order: chunk k+1's DMA reuses buffer (k+1)&1 only after
                                            // chunk k-1 was copied out below (host order)
            ZK_CUDA(cudaEventSynchronize(c->bounce_ev[k & 1]));
            const size_t off = k * kBounce, len = std::min(kBounce, bytes - off);
            // the copy-out also first-touches the destination's pages: split it over 4 threads
            char* d = static_cast<char*>(dst) + off;
            const char* b = c->bounce + (k & 1) * kBounce;
            const size_t q = (len / 4 + 4095) & ~size_t(4095);
            std::thread t[3];
            for (int i = 1; i < 4; ++i) {
                const size_t lo = std::min(len, i * q), hi = std::min(len, (i + 1) * q);
                if (hi > lo) t[i - 1] = std::thread([=] { std::memcpy(d + lo, b + lo, hi - lo); });
            }
            std::memcpy(d, b, std::min(len, q));
            for (auto& th : t)
                if (th.joinable()) th.join();
        }
    });
}

zk_status zk_memcpy_d2d(zk_context* c, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        need_ctx(c);
        if (!bytes) return;
        ZK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    });
}

zk_status zk_memset(zk_context* c, void* dst, int value, size_t bytes) {
    return guarded([&] {
        need_ctx(c);
        if (!bytes) return;
        ZK_CUDA(cudaMemsetAsync(dst, value, bytes, c->stream));
    });
}


zk_status zk_synchronize(zk_context* c) {
    return guarded([&] {
        need_ctx(c);
        ZK_CUDA(cudaStreamSynchronize(c->stream));
    });
}

zk_status zk_launch_count(zk_context* c, int64_t* count) {
    return guarded([&] {
        need_ctx(c);
        *count = c->launches;
    });
}

zk_status zk_stream(zk_context* c, void** stream) {
    return guarded([&] {
        need_ctx(c);
        *stream = static_cast<void*>(c->stream);
    });
}

zk_status zk_host_register(void* hptr, size_t bytes) {
    return guarded([&] {
        if (!hptr || !bytes) return;
        ZK_CUDA(cudaHostRegister(hptr, bytes, cudaHostRegisterDefault));
    });
}

zk_status zk_host_unregister(void* hptr) {
    return guarded([&] {
        if (!hptr) return;
        ZK_CUDA(cudaHostUnregister(hptr));
    });
}

zk_status zk_event_record(zk_context* c, int slot) {
    return guarded([&] {
        need_ctx(c);
        need(slot >= 0 && slot < 32, ZK_ERR_PARAMETER, "event slot out of range");
        if (!c->events[slot]) ZK_CUDA(cudaEventCreate(&c->events[slot]));
        ZK_CUDA(cudaEventRecord(c->events[slot], c->stream));
    });
}

zk_status zk_event_elapsed(zk_context* c, int a, int b, double* ms) {
    return guarded([&] {
        need_ctx(c);
        need(a >= 0 && a < 32 && b >= 0 && b < 32 && c->events[a] && c->events[b], ZK_ERR_PARAMETER,
             "event slot not recorded");
        ZK_CUDA(cudaEventSynchronize(c->events[b]));
        float f = 0.f;
        ZK_CUDA(cudaEventElapsedTime(&f, c->events[a], c->events[b]));
        *ms = f;
    });
}

zk_status zk_profile_enable(zk_context* c, int on) {
    return guarded([&] {
        need_ctx(c);
        c->profile = on != 0;
        for (int i = 0; i < 16; ++i) {
            c->prof_ms[i] = 0.0;
            c->prof_n[i] = 0;
        }
    });
}

zk_status zk_profile_read(zk_context* c, double* total_ms, int64_t* launches) {
    return guarded([&] {
        need_ctx(c);
        for (int i = 0; i < ZK_NPHASES; ++i) {
            total_ms[i] = c->prof_ms[i];
            launches[i] = c->prof_n[i];
        }
    });
}

zk_status zk_zscal(zk_context* c, int64_t n, double ar, double ai, double* x) {
    return guarded([&] {
        need_ctx(c);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need_ptr(x, n, "x");
        launch_zscal(c, n, make_double2(ar, ai), D2(x));
    });
}

zk_status zk_zaxpy(zk_context* c, int64_t n, double ar, double ai, const double* x, double* y) {
    return guarded([&] {
        need_ctx(c);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need_ptr(x, n, "x");
        need_ptr(y, n, "y");
        launch_zaxpy(c, n, make_double2(ar, ai), D2(x), D2(y));
    });
}

zk_status zk_zaxmy(zk_context* c, int64_t n, const double* x, double* y) {
    return guarded([&] {
        need_ctx(c);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need_ptr(x, n, "x");
        need_ptr(y, n, "y");
        launch_zaxmy(c, n, D2(x), D2(y));
    });
}

zk_status zk_zassign(zk_context* c, int64_t n, double* dst, const double* src) {
    return guarded([&] {
        need_ctx(c);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        if (n == 0 || dst == src) return;
        ZK_CUDA(cudaMemcpyAsync(dst, src, sizeof(double2) * n, cudaMemcpyDeviceToDevice, c->stream));
    });
}

zk_status zk_jacobi_apply(zk_context* c, int64_t n, const double* v, const double* minv, double* out) {
    return guarded([&] {
        need_ctx(c);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need_ptr(v, n, "v");
        need_ptr(minv, n, "minv");
        need_ptr(out, n, "out");
        launch_jacobi(c, n, D2(v), D2(minv), D2(out));
    });
}

zk_status zk_zdotc(zk_context* c, int64_t n, const double* x, const double* y, int conjugate, int64_t block_size,
                   int mode, double* result_host) {
    return guarded([&] {
        need_ctx(c);
        check_plan(block_size, mode);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need(result_host != nullptr, ZK_ERR_PARAMETER, "null result");
        if (n == 0) {  // vecops.py:173-174
            result_host[0] = 0.0;
            result_host[1] = 0.0;
            return;
        }
        need_ptr(x, n, "x");
        need_ptr(y, n, "y");
        zdot_device(c, n, D2(x), D2(y), conjugate != 0, block_size, mode, reinterpret_cast<double2*>(c->d_result));
        ZK_CUDA(cudaMemcpyAsync(c->h_result, c->d_result, sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
        ZK_CUDA(cudaStreamSynchronize(c->stream));
        result_host[0] = c->h_result[0];
        result_host[1] = c->h_result[1];
    });
}

zk_status zk_zdotc_dev(zk_context* c, int64_t n, const double* x, const double* y, int conjugate, int64_t block_size,
                       int mode, double* result_dev) {
    return guarded([&] {
        need_ctx(c);
        check_plan(block_size, mode);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need(result_dev != nullptr, ZK_ERR_PARAMETER, "null result");
        if (n == 0) {
            ZK_CUDA(cudaMemsetAsync(result_dev, 0, sizeof(double2), c->stream));
            return;
        }
        need_ptr(x, n, "x");
        need_ptr(y, n, "y");
        zdot_device(c, n, D2(x), D2(y), conjugate != 0, block_size, mode, reinterpret_cast<double2*>(result_dev));
    });
}

zk_status zk_znorm2_dev(zk_context* c, int64_t n, const double* x, int64_t block_size, int mode, double* result_dev) {
    return guarded([&] {
        need_ctx(c);
        check_plan(block_size, mode);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need(result_dev != nullptr, ZK_ERR_PARAMETER, "null result");
        if (n == 0) {
            ZK_CUDA(cudaMemsetAsync(result_dev, 0, sizeof(double), c->stream));
            return;
        }
        need_ptr(x, n, "x");
        znorm2_device(c, n, D2(x), block_size, mode, result_dev);
    });
}

zk_status zk_znorm2(zk_context* c, int64_t n, const double* x, int64_t block_size, int mode, double* result_host) {
    return guarded([&] {
        need_ctx(c);
        check_plan(block_size, mode);
        need(n >= 0, ZK_ERR_DIMENSION, "negative length");
        need(result_host != nullptr, ZK_ERR_PARAMETER, "null result");
        if (n == 0) {  // vecops.py:192-193
            result_host[0] = 0.0;
            return;
        }
        need_ptr(x, n, "x");
        znorm2_device(c, n, D2(x), block_size, mode, c->d_result);
        ZK_CUDA(cudaMemcpyAsync(c->h_result, c->d_result, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        ZK_CUDA(cudaStreamSynchronize(c->stream));
        result_host[0] = c->h_result[0];
    });
}

static void validate_csr_host(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia, bool monotone = true) {
    need(n_rows >= 0 && n_cols >= 0 && nnz >= 0, ZK_ERR_FORMAT, "negative dimensions");
    need(n_cols <= INT32_MAX, ZK_ERR_FORMAT, "n_cols exceeds the int32 column-index range of the device layout");
    if (n_rows == 0) {
        need(nnz == 0, ZK_ERR_FORMAT, "nonzeros in a 0-row matrix");
        return;
    }
    need(ia != nullptr, ZK_ERR_FORMAT, "null row pointers");
    need(ia[0] == 0 && ia[n_rows] == nnz, ZK_ERR_FORMAT, "row pointers must span [0, nnz]");
    if (monotone)
        for (int64_t i = 0; i < n_rows; ++i) need(ia[i + 1] >= ia[i], ZK_ERR_FORMAT, "row pointers are not nondecreasing");
    // column indices are range-checked on the device while scattering (zk_spmv.cu)
}

zk_status zk_csr_create(zk_context* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia_host,
                        const int64_t* ja_host, const double* aa_host, zk_csr** out) {
    return guarded([&] {
        need_ctx(c);
        need(out != nullptr, ZK_ERR_PARAMETER, "null output");
        validate_csr_host(n_rows, n_cols, nnz, ia_host, /*monotone=*/false);  // monotonicity: on the device
        need(nnz == 0 || (ja_host && aa_host), ZK_ERR_FORMAT, "null column/value arrays");
        std::vector<int64_t> ia0;
        if (n_rows == 0) {
            ia0.assign(1, 0);
            ia_host = ia0.data();
        }
        if (n_rows > 0 && nnz > 0) {  // pipelined upload + device layout build (zk_spmv.cu)
            zk_csr* A = build_sell_streamed(c, n_rows, n_cols, nnz, ia_host, ja_host, D2(aa_host));
            if (A) {
                *out = A;
                return;
            }
        }
        int64_t* ia_d = static_cast<int64_t*>(c->alloc.alloc(sizeof(int64_t) * (n_rows + 1)));
        int64_t* ja_d = static_cast<int64_t*>(c->alloc.alloc(sizeof(int64_t) * (nnz ? nnz : 1)));
        double2* aa_d = static_cast<double2*>(c->alloc.alloc(sizeof(double2) * (nnz ? nnz : 1)));
        ZK_CUDA(cudaMemcpyAsync(ia_d, ia_host, sizeof(int64_t) * (n_rows + 1), cudaMemcpyHostToDevice, c->stream));
        if (nnz) {
            ZK_CUDA(cudaMemcpyAsync(ja_d, ja_host, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, c->stream));
            ZK_CUDA(cudaMemcpyAsync(aa_d, aa_host, sizeof(double2) * nnz, cudaMemcpyHostToDevice, c->stream));
        }
        zk_csr* A = build_sell(c, n_rows, n_cols, nnz, ia_host, ia_d, ja_d, aa_d);
        c->alloc.free(ia_d);
        c->alloc.free(ja_d);
        c->alloc.free(aa_d);
        *out = A;
    });
}

zk_status zk_csr_create_device(zk_context* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* ia,
                               const int64_t* ja, const double* aa, zk_csr** out) {
    return guarded([&] {
        need_ctx(c);
        need(out != nullptr, ZK_ERR_PARAMETER, "null output");
        std::vector<int64_t> ia_h(n_rows + 1, 0);
        if (n_rows > 0)
            ZK_CUDA(cudaMemcpyAsync(ia_h.data(), ia, sizeof(int64_t) * (n_rows + 1), cudaMemcpyDeviceToHost, c->stream));
        ZK_CUDA(cudaStreamSynchronize(c->stream));
        validate_csr_host(n_rows, n_cols, nnz, ia_h.data());
        *out = build_sell(c, n_rows, n_cols, nnz, ia_h.data(), ia, ja, D2(aa));
    });
}

zk_status zk_csr_destroy(zk_csr* A) {
    return guarded([&] {
        if (!A) return;
        zk_context* c = A->ctx;
        cudaStreamSynchronize(c->stream);
        for (int k = 0; k < 2; ++k) destroy_solver_plan(c, A->solver[k]);
        for (int k = 0; k < 4; ++k) destroy_krylov_plan(c, A->kplan[k]);
        destroy_sell(A);
    });
}

zk_status zk_csr_bytes(const zk_csr* A, int64_t* bytes, int64_t* padded) {
    return guarded([&] {
        need(A != nullptr, ZK_ERR_PARAMETER, "null matrix");
        int64_t b = A->sell_elems * (int64_t)(sizeof(double2) + sizeof(int32_t)) + (A->nslices + 1) * 8 +
                    A->nslices * 32;
        if (A->n_long) b += A->n_long * 4 + (A->nblocks + 1) * 4 + (A->n_long + 1) * 8;
        *bytes = b;
        *padded = A->sell_elems;
    });
}

zk_status zk_spmv_dotc(zk_context* c, const zk_csr* A, const double* x, double* y, const double* w, int conjugate,
                       double* result_host) {
    return guarded([&] {
        need_ctx(c);
        need(A != nullptr, ZK_ERR_PARAMETER, "null matrix");
        need(result_host != nullptr, ZK_ERR_PARAMETER, "null result");
        if (A->n_rows == 0) {  // empty y: zdot of empty vectors is (0, 0) (vecops.py:173-174)
            result_host[0] = result_host[1] = 0.0;
            return;
        }
        need_ptr(x, A->n_cols, "x");
        need_ptr(y, A->n_rows, "y");
        need_ptr(w, A->n_rows, "w");
        spmv_dot_device(c, A, D2(x), D2(y), D2(w), conjugate != 0, reinterpret_cast<double2*>(c->d_result));
        ZK_CUDA(cudaMemcpyAsync(c->h_result, c->d_result, sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
        ZK_CUDA(cudaStreamSynchronize(c->stream));
        result_host[0] = c->h_result[0];
        result_host[1] = c->h_result[1];
    });
}

zk_status zk_jacobi_build(zk_context* c, const zk_csr* A, double* minv, int64_t* zero_row) {
    return guarded([&] {
        need_ctx(c);
        need(A != nullptr, ZK_ERR_PARAMETER, "null matrix");
        need(zero_row != nullptr, ZK_ERR_PARAMETER, "null zero_row");
        const int64_t n = A->n_rows < A->n_cols ? A->n_rows : A->n_cols;
        need_ptr(minv, n, "minv");
        const int64_t z = jacobi_build_device(c, A, D2(minv));
        *zero_row = z;
        if (z >= 0)
            throw ZkError{ZK_ERR_SINGULAR, "zero diagonal entry at row " + std::to_string(z) +
                                               "; Jacobi preconditioner is singular"};
    });
}

zk_status zk_spmv(zk_context* c, const zk_csr* A, const double* x, double* y) {
    return guarded([&] {
        need_ctx(c);
        need(A != nullptr, ZK_ERR_PARAMETER, "null matrix");
        need_ptr(x, A->n_cols, "x");
        need_ptr(y, A->n_rows, "y");
        spmv_device(c, A, D2(x), D2(y));
    });
}

zk_status zk_bicgstab(zk_context* c, const zk_csr* A, const double* b, const double* minv, const double* x0,
                      double tol, int64_t maxit, double* x_out, double* history_host, zk_solve_report* rep) {
    int rc = ZK_OK;
    zk_status st = guarded([&] {
        need_ctx(c);
        need(A != nullptr, ZK_ERR_PARAMETER, "null matrix");
        need(A->n_rows == A->n_cols, ZK_ERR_DIMENSION,
             "matrix is " + std::to_string(A->n_rows) + "x" + std::to_string(A->n_cols) + ", not square");
        need(tol > 0, ZK_ERR_PARAMETER, "tolerance must be positive");
        need(maxit >= 1, ZK_ERR_PARAMETER, "max_iterations must be >= 1");
        need(history_host && rep, ZK_ERR_PARAMETER, "null history/report");
        need_ptr(b, A->n_rows, "b");
        need_ptr(x_out, A->n_rows, "x_out");
        std::memset(rep, 0, sizeof(*rep));
        if (A->n_rows == 0) {  // ||b|| = 0: trivial_result (krylov.py:174-178)
            history_host[0] = 0.0;
            rep->converged = 1;
            rep->history_len = 1;
            return;
        }
        rc = bicgstab_device(c, const_cast<zk_csr*>(A), D2(b), minv ? D2(minv) : nullptr, x0 ? D2(x0) : nullptr, tol,
                             maxit, D2(x_out), history_host, rep);
    });
    if (st != ZK_OK) return st;
    if (rc == ZK_ERR_BREAKDOWN) set_error("breakdown");
    return rc;
}

static zk_status krylov_entry(zk_context* c, const zk_csr* A, int solver, int ell, const double* b, const double* minv,
                              const double* x0, double tol, int64_t maxit, double* x_out, double* history_host,
                              zk_solve_report* rep, int32_t* breakdown_index) {
    int rc = ZK_OK;
    zk_status st = guarded([&] {
        need_ctx(c);
        need(A != nullptr, ZK_ERR_PARAMETER, "null matrix");
        need(A->n_rows == A->n_cols, ZK_ERR_DIMENSION,
             "matrix is " + std::to_string(A->n_rows) + "x" + std::to_string(A->n_cols) + ", not square");
        need(tol > 0, ZK_ERR_PARAMETER, "tolerance must be positive");
        need(maxit >= 1, ZK_ERR_PARAMETER, "max_iterations must be >= 1");
        need(ell >= 1, ZK_ERR_PARAMETER, "polynomial degree l must be >= 1");
        need(history_host && rep, ZK_ERR_PARAMETER, "null history/report");
        need_ptr(b, A->n_rows, "b");
        need_ptr(x_out, A->n_rows, "x_out");
        std::memset(rep, 0, sizeof(*rep));
        int32_t j = 0;
        if (A->n_rows == 0) {  // ||b|| = 0: trivial_result (krylov.py:174-178)
            history_host[0] = 0.0;
            rep->converged = 1;
            rep->history_len = 1;
        } else {
            rc = krylov_device(c, const_cast<zk_csr*>(A), solver, ell, D2(b), minv ? D2(minv) : nullptr,
                               x0 ? D2(x0) : nullptr, tol, maxit, D2(x_out), history_host, rep, &j);
        }
        if (breakdown_index) *breakdown_index = j;
    });
    if (st != ZK_OK) return st;
    if (rc == ZK_ERR_BREAKDOWN) set_error("breakdown");
    return rc;
}

zk_status zk_bicgstab_l(zk_context* c, const zk_csr* A, const double* b, const double* minv, const double* x0,
                        double tol, int64_t maxit, int ell, double* x_out, double* history_host,
                        zk_solve_report* rep, int32_t* breakdown_index) {
    return krylov_entry(c, A, 0, ell, b, minv, x0, tol, maxit, x_out, history_host, rep, breakdown_index);
}

zk_status zk_tfqmr(zk_context* c, const zk_csr* A, const double* b, const double* minv, const double* x0, double tol,
                   int64_t maxit, double* x_out, double* history_host, zk_solve_report* rep) {
    return krylov_entry(c, A, 1, 1, b, minv, x0, tol, maxit, x_out, history_host, rep, nullptr);
}

// ---- row-sharded BiCGStab ----------------------------------------------------
struct zk_dshard {
    zk_context* ctx;
    zk::DistSolver* d;
};

zk_status zk_dshard_create(zk_context* c, zk_csr* A, int64_t n_halo, int64_t nnz_global, int jacobi, int64_t maxit,
                           int nranks, int64_t maxb, zk_dshard** out) {
    return guarded([&] {
        need_ctx(c);
        need(A != nullptr && out != nullptr, ZK_ERR_PARAMETER, "null matrix/output");
        need(n_halo >= 0 && A->n_cols == A->n_rows + n_halo, ZK_ERR_DIMENSION,
             "shard columns must be its rows plus the halo");
        need(A->n_rows > 0, ZK_ERR_DIMENSION, "empty shard");
        need(maxit >= 1, ZK_ERR_PARAMETER, "max_iterations must be >= 1");
        need(nranks >= 1 && nranks <= 64, ZK_ERR_PARAMETER, "1..64 ranks");
        need(maxb >= (A->n_rows + 4095) / 4096, ZK_ERR_PARAMETER, "max_blocks below this shard's block count");
        need(nnz_global >= A->nnz, ZK_ERR_PARAMETER, "global nnz below the shard's");
        zk_dshard* h = new zk_dshard{c, zk::dist_create(c, A, n_halo, nnz_global, jacobi != 0, maxit, nranks, maxb)};
        *out = h;
    });
}

zk_status zk_dshard_destroy(zk_dshard* h) {
    return guarded([&] {
        if (!h) return;
        zk::dist_destroy(h->d);
        delete h;
    });
}

zk_status zk_dshard_vector(zk_dshard* h, int which, double** dptr, int64_t* len) {
    return guarded([&] {
        need(h && dptr && len, ZK_ERR_PARAMETER, "null argument");
        *dptr = static_cast<double*>(zk::dist_vector(h->d, which, len));
    });
}

zk_status zk_dshard_reset(zk_dshard* h, double tol, int64_t maxit, int has_x0) {
    return guarded([&] {
        need(h != nullptr, ZK_ERR_PARAMETER, "null shard");
        need(tol > 0, ZK_ERR_PARAMETER, "tolerance must be positive");
        need(maxit >= 1, ZK_ERR_PARAMETER, "max_iterations must be >= 1");
        zk::dist_reset(h->d, tol, maxit, has_x0 != 0);
    });
}

zk_status zk_dshard_phase(zk_dshard* h, int phase) {
    return guarded([&] {
        need(h != nullptr, ZK_ERR_PARAMETER, "null shard");
        zk::dist_phase(h->d, phase);
    });
}

zk_status zk_dshard_finish(zk_dshard* h, int phase, const int64_t* rank_blocks) {
    return guarded([&] {
        need(h != nullptr && rank_blocks != nullptr, ZK_ERR_PARAMETER, "null argument");
        zk::dist_finish(h->d, phase, rank_blocks);
    });
}

zk_status zk_dshard_pack(zk_dshard* h, int which, const int64_t* idx, int64_t count, double* out) {
    return guarded([&] {
        need(h != nullptr, ZK_ERR_PARAMETER, "null shard");
        need(count >= 0, ZK_ERR_DIMENSION, "negative count");
        zk::dist_pack(h->d, which, idx, count, D2(out));
    });
}

zk_status zk_dshard_status(zk_dshard* h, zk_solve_report* rep, int32_t* done) {
    return guarded([&] {
        need(h && rep && done, ZK_ERR_PARAMETER, "null argument");
        zk::dist_status(h->d, rep, done);
    });
}

zk_status zk_dshard_history(zk_dshard* h, double* host, int64_t count) {
    return guarded([&] {
        need(h && host, ZK_ERR_PARAMETER, "null argument");
        zk::dist_history(h->d, host, count);
    });
}

}  // extern "C"
