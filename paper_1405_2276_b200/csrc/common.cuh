// common.cuh — shared definitions for the fastkf B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace fkb {

// Error classes mirror the reference's exception taxonomy:
//   invalid_argument → status 1, runtime_error → status 2, CUDA failure → status 3.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define FKB_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            throw ::fkb::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                                   __FILE__ + ":" + std::to_string(__LINE__));                \
    } while (0)

#define FKB_LAUNCH_CHECK() FKB_CUDA(cudaGetLastError())

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }

// Device buffer with RAII; plain pointers cross the C-ABI.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) FKB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Launch counter: every kernel launch of this library goes through count_launch()
// so bench.py can report gpu_launches honestly.
extern unsigned long long g_launches;
extern int g_sync_check;  // FKB_SYNC_CHECK=1: synchronize + check after every launch (debug)
void sync_check(const char* where);
inline void count_launch(int k = 1) {
    g_launches += (unsigned long long)k;
    if (g_sync_check) sync_check("count_launch");
}

}  // namespace fkb
