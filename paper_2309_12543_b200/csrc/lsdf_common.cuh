// lsdf_common.cuh — error plumbing and launch bookkeeping shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/linksdf_b200.h"

namespace lsdf {

std::string& last_error();
std::atomic<uint64_t>& launch_counter();
size_t& l2_persist_bytes(int dev);
// raises the kernel's dynamic shared-memory limit to `bytes` on the current device (once per device)
int ensure_smem(const void* func, size_t bytes, const char* what);

inline int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error() = buf;
    return code;
}

inline int check_launch(const char* what) {
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LSDF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return LSDF_OK;
}

inline int check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) return fail(LSDF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return LSDF_OK;
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// SM count of the current device (cached per thread and device)
inline int sm_count() {
    thread_local int dev_cached = -1, n_sm = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        dev_cached = dev;
    }
    return n_sm;
}

#define LSDF_TRY(expr)                 \
    do {                               \
        int _rc = (expr);              \
        if (_rc != LSDF_OK) return _rc; \
    } while (0)

}  // namespace lsdf
