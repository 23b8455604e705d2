// lsdf_capi.cu — library-wide state: thread-local error text, launch counter, version.
#include <map>
#include <mutex>
#include <utility>

#include "lsdf_common.cuh"

namespace lsdf {
std::string& last_error() {
    static thread_local std::string s;
    return s;
}
std::atomic<uint64_t>& launch_counter() {
    static std::atomic<uint64_t> n{0};
    return n;
}

// Static + dynamic shared memory above 48 KB needs a per-function attribute,
// and function attributes live in each device's context: track what was
// granted per (device, kernel) so a process driving several GPUs raises it on
// each (one attribute call per device and kernel, then a map lookup).
int ensure_smem(const void* func, size_t bytes, const char* what) {
    int dev = 0;
    LSDF_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> granted;
    std::lock_guard<std::mutex> lock(mu);
    size_t& g = granted[{dev, func}];
    if (bytes <= g) return LSDF_OK;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(LSDF_ERR_UNSUPPORTED, "%s: %zu B of shared memory: %s", what, bytes, cudaGetErrorString(e));
    }
    g = bytes;
    return LSDF_OK;
}
}  // namespace lsdf

extern "C" const char* lsdf_version(void) { return "linksdf-b200 0.1.0 (sm_100a)"; }
extern "C" const char* lsdf_last_error(void) { return lsdf::last_error().c_str(); }
extern "C" uint64_t lsdf_launch_count(void) { return lsdf::launch_counter().load(); }

// Device address of page-locked host memory (mapped under UVA), so kernels
// can read inputs / write results across PCIe without staging copies.
extern "C" int lsdf_host_device_pointer(void* host, void** dev) {
    cudaError_t e = cudaHostGetDevicePointer(dev, host, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return lsdf::fail(LSDF_ERR_CUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
    }
    return LSDF_OK;
}

// Persisting-L2 set-aside (bytes granted per device), read by the query
// launches that attach an access-policy window over the link grids.
namespace lsdf {
size_t& l2_persist_bytes(int dev) {
    static size_t granted[64] = {0};
    return granted[dev & 63];
}
}  // namespace lsdf

extern "C" int lsdf_l2_reserve(size_t bytes, size_t* granted) {
    int dev = 0;
    LSDF_TRY(lsdf::check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
    int max_persist = 0;
    LSDF_TRY(lsdf::check_cuda(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev),
                              "cudaDevAttrMaxPersistingL2CacheSize"));
    size_t want = bytes < (size_t)max_persist ? bytes : (size_t)max_persist;
    // the set-aside only grows: several trajectories may share the device
    if (want < lsdf::l2_persist_bytes(dev)) want = lsdf::l2_persist_bytes(dev);
    LSDF_TRY(lsdf::check_cuda(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want), "persisting L2 limit"));
    size_t got = 0;
    LSDF_TRY(lsdf::check_cuda(cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize), "persisting L2 limit"));
    lsdf::l2_persist_bytes(dev) = got;
    if (granted) *granted = got;
    return LSDF_OK;
}
