// lsdf_capi.cu — library-wide state: thread-local error text, launch counter, version.
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
