// lsdf_mlp_tc.cu — TinyMlp layer 2 on tcgen05 tensor cores (placeholder until
// the kind::tf32 kernel lands; returns LSDF_ERR_UNSUPPORTED so callers fall
// back to the CUDA-core kernel explicitly, never silently).
#include "lsdf_common.cuh"

int lsdf_mlp_predict_tc(const float*, const float*, const float*, const float*, int32_t, int64_t, const double*,
                        int64_t, float*, cudaStream_t) {
    return lsdf::fail(LSDF_ERR_UNSUPPORTED, "tcgen05 TinyMlp path not built yet");
}
