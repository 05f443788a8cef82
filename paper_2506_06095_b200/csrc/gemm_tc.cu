// gemm_tc.cu — tcgen05 GEMM with fused epilogue (placeholder).
#include "common.cuh"
using namespace sf;
extern "C" sf_status sf_gemm_fused(const sf_gemm_args*, void*) {
    return fail(SF_BACKEND_ERROR, "sf_gemm_fused: not built yet");
}
extern "C" sf_status sf_mi_chain(int32_t, int32_t, int32_t, const void*, int64_t, const sf_gemm_epilogue*, void*,
                                 int64_t, void*) {
    return fail(SF_BACKEND_ERROR, "sf_mi_chain: not built yet");
}
