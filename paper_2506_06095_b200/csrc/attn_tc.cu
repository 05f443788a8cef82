// attn_tc.cu — tcgen05/TMEM/TMA block-wise masked attention (placeholder until the kernel lands).
#include "common.cuh"

namespace sf {
sf_status attn_tc(const sf_attn_args&, const sf_bsr_dev&, cudaStream_t, bool) {
    return fail(SF_PLAN_ERROR, "tcgen05 attention kernel not built for this shape");
}
}  // namespace sf
