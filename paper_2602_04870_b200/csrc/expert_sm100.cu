// expert_sm100.cu — tcgen05/TMEM block-sparse expert FFN kernels (sm_100a).  [in progress]
#include "kernels.h"

namespace mhl {

bool expert_fwd_sm100_supported(int d_h, int d_e) { (void)d_h; (void)d_e; return false; }

void launch_expert_fwd_sm100(const Tile*, const int32_t*, int, const void*, int64_t, const int32_t*, const float*,
                             const void*, const void*, int64_t, int, int, int, int, void*, int, cudaStream_t) {}

}  // namespace mhl
