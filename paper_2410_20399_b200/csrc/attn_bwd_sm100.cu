// attn_bwd_sm100.cu — attention backward (placeholder until the sm_100a kernel lands).
#include <cuda_runtime.h>

#include "attn_common.cuh"

namespace tkb {
int launch_attn_bwd(int, bool, const BwdParams&, int, const void*, const void*, int64_t, int64_t, int64_t, void*,
                    cudaStream_t, int* launches) {
    *launches = 0;
    return (int)cudaErrorNotSupported;
}
}  // namespace tkb
