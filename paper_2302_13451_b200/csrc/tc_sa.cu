// tc_sa.cu — tcgen05 / TMA SA kernels for bf16, D = 64 (placeholder until implemented).
#include "tc_dispatch.h"
#include "ffma_attn.cuh"

namespace sattn {
bool tc_supported(int, int, int, int, bool) { return false; }
sattn_status tc_forward(const AttnArgs&, cudaStream_t) { return SATTN_EUNSUPPORTED; }
sattn_status tc_backward(const AttnArgs&, cudaStream_t) { return SATTN_EUNSUPPORTED; }
int tc_backward_launches() { return 0; }
const char* tc_last_error() { return "tensor-core kernels not built"; }
}  // namespace sattn
