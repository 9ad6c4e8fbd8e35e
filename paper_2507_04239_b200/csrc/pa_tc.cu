// bf16 tcgen05 pipeline (placeholder until the tensor-core kernels land).
#include "pa_tc.cuh"

namespace pa {
bool tc_supported(const Geo&, int) { return false; }
size_t tc_fwd_workspace_bytes(const Geo&) { return 0; }
size_t tc_bwd_workspace_bytes(const Geo&) { return 0; }
int tc_forward(const Geo&, const void*, const void*, const void*, const float*, void*, float*, void*,
               cudaStream_t) { return 4; }
int tc_backward(const Geo&, const void*, const void*, const void*, const float*, const void*,
                const float*, const void*, void*, void*, void*, float*, const void*, void*,
                cudaStream_t) { return 4; }
}  // namespace pa
