// bf16 tcgen05 dense transform (placeholder until the tensor-core kernels land).
#include "common.cuh"

namespace gnnv {
bool gemm_fwd_tc(const GemmFwdArgs&, cudaStream_t) { return false; }
bool gemm_dx_tc(const GemmDxArgs&, cudaStream_t) { return false; }
bool gemm_dw_tc(const GemmDwArgs&, cudaStream_t) { return false; }
}  // namespace gnnv
