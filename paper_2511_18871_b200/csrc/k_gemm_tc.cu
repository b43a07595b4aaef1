// tcgen05 GEMM (placeholder until the tensor-core kernel lands).
#include "internal.cuh"
namespace parl_gpu {
bool gemm_tc(const GemmArgs&, cudaStream_t) { return false; }
}  // namespace parl_gpu
