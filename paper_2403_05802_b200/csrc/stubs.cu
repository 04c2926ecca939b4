// stubs.cu — entry points not built yet.
#include "internal.cuh"

namespace sfg {
// Tensor-core BCSR SpMM: not built yet, the CUDA-core path handles BCSR.
bool spmm_bcsr_tc(sfg_context*, const sfg_tensor*, const void*, int, int64_t, int64_t, float*,
                  int64_t, bool) {
  return false;
}
}  // namespace sfg
