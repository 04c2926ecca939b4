// stubs.cu — entry points not built yet (raise InvalidOperation).
#include "internal.cuh"

namespace sfg {
sfg_tensor* coo_to_csc(sfg_context*, const sfg_tensor*) { raise(SFG_ERR_INVALID_OPERATION, "CSC: not built yet"); }
sfg_tensor* coo_to_bcsr(sfg_context*, const sfg_tensor*, int64_t, int64_t, int) { raise(SFG_ERR_INVALID_OPERATION, "BCSR: not built yet"); }
void spmm(sfg_context*, const sfg_tensor*, const void*, int, int64_t, int64_t, float*, int64_t, bool) { raise(SFG_ERR_INVALID_OPERATION, "spmm: not built yet"); }
}  // namespace sfg
