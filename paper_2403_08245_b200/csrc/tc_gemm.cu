// tcgen05 grouped GEMM engine (placeholder until the kernel lands).
#include "common.cuh"

namespace smoe {
bool tc_available() { return false; }
int tc_scatter2scatter(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                       const int32_t *, int64_t, int, int, int, int, int, int, void *, void *,
                       const void *, cudaStream_t) {
  return fail(SMOE_ENOTSUP, "tcgen05 engine not built");
}
int tc_group_xty(const void *, const void *, const int32_t *, int, int64_t, int64_t, int64_t, void *,
                 cudaStream_t) {
  return fail(SMOE_ENOTSUP, "tcgen05 engine not built");
}
}  // namespace smoe
