// lopt_fast.cu -- phases 1 and 2 in fast mode (placeholder until the
// tensor-core path lands; plans in fast mode report LOPT_ERR_UNSUPPORTED).
#include "lopt_common.cuh"

namespace lopt {

int fast_supported(const DevicePlan &) { return 0; }
void launch_fast_stats(const DevicePlan &, cudaStream_t) {}
void launch_fast_apply(const DevicePlan &, cudaStream_t) {}
int64_t fast_stat_chunk() { return 8192; }
int64_t fast_apply_chunk() { return 4096; }

}  // namespace lopt
