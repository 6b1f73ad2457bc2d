// tcgen05 crossbar VMM kernels (placeholder until the UMMA path lands).
#include "xbs_internal.cuh"

namespace xbs {
bool launch_fwd_tc(xbs_core*, int64_t, double*, cudaStream_t) { return false; }
bool launch_bwd_tc(xbs_core*, int64_t, double*, cudaStream_t) { return false; }
}  // namespace xbs
