// delta-chunked P.C.P^T ablation kernel — see DESIGN.md.
#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {
int assign_delta_f32(const float*, const float*, int64_t, int, const float*, const float*, int,
                     const int32_t*, int32_t*, float*, double*, const long long*, cudaStream_t) {
  return PCB_EUNSUP;
}
}  // namespace pcb
