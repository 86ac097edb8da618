// placeholder until the tcgen05 engine lands
#include "common.cuh"
#include "ops.h"
namespace gpic {
int launch_affinity_tc(const float*, const float*, const float*, int64_t, int32_t, int64_t,
                       int64_t, float, float*, int64_t, float*, int64_t, cudaStream_t) {
  return fail(GPIC_E_UNSUPPORTED, "tcgen05 affinity engine not built");
}
}  // namespace gpic
