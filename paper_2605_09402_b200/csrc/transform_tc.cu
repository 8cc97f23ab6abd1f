// tcgen05 transform backend: placeholder until the tensor-core kernel lands.
#include "internal.cuh"

namespace atlas {

bool launch_transform_tc(const float*, int64_t, int64_t, int64_t,
                         const float*, const float*, int64_t, int, void*, int,
                         int64_t, cudaStream_t) {
  return false;
}

}  // namespace atlas
