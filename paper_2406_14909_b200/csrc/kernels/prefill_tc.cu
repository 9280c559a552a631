// prefill_tc.cu -- placeholder until the tcgen05 kernel lands.
#include <cuda_runtime.h>

#include "../moa_internal.h"

namespace moa {
int launch_prefill_bf16_tc(const PrefillArgs &a, void *stream) {
  (void)a;
  (void)stream;
  return (int)cudaErrorNotSupported;
}
}  // namespace moa
