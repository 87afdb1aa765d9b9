// GPU operand assembly (assemble_hmatrix, /root/reference/pkg/src/hmat/hmatrix.py:97-118).
// Placeholder until the batched ACA kernel lands: reports "unsupported".
#include <cuda_runtime.h>

#include "hx_internal.h"

extern "C" int hx_assemble(hx_ctx*, int, const hx_tree*, const double*, int, int, double,
                           double, int8_t*, int32_t*, int64_t*, int64_t*, int64_t*, int64_t*) {
  return hx::fail(HX_EUNSUPPORTED, "GPU assembly not built yet");
}
