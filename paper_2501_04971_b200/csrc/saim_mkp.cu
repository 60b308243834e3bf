// saim_mkp.cu -- fused SAIM kernel for linear objectives with M <= 32 constraints (MKP).
// (placeholder: planned in DESIGN.md; saim_create rejects MKP until it lands)
#include <cuda_runtime.h>
#include <cstdint>
#include "saim_layout.h"

namespace saim {
int mkp_plan(int, int, int, int *, int *, int *) { return -1; }
void mkp_blob_layout(int, int, int, uint32_t *a, uint32_t *c, uint32_t *x, uint32_t *bytes) { *a = *c = *x = *bytes = 0; }
cudaError_t mkp_launch(const RunArgs &, int, int, int, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace saim
