// Tensor-core (mma.sync IMMA u8 x s8) quantized decode -- see DESIGN.md 4.2.
#include "common.cuh"
#include "qcache.cuh"

namespace tkv {

bool imma_supported(const QC &c, int G) { (void)c; (void)G; return false; }

int quant_decode_imma(const QC &c, const uint16_t *q, int G, float *out, void *ws, cudaStream_t st) {
  (void)c; (void)q; (void)G; (void)out; (void)ws; (void)st;
  return fail(TKV_ERR_PARAMETER, "tensor-core decode not built");
}

}  // namespace tkv
