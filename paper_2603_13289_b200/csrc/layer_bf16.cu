// layer_bf16.cu -- RK_BF16 layer path (tcgen05 GEMMs + flash attention).
#include "layer.h"

namespace rk {
void run_layer_bf16(rk_engine*, rk_weights*, rk_context*, int, float*, Rows, bool, int, float*, int, int,
                    void*, void*) {
  raise(RK_ERR_RUNTIME, "bf16 path not built yet");
}
void last_row_logits_bf16(rk_engine*, rk_weights*, const float*, float*) {
  raise(RK_ERR_RUNTIME, "bf16 path not built yet");
}
}  // namespace rk
