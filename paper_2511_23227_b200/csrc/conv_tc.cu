// conv_tc.cu -- tcgen05 / TMEM tensor-core engines (placeholder).
#include "conv.cuh"

namespace npcg {
struct TcPlan {};
void destroy_tc_plan(TcPlan* p) { delete p; }
bool tc_supported(int64_t, int64_t, int64_t, int64_t) { return false; }
void tc_forward(npcg_context*, npcg_neighbors*, const float*, const float*, float*) {
  fail(NPCG_ERR_UNSUPPORTED, "tensor-core path not built");
}
void tc_backward(npcg_context*, npcg_neighbors*, const float*, const float*, const float*, float*,
                 float*) {
  fail(NPCG_ERR_UNSUPPORTED, "tensor-core path not built");
}
void tc_prepare(npcg_context*, npcg_neighbors*) {}
}  // namespace npcg
