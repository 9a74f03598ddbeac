// Data-parallel replicas over NCCL (placeholder until the DP path lands).
#include "common.cuh"
#include "engine.cuh"
#include "ht.cuh"

namespace skg {
struct DpState {};
void dp_destroy(skg_ctx* ctx) {
  delete ctx->dp;
  ctx->dp = nullptr;
}
void dp_train_epoch(skg_ctx*, const skg_model_config&, const skg_train_config&, int64_t, float, skg_epoch_report*) {
  throw CudaError("data-parallel path not built yet");
}
}  // namespace skg

extern "C" {
skg_status skg_nccl_unique_id(char out[128]) {
  (void)out;
  return SKG_ERR_CUDA;
}
skg_status skg_dp_init(skg_ctx* ctx, const char*, int, int) {
  ctx->err = "data-parallel path not built yet";
  return SKG_ERR_CUDA;
}
}
