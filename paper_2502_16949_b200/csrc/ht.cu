// TransH / TransR kernels (placeholder until the ht path lands).
#include "common.cuh"
#include "ht.cuh"

namespace skg {

int64_t ht_work_floats(int, int64_t rows, int64_t de, int64_t dr, int64_t R) {
  return 4 * rows * (de > dr ? de : dr) + R * (de * dr + de + dr) + 64;
}
void ht_train_batch(int, const FwdArgs&, const BwdArgs&, float*, int, cudaStream_t, const std::function<void()>*) {
  throw CudaError("TransH/TransR training path not built yet");
}
void ht_score(int, const FwdArgs&, float*, int, cudaStream_t) { throw CudaError("ht score not built yet"); }
void ht_score_backward(int, const FwdArgs&, const BwdArgs&, float*, float*, float*, int, cudaStream_t) {
  throw CudaError("ht backward not built yet");
}

}  // namespace skg

namespace skg {
void configure_ht_kernels() {}
}  // namespace skg
