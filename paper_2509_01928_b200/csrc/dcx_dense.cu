// Dense tensor-core path -- placeholder until the tcgen05 kernel lands.
#include <stdexcept>
#include "dcx_dense.h"

namespace dcx {

void DenseDev::release() {
  if (q16) cudaFree(q16);
  q16 = nullptr;
  n = 0;
}

void dense_upload(DenseDev& d, int64_t n, const double*, cudaStream_t) {
  d.release();
  d.n = n;
}
void dense_begin(DenseDev&, MultiPass&, cudaStream_t) {
  throw std::runtime_error("dense tensor-core path not built yet");
}
void dense_step(DenseDev&, MultiPass&, int, cudaStream_t) {
  throw std::runtime_error("dense tensor-core path not built yet");
}
void dense_finish(DenseDev&, MultiPass&, cudaStream_t) {}
void dense_profile(DenseDev&, MultiPass&, int, cudaEvent_t, cudaEvent_t, cudaStream_t) {
  throw std::runtime_error("dense tensor-core path not built yet");
}

}  // namespace dcx
