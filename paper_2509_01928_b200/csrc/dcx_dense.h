// Dense tensor-core path (K2000-style fully connected couplings): declarations.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "dcx_internal.h"

namespace dcx {

// Device operands of the dense path. J is held as exact small integers
// (J = scale * Q, Q in int8) expanded once into the MMA operand layout.
struct DenseDev {
  int64_t n = 0;
  void* q16 = nullptr;  // fp16 operand tiles of Q (padded)
  double scale = 1.0;
  bool exact_int = false;
  void release();
};

void dense_upload(DenseDev& d, int64_t n, const double* A, cudaStream_t s);
void dense_begin(DenseDev& d, MultiPass& m, cudaStream_t s);
void dense_step(DenseDev& d, MultiPass& m, int chunk, cudaStream_t s);
void dense_finish(DenseDev& d, MultiPass& m, cudaStream_t s);
void dense_profile(DenseDev& d, MultiPass& m, int launches, cudaEvent_t a, cudaEvent_t b, cudaStream_t s);

}  // namespace dcx
