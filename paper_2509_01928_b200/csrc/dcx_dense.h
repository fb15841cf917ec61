// Dense tensor-core path (K2000-style fully connected integer couplings).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "dcx_internal.h"

namespace dcx {

// Device operands of the dense path. J = jscale * Q with Q a small integer
// matrix, held exactly as f16 in the MMA operand layout [npad][npad].
struct DenseDev {
  int64_t n = 0, npad = 0;
  bool exact = false;    // Q exactly representable in int8 (|q| <= 127)
  float jscale = 1.0f;    // J = jscale * Q (the f32 epilogue's factor)
  double jscale_d = 1.0;  // the same scale in double (energy scale: exact for non-dyadic scales)
  void* q16 = nullptr;   // f16 Q [npad][npad]
  void* q8 = nullptr;    // int8 Q [npad][npad] (energy GEMM)
  void* q8e = nullptr;   // e4m3 Q [npad][npad] (f8 products; exact when |q| <= 16)
  bool f8ok = false;     // Q exact in e4m3
  bool f8 = false;       // this run multiplies e4m3 deltas (iterations >= 1)
  void* dsc = nullptr;   // f8: per-replica descale of the last written delta [Rpad] (between launches)
  // per-run buffers
  int R = 0, Rpad = 0;
  int nc = 1;  // CTAs per MMA (2: cta_group::2 pairs)
  int tn = 128, tiles_n = 0;
  bool ad = false;         // ADOCH (economy window) kernel
  void* xm[2] = {nullptr, nullptr};  // f32 master states [Rpad][npad]
  void* xh[2] = {nullptr, nullptr};  // f16 MMA operand A [Rpad][npad]: DOCH the delta Dh, ADOCH x / lambda_r
  void* s8[2] = {nullptr, nullptr};  // int8 energy GEMM operand A [Rpad][npad]: DOCH dS, ADOCH sign(x)
  int8_t* best8 = nullptr;           // [Rpad][npad]
  int8_t* sgnl = nullptr;            // sign(x_{p-1}) at a launch end [Rpad][npad]
  void* xhat = nullptr;              // DOCH: xhat / lambda [Rpad][npad] f32 (between launches)
  void* d1g = nullptr;               // DOCH: D1 = Q xhat / lambda [Rpad][npad] f32 (between launches)
  void* d2g = nullptr;               // DOCH: D2 = Q sign(x) [Rpad][npad] s32 (between launches)
  double* part = nullptr;            // [tiles_n][Rpad][4]
  void* sync = nullptr;              // grid barrier words
  void* tmaps = nullptr;             // host-side CUtensorMap storage (3 maps)
  int chunk_hint = 0;
  void* dbg = nullptr;                // phase timestamps (DCX_DENSE_TRACE)
  void* scratch = nullptr;            // f64 upload staging (grow-only)
  size_t scratch_bytes = 0;
  void release();
  void release_run();
};

void dense_upload(DenseDev& d, int64_t n, const double* A, cudaStream_t s);
// J = scale * q with q int8 (classified on the host; q in pinned memory)
void dense_upload_int8(DenseDev& d, int64_t n, const int8_t* q_pinned, double scale, cudaStream_t s);
void dense_begin(DenseDev& d, MultiPass& m, cudaStream_t s);
void dense_step(DenseDev& d, MultiPass& m, int chunk, cudaStream_t s);
void dense_finish(DenseDev& d, MultiPass& m, cudaStream_t s);
void dense_profile(DenseDev& d, MultiPass& m, cudaEvent_t a, cudaEvent_t b, cudaStream_t s);
int dense_iters_per_profile_launch();

}  // namespace dcx
