// Device power iteration: dc/spectral.py:60-111 (_power_core) as one
// persistent cooperative kernel, for derive_params' lambda_max(-J)
// (dc/spectral.py:143-162). The reference runs one Python-level iteration per
// product (23,578 products at K2000, 8.1 s on the host); here every iteration
// stays on the device: w = M v over the CSR rows (warp per row, f64, fixed
// lane-tree order), then fixed-order grid reductions of |w|^2, v.w and
// |w - ray v|^2, and the reference's decisions (convergence, stall counter,
// one seeded restart), replicated identically in every CTA.
#include "dcx_internal.h"

namespace dcx {

struct PowerArgs {
  const uint32_t* rp;
  const int32_t* col;
  const void* val;
  double scale;
  int64_t n;
  int use_shift;
  double shift;
  double tol;
  int64_t max_iters;
  double* v;
  double* w;
  const double* restart;  // normalised seeded restart vector (host numpy, as the reference draws it)
  double* part;           // [grid][2]
  double* part2;          // [grid]
  unsigned* bar;          // [2]: arrival count, generation
  double* out;            // mag, ray, iterations, converged
};

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// fixed-order sum of per-CTA partials (every CTA computes the same value)
__device__ double sum_parts(const double* p, int stride, int count, double* sh) {
  double s = 0.0;
  for (int b = threadIdx.x; b < count; b += blockDim.x) s += __ldcg(p + b * stride);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__device__ double block_sum(double x, double* sh) {
  sh[threadIdx.x] = x;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

template <int VK>
__global__ void __launch_bounds__(256) power_kernel(PowerArgs a) {
  __shared__ double sh[256];
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  const int64_t n = a.n;
  const double scale = a.scale;
  // v = full(n, 1/sqrt(n))
  const double v0 = 1.0 / sqrt(double(n));
  for (int64_t i = tid; i < n; i += nth) a.v[i] = v0;
  grid_barrier(a.bar);
  bool restarted = false;
  double best_resid = INFINITY, mag = 0.0, ray = 0.0;
  int since = 0;
  int64_t k = 0;
  int conv = 0;
  while (k < a.max_iters) {
    // w = M v, partial |w|^2 and v.w
    double ww = 0.0, vw = 0.0;
    for (int64_t i = gw; i < n; i += nw) {
      const uint32_t lo = a.rp[i], hi = a.rp[i + 1];
      double acc = 0.0;
      for (uint32_t e = lo + lane; e < hi; e += 32) {
        int q;
        const double jv = load_entry<VK, true, double>(a.val, e, scale, q);
        acc = __dadd_rn(acc, __dmul_rn(jv, __ldcg(a.v + a.col[e])));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (lane == 0) {
        const double vi = __ldcg(a.v + i);
        const double wi = a.use_shift ? __dsub_rn(__dmul_rn(a.shift, vi), acc) : -acc;
        a.w[i] = wi;
        ww += wi * wi;
        vw += vi * wi;
      }
    }
    ww = block_sum(ww, sh);
    vw = block_sum(vw, sh);
    if (threadIdx.x == 0) {
      a.part[blockIdx.x * 2] = ww;
      a.part[blockIdx.x * 2 + 1] = vw;
    }
    grid_barrier(a.bar);
    mag = sqrt(sum_parts(a.part, 2, gridDim.x, sh));
    if (mag == 0.0) {
      if (restarted) {  // (0, 0, k, False)
        mag = 0.0;
        ray = 0.0;
        break;
      }
      for (int64_t i = tid; i < n; i += nth) a.v[i] = a.restart[i];
      restarted = true;
      ++k;
      grid_barrier(a.bar);
      continue;
    }
    ray = sum_parts(a.part + 1, 2, gridDim.x, sh);
    double r2 = 0.0;
    for (int64_t i = tid; i < n; i += nth) {
      const double d = __ldcg(a.w + i) - ray * __ldcg(a.v + i);
      r2 += d * d;
    }
    r2 = block_sum(r2, sh);
    if (threadIdx.x == 0) a.part2[blockIdx.x] = r2;
    grid_barrier(a.bar);
    const double resid = sqrt(sum_parts(a.part2, 1, gridDim.x, sh)) / mag;
    if (resid <= a.tol) {
      ++k;
      conv = 1;
      break;
    }
    bool restart_now = false;
    if (resid < 0.999 * best_resid) {
      best_resid = resid;
      since = 0;
    } else {
      ++since;
      if (since > 50 && !restarted) {
        restart_now = true;
        restarted = true;
        since = 0;
      }
    }
    if (restart_now) {
      for (int64_t i = tid; i < n; i += nth) a.v[i] = a.restart[i];
    } else {
      for (int64_t i = tid; i < n; i += nth) a.v[i] = __ldcg(a.w + i) / mag;
    }
    ++k;
    grid_barrier(a.bar);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = mag;
    a.out[1] = ray;
    a.out[2] = double(k);
    a.out[3] = double(conv);
  }
}

void launch_power(const CsrDev& J, int use_shift, double shift, double tol, int64_t max_iters, double* v, double* w,
                  const double* restart, double* part, double* part2, unsigned* bar, double* out, int grid,
                  cudaStream_t s) {
  PowerArgs a{J.rp, J.col, J.val, J.scale, J.n, use_shift, shift, tol, max_iters, v, w, restart, part, part2, bar, out};
  void* args[] = {&a};
  const void* fn;
  switch (J.vk) {
    case VK_UNIFORM: fn = reinterpret_cast<const void*>(power_kernel<VK_UNIFORM>); break;
    case VK_I8: fn = reinterpret_cast<const void*>(power_kernel<VK_I8>); break;
    case VK_I16: fn = reinterpret_cast<const void*>(power_kernel<VK_I16>); break;
    case VK_F32: fn = reinterpret_cast<const void*>(power_kernel<VK_F32>); break;
    default: fn = reinterpret_cast<const void*>(power_kernel<VK_F64>); break;
  }
  cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, s);
}

}  // namespace dcx
