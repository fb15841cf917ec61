// Procedural couplings J_ij = sin(i*j + seed) (i != j), generated on the fly.
//
// Replaces ProceduralCoupling (dc/coupling.py:209-290, formula "sin_product"
// :293-294) and its blocked product (dc/matvec.py:117-155): the reference
// materialises b x b tiles with np.sin and multiplies them with BLAS; here
// every warp generates its row of J in registers and never stores it, so the
// product is bound by the FMA pipe, not by memory.
//
// Generation. theta = i*j + seed is an exact integer (|theta| < 2^63; the
// reference's float64 argument is exact while i*j < 2^53). Its angle modulo
// 2 pi is reduced exactly in integer arithmetic: frac(theta / 2 pi) is the low
// 128 bits of theta * floor(2^128 / 2 pi), of which the top 64 bits are kept
// (error < 2^-60 turns), then sin / cos come from sincospi on [-1, 1). Along a
// row, lane l walks j = jb + l, jb + l + 32, ...: consecutive entries of one
// lane differ by the fixed angle 32*i, so after one exact seed per L entries
// the lane rotates (sin, cos) by that angle (4 FMAs per entry). The diagonal
// is forced to zero like ProceduralCoupling.block.
//
// Sums: each lane accumulates its columns in order, then a fixed xor-shuffle
// tree combines the lanes: deterministic for a given n, not the reference's
// tile order (parity by tolerance, as for every real-valued coupling).
#include <algorithm>

#include "dcx_internal.h"
#include "dcx_rows.cuh"

namespace dcx {

namespace {

// floor(2^128 / (2 pi)) as two 64-bit halves
constexpr unsigned long long INV2PI_HI = 0x28BE60DB9391054AULL;
constexpr unsigned long long INV2PI_LO = 0x7F09D5F47D4D3770ULL;

// theta mod 2 pi as a signed 64-bit fraction of a turn: angle = q * 2 pi / 2^64
__device__ __forceinline__ long long turns_q64(long long theta) {
  const unsigned long long a = (unsigned long long)(theta < 0 ? -theta : theta);
  const unsigned long long q = a * INV2PI_HI + __umul64hi(a, INV2PI_LO);
  const long long s = (long long)q;
  return theta < 0 ? -s : s;
}

// sin / cos of the angle q * 2 pi / 2^64 (= pi * q / 2^63)
__device__ __forceinline__ void sincos_turns(long long q, double& s, double& c) {
  const double hi = double(q);
  const double lo = double(q - (long long)hi);  // exact remainder of the rounding to 53 bits
  sincospi(hi * 0x1p-63, &s, &c);
  const double d = lo * (3.141592653589793 * 0x1p-63);  // sin(a + d) = s + d c, cos(a + d) = c - d s
  const double s2 = fma(d, c, s);
  c = fma(-d, s, c);
  s = s2;
}
__device__ __forceinline__ void sincos_turns(long long q, float& s, float& c) {
  sincospif(float(q) * 0x1p-63f, &s, &c);
}

template <typename T>
struct ProcL;
template <> struct ProcL<double> { static constexpr int value = 16; };
template <> struct ProcL<float> { static constexpr int value = 16; };

// Row i of J times RC vectors: lane partial sums of (J x)_i and (J sign x)_i.
// gather(j, k) returns the k-th vector's entry j.
template <typename T, int RC, bool ES, typename Gather>
__device__ __forceinline__ void proc_row(int64_t i, int64_t n, long long seed, int lane, Gather gather, T (&acc)[RC],
                                         T (&es)[RC]) {
  constexpr int L = ProcL<T>::value;
#pragma unroll
  for (int k = 0; k < RC; ++k) acc[k] = es[k] = T(0);
  T sd, cd;  // rotation by 32 * i
  sincos_turns(turns_q64(32ll * i), sd, cd);
  for (int64_t jb = 0; jb < n; jb += 32 * L) {
    const int64_t j0 = jb + lane;
    T s, c;
    sincos_turns(turns_q64((long long)(i * j0) + seed), s, c);
#pragma unroll 4
    for (int t = 0; t < L; ++t) {
      const int64_t j = j0 + 32 * t;
      if (j < n) {
        const T v = j == i ? T(0) : s;
#pragma unroll
        for (int k = 0; k < RC; ++k) {
          const T xj = gather(j, k);
          acc[k] = fma(v, xj, acc[k]);
          if constexpr (ES) es[k] += xj >= T(0) ? v : -v;
        }
      }
      const T s2 = fma(s, cd, c * sd);
      c = fma(c, cd, -(s * sd));
      s = s2;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int k = 0; k < RC; ++k) {
      acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
      if constexpr (ES) es[k] += __shfl_xor_sync(0xffffffffu, es[k], off);
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Fused DOCH / ADOCH pass over a procedural coupling. One warp per row
// (grid-stride), blockIdx.y = a chunk of RC replicas; the row products feed
// the shared row epilogue (dcx_csr.cu). One partial slot per block.
template <typename T, int MODE, int RC>
__global__ void __launch_bounds__(256) pass_proc(PassArgs a) {
  if (!a.g->live) return;
  const int p = a.g->p;
  if (MODE == MODE_ADOCH_Y && p == 0) return;
  const int R = a.cfg.R;
  const int r0 = blockIdx.y * RC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  RowCtl<T> c[RC];
  bool any = false;
#pragma unroll
  for (int k = 0; k < RC; ++k) {
    const int r = min(r0 + k, R - 1);
    c[k] = row_ctl<T>(a.ctl[r], p);
    if (r0 + k >= R) {  // padding lanes of the last chunk
      c[k].running = false;
      c[k].pend = -2;
    }
    any |= c[k].running || (MODE == MODE_DOCH && c[k].pend == p - 1 && p > 0);
  }
  const int64_t n = a.cfg.n;
  const T* xc = reinterpret_cast<const T*>(a.gx[p & 1]);
  const T* xp = reinterpret_cast<const T*>(a.gx[(p + 1) & 1]);
  RowOut<T, MODE> o[RC];
  if (any) {
    auto gather = [&](int64_t j, int k) -> T {
      const int r = min(r0 + k, R - 1);
      if constexpr (MODE == MODE_ADOCH_Y) return extrap(xc[j * R + r], xp[j * R + r], c[k].cm);
      else return xc[j * R + r];
    };
    for (int64_t i = int64_t(blockIdx.x) * 8 + warp; i < n; i += int64_t(gridDim.x) * 8) {
      T acc[RC], es[RC];
      proc_row<T, RC, MODE != MODE_ADOCH_Y>(i, n, a.proc_seed, lane, gather, acc, es);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < RC; ++k) {
          const int64_t idx = i * R + r0 + k;
          if (c[k].running) row_epilogue<T, MODE>(a, c[k], p, idx, acc[k], double(es[k]), o[k]);
          else if (MODE == MODE_DOCH && c[k].pend == p - 1 && p > 0)  // stopped: only the pending copy
            a.best[idx] = reinterpret_cast<const T*>(a.x[(p + 1) & 1])[idx] >= T(0) ? 1 : -1;
        }
      }
    }
  }
  // block partials: the 8 warp sums (lane 0) in warp order
  __shared__ double red[8][RC][NQ];
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < RC; ++k) {
      red[warp][k][Q_S4] = o[k].s4;
      red[warp][k][Q_SXAX] = o[k].sxax;
      red[warp][k][Q_ES] = o[k].es;
      red[warp][k][Q_STEP] = o[k].step;
      red[warp][k][Q_SY4] = o[k].sy4;
      red[warp][k][Q_SYAY] = o[k].syay;
    }
  __syncthreads();
  if (threadIdx.x < RC && r0 + int(threadIdx.x) < R) {
    const int k = threadIdx.x;
    RowOut<T, MODE> b;
    b.s4 = red[0][k][Q_S4]; b.sxax = red[0][k][Q_SXAX]; b.es = red[0][k][Q_ES];
    b.step = red[0][k][Q_STEP]; b.sy4 = red[0][k][Q_SY4]; b.syay = red[0][k][Q_SYAY];
    for (int w = 1; w < 8; ++w) {
      b.s4 += red[w][k][Q_S4]; b.sxax += red[w][k][Q_SXAX]; b.es += red[w][k][Q_ES];
      b.step = fmax(b.step, red[w][k][Q_STEP]); b.sy4 += red[w][k][Q_SY4]; b.syay += red[w][k][Q_SYAY];
    }
    write_partials<T, MODE>(a, r0 + k, (int)blockIdx.x, b);
  }
}

// Operator seam: jv = J v and es_rows = J sign(v) (f64) for R vectors, [n][R].
template <typename T, int RC>
__global__ void __launch_bounds__(256) proc_apply(int64_t n, long long seed, const T* v, int R, T* jv,
                                                  double* es_rows) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = blockIdx.y * RC;
  auto gather = [&](int64_t j, int k) -> T { return v[j * R + min(r0 + k, R - 1)]; };
  for (int64_t i = int64_t(blockIdx.x) * 8 + warp; i < n; i += int64_t(gridDim.x) * 8) {
    T acc[RC], es[RC];
    proc_row<T, RC, true>(i, n, seed, lane, gather, acc, es);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < RC; ++k)
        if (r0 + k < R) {
          jv[i * R + r0 + k] = acc[k];
          if (es_rows) es_rows[i * R + r0 + k] = double(es[k]);
        }
  }
}

// Per-row sum, sum of squares and sum of |J_ij| (f64): offdiag_moments and
// abs_row_sums (dc/coupling.py:248-268) without materialising a tile.
__global__ void __launch_bounds__(256) proc_row_stats(int64_t n, long long seed, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = int64_t(blockIdx.x) * 8 + warp; i < n; i += int64_t(gridDim.x) * 8) {
    double s1 = 0, s2 = 0, s3 = 0;
    constexpr int L = ProcL<double>::value;
    double sd, cd;
    sincos_turns(turns_q64(32ll * i), sd, cd);
    for (int64_t jb = 0; jb < n; jb += 32 * L) {
      const int64_t j0 = jb + lane;
      double s, c;
      sincos_turns(turns_q64((long long)(i * j0) + seed), s, c);
      for (int t = 0; t < L; ++t) {
        const int64_t j = j0 + 32 * t;
        if (j < n && j != i) {
          s1 += s;
          s2 = fma(s, s, s2);
          s3 += fabs(s);
        }
        const double t2 = fma(s, cd, c * sd);
        c = fma(c, cd, -(s * sd));
        s = t2;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
      s3 += __shfl_xor_sync(0xffffffffu, s3, off);
    }
    if (lane == 0) {
      out[i * 3 + 0] = s1;
      out[i * 3 + 1] = s2;
      out[i * 3 + 2] = s3;
    }
  }
}

static int proc_rows_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, 148 * 8));
}

int proc_replica_chunk(int R) { return R == 1 ? 1 : 4; }

template <typename T, int MODE>
static void launch_proc_mode(const PassArgs& a, int grid, cudaStream_t s) {
  const int R = a.cfg.R;
  if (R == 1) pass_proc<T, MODE, 1><<<dim3(grid, 1), 256, 0, s>>>(a);
  else pass_proc<T, MODE, 4><<<dim3(grid, (R + 3) / 4), 256, 0, s>>>(a);
}

template <typename T>
void launch_proc_pass(int mode, const PassArgs& a, int grid, cudaStream_t s) {
  if (mode == MODE_DOCH) launch_proc_mode<T, MODE_DOCH>(a, grid, s);
  else if (mode == MODE_ADOCH_X) launch_proc_mode<T, MODE_ADOCH_X>(a, grid, s);
  else launch_proc_mode<T, MODE_ADOCH_Y>(a, grid, s);
}
template void launch_proc_pass<double>(int, const PassArgs&, int, cudaStream_t);
template void launch_proc_pass<float>(int, const PassArgs&, int, cudaStream_t);

int proc_pass_grid(int64_t n) { return proc_rows_grid(n); }

template <typename T>
void launch_proc_apply(int64_t n, long long seed, const T* v, int R, T* jv, double* es_rows, cudaStream_t s) {
  const int grid = proc_rows_grid(n);
  if (R == 1) proc_apply<T, 1><<<dim3(grid, 1), 256, 0, s>>>(n, seed, v, R, jv, es_rows);
  else proc_apply<T, 4><<<dim3(grid, (R + 3) / 4), 256, 0, s>>>(n, seed, v, R, jv, es_rows);
}
template void launch_proc_apply<double>(int64_t, long long, const double*, int, double*, double*, cudaStream_t);
template void launch_proc_apply<float>(int64_t, long long, const float*, int, float*, double*, cudaStream_t);

void launch_proc_row_stats(int64_t n, long long seed, double* out, cudaStream_t s) {
  proc_row_stats<<<proc_rows_grid(n), 256, 0, s>>>(n, seed, out);
}

}  // namespace dcx
