// Persistent small-n path: one CTA per replica keeps the whole CSR pattern,
// its values and every state vector in shared memory and runs the complete
// DOCH / ADOCH loop (dc/solvers/doch.py:199-232 / :294-342) on chip, with the
// control logic of dcx_device.cuh executed by thread 0 between block barriers.
// For the G1-shape config (n = 800, 38,352 nnz) the pattern is 77 KB of uint16
// column indices; there is no HBM traffic per iteration except the history
// ring and best-spin copies.
#include <cstdio>
#include <cstdlib>

#include "dcx_internal.h"

namespace dcx {

constexpr int SMALL_THREADS = 512;
constexpr int SMALL_WARPS = SMALL_THREADS / 32;

struct SmallArgs {
  PassArgs a;
  const uint16_t* col16;
  int V;
  int p_end;  // stop after executing pass p_end - 1 (chunk end)
  int col_is16;
  int ell;    // columns held as 32-row sliced ELL (V == 1): one conflict-free load per 32 rows and entry
  int pow2;   // uniform values, power-of-two scale: sum x_j, multiply once (bit-identical to sum v x_j)
  int trace;  // DCX_SMALL_TRACE: phase stamps of block 0
};

__host__ __device__ constexpr int val_bytes(int vk) {
  return vk == VK_UNIFORM ? 0 : vk == VK_I8 ? 1 : vk == VK_I16 ? 2 : vk == VK_F32 ? 4 : 8;
}

// Shared-memory carve-up (16-byte aligned regions), identical on host and device.
struct SmemLayout {
  uint32_t x0, x1, ax0, ax1, ay, rp, col, val, sofs, total;
};
__host__ __device__ inline uint32_t align16(uint64_t v) { return uint32_t((v + 15) & ~uint64_t(15)); }
__host__ __device__ inline SmemLayout small_layout(int n, uint32_t nnz, int tb, bool adoch, bool exact, bool col16,
                                                   int vb, uint32_t ell = 0) {
  SmemLayout L;
  uint32_t o = 0;
  const uint32_t vec = align16(uint64_t(n) * tb);
  L.x0 = o; o += vec;
  L.x1 = o; o += vec;
  L.ax0 = o; if (adoch) o += vec;
  L.ax1 = o; if (adoch) o += vec;
  L.ay = o; if (adoch && exact) o += vec;
  L.rp = o; o += align16(uint64_t(n + 1) * 4);
  L.col = o; o += ell ? align16(uint64_t(ell) * 2) : align16(uint64_t(nnz) * (col16 ? 2 : 4));
  L.val = o; o += align16(uint64_t(nnz) * vb);
  L.sofs = o; if (ell) o += align16(uint64_t((n + 31) / 32 + 1) * 4);
  L.total = o;
  return L;
}

// fixed-order block reduction of NQ values (sum, except the step max)
__device__ __forceinline__ void block_reduce(double* v, double (*sh)[NQ], double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = (q == Q_STEP) ? warp_max(v[q]) : warp_sum(v[q]);
  if (lane == 0)
    for (int q = 0; q < NQ; ++q) sh[w][q] = v[q];
  __syncthreads();
  if (threadIdx.x < NQ) {  // one thread per quantity, warps summed in order
    const int q = threadIdx.x;
    double acc = sh[0][q];
    for (int i = 1; i < SMALL_WARPS; ++i) acc = (q == Q_STEP) ? fmax(acc, sh[i][q]) : acc + sh[i][q];
    out[q] = acc;
  }
  __syncthreads();
}

// DCX_SMALL_TRACE: phase stamps of block 0, thread 0, iterations 10..73 (clock64)
__device__ unsigned long long g_small_trace[64 * 4];

template <typename T, int VK>
__global__ void __launch_bounds__(SMALL_THREADS) small_kernel(SmallArgs s) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PassArgs& a = s.a;
  const int r = blockIdx.x;
  const int R = a.cfg.R;
  const int n = (int)a.cfg.n;
  const bool adoch = a.cfg.solver == DCX_SOLVER_ADOCH;
  const bool exact = a.cfg.window_mode == DCX_WINDOW_EXACT;
  // ---- carve shared memory
  const uint32_t NNZ = __ldg(a.rp + n);
  constexpr int VB = val_bytes(VK);
  const SmemLayout L = small_layout(n, NNZ, sizeof(T), adoch, exact, s.col_is16, VB, uint32_t(s.ell));
  T* xb0 = reinterpret_cast<T*>(smem + L.x0);
  T* xb1 = reinterpret_cast<T*>(smem + L.x1);
  T* axb0 = reinterpret_cast<T*>(smem + L.ax0);
  T* axb1 = reinterpret_cast<T*>(smem + L.ax1);
  T* ayb = reinterpret_cast<T*>(smem + L.ay);
  uint32_t* rp = reinterpret_cast<uint32_t*>(smem + L.rp);
  void* colp = smem + L.col;
  void* valp = smem + L.val;
  __shared__ double red[SMALL_WARPS][NQ];
  __shared__ double tot[NQ];
  __shared__ RepCtl c;
  __shared__ int flag_stop;

  for (int i = threadIdx.x; i <= n; i += blockDim.x) rp[i] = a.rp[i];
  uint32_t* sofs = reinterpret_cast<uint32_t*>(smem + L.sofs);
  if (s.ell) {
    // 32-row slices: entry k of row i at sofs[i / 32] + 32 k + i % 32
    __syncthreads();
    const int ns = (n + 31) / 32;
    if (threadIdx.x == 0) {
      uint32_t o = 0;
      for (int sl = 0; sl < ns; ++sl) {
        uint32_t mx = 0;
        for (int i = sl * 32; i < min(n, sl * 32 + 32); ++i) mx = max(mx, rp[i + 1] - rp[i]);
        sofs[sl] = o;
        o += 32 * mx;
      }
      sofs[ns] = o;
    }
    __syncthreads();
    uint16_t* ell = reinterpret_cast<uint16_t*>(colp);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t base = sofs[i >> 5] + (i & 31), lo = rp[i], len = rp[i + 1] - lo;
      for (uint32_t k = 0; k < len; ++k) ell[base + 32 * k] = s.col16[lo + k];
    }
  } else if (s.col_is16) {
    uint16_t* c16 = reinterpret_cast<uint16_t*>(colp);
    for (uint32_t e = threadIdx.x; e < NNZ; e += blockDim.x) c16[e] = s.col16[e];
  } else {
    int32_t* c32 = reinterpret_cast<int32_t*>(colp);
    for (uint32_t e = threadIdx.x; e < NNZ; e += blockDim.x) c32[e] = a.col[e];
  }
  if (VB) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(a.val);
    unsigned char* dst = reinterpret_cast<unsigned char*>(valp);
    for (uint32_t b = threadIdx.x; b < NNZ * VB; b += blockDim.x) dst[b] = src[b];
  }
  if (threadIdx.x == 0) c = a.ctl[r];
  __syncthreads();
  int p = a.g->p;
  if (c.status != DCX_STOP_RUNNING) return;
  // ---- load state (layout [n][R] in global)
  {
    const T* gx0 = reinterpret_cast<const T*>(a.x[p & 1]);
    const T* gx1 = reinterpret_cast<const T*>(a.x[(p + 1) & 1]);
    T* xc = (p & 1) ? xb1 : xb0;
    T* xo = (p & 1) ? xb0 : xb1;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      xc[i] = gx0[(int64_t)i * R + r];
      xo[i] = gx1[(int64_t)i * R + r];
    }
    if (adoch) {
      const T* ga0 = reinterpret_cast<const T*>(a.ax[p & 1]);
      const T* ga1 = reinterpret_cast<const T*>(a.ax[(p + 1) & 1]);
      T* ac = (p & 1) ? axb1 : axb0;
      T* ao = (p & 1) ? axb0 : axb1;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        ac[i] = ga0[(int64_t)i * R + r];
        ao[i] = ga1[(int64_t)i * R + r];
      }
    }
  }
  __syncthreads();
  const int V = s.V;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int rpw = 32 / V;
  const T scale = T(a.scale);
  auto colat = [&](uint32_t e) -> int {
    return s.col_is16 ? int(reinterpret_cast<const uint16_t*>(colp)[e]) : reinterpret_cast<const int32_t*>(colp)[e];
  };
  // row product over smem; mode 0: v = x (returns es too), mode 1: v = y
  auto rowdot = [&](int i, const T* xv, const T* xpv, T cmv, bool ymode, T& acc,
                    typename EsAcc<VK>::type& es) {
    acc = T(0);
    es = 0;
    if (s.ell) {  // V == 1: lane = row % 32, column order as in the CSR row
      if (i < n) {
        const uint32_t lo = rp[i], len = rp[i + 1] - lo;
        const uint16_t* ell = reinterpret_cast<const uint16_t*>(colp) + sofs[i >> 5] + (i & 31);
        if (VK == VK_UNIFORM && s.pow2 && !ymode) {
          // unit pattern, power-of-two weight: sum x_j in column order, scale once
          // (bit-identical to sum v x_j); spin sum = len - 2 #negative (x is never -0.0)
          uint32_t neg = 0;
          for (uint32_t k = 0; k < len; ++k) {
            const T xj = xv[ell[32 * k]];
            acc = add_rn(acc, xj);
            neg += negbit(xj);
          }
          acc = mul_rn(acc, scale);
          es = typename EsAcc<VK>::type(int(len) - 2 * int(neg));
        } else {
          for (uint32_t k = 0; k < len; ++k) {
            const int j = ell[32 * k];
            int q;
            const T v = load_entry<VK, false, T>(valp, lo + k, scale, q);
            if (ymode) {
              acc = madd(acc, v, extrap(xv[j], xpv[j], cmv));
            } else {
              const T xj = xv[j];
              acc = madd(acc, v, xj);
              es += es_term<VK, T>(q, v, xj);
            }
          }
        }
      }
      return;
    }
    if (i < n) {
      const uint32_t lo = rp[i], hi = rp[i + 1];
      for (uint32_t e = lo + sub; e < hi; e += V) {
        const int j = colat(e);
        int q;
        const T v = load_entry<VK, false, T>(valp, e, scale, q);
        if (ymode) {
          acc = madd(acc, v, extrap(xv[j], xpv[j], cmv));
        } else {
          const T xj = xv[j];
          acc = madd(acc, v, xj);
          es += es_term<VK, T>(q, v, xj);
        }
      }
    }
    for (int off = V >> 1; off > 0; off >>= 1) {
      acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
      es += __shfl_xor_sync(0xffffffffu, es, off);
    }
  };
  const int nwarps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5;
  T* states = reinterpret_cast<T*>(a.states);

  while (p < s.p_end) {
    const bool trc = s.trace && blockIdx.x == 0 && threadIdx.x == 0 && p >= 10 && p < 74;
    if (trc) g_small_trace[(p - 10) * 4 + 0] = clock64();
    T* xc = (p & 1) ? xb1 : xb0;  // x_p
    T* xo = (p & 1) ? xb0 : xb1;  // DOCH: x_{p-1} -> x_{p+1}; ADOCH: x_{p-1}
    T* ac = (p & 1) ? axb1 : axb0;
    T* ao = (p & 1) ? axb0 : axb1;
    const T alpha = T(c.alpha), beta = T(c.beta), cm = T(c.cm[p & 1]);
    double v[NQ] = {0, 0, 0, 0, 0, 0};
    // ---- pass over x_p
    auto row_done = [&](int i, T acc, typename EsAcc<VK>::type es) {
      if (i < n && sub == 0) {
        const T xi = xc[i];
        const T ax = shifted(acc, alpha, xi);
        double x2 = double(mul_rn(xi, xi));
        v[Q_S4] += x2 * x2;
        v[Q_SXAX] += double(xi) * double(ax);
        v[Q_ES] += xi >= T(0) ? double(es) : -double(es);
        if (!adoch) {
          if (p > 0 && c.pend == p - 1) a.best[(int64_t)i * R + r] = xo[i] >= T(0) ? 1 : -1;
          const T xn = tmap_pass(ax, beta, inv_beta(beta));
          v[Q_STEP] = fmax(v[Q_STEP], double(fabs(xn - xi)));
          xo[i] = xn;  // own row only: no other thread reads xo in this phase
          if (states && p < a.cfg.max_iters) states[((int64_t)(p + 1) * n + i) * R + r] = xn;
        } else {
          ac[i] = ax;
          if (p > 0 && !exact) {
            const T yi = extrap(xi, xo[i], cm);
            const T ayi = extrap(ax, ao[i], cm);
            double y2 = double(mul_rn(yi, yi));
            v[Q_SY4] += y2 * y2;
            v[Q_SYAY] += double(yi) * double(ayi);
          }
        }
      }
    };
    if (VK == VK_UNIFORM && s.pow2 && s.ell) {
      // sliced ELL, unit weights: each thread owns rows t and t + blockDim (same
      // lane of two slices) and walks both sums together, two independent
      // column-order chains in flight
      const int nb = blockDim.x;
      const uint16_t* ell = reinterpret_cast<const uint16_t*>(colp);
      for (int i0 = threadIdx.x; i0 < n; i0 += 2 * nb) {
        const int i1 = i0 + nb;
        const uint32_t len0 = rp[i0 + 1] - rp[i0];
        const uint32_t len1 = i1 < n ? rp[i1 + 1] - rp[i1] : 0u;
        const uint16_t* e0 = ell + sofs[i0 >> 5] + (i0 & 31);
        const uint16_t* e1 = ell + (i1 < n ? sofs[i1 >> 5] + (i1 & 31) : 0);
        T a0 = T(0), a1 = T(0);
        uint32_t n0 = 0, n1 = 0;
        const uint32_t m = max(len0, len1);
        for (uint32_t k = 0; k < m; ++k) {
          if (k < len0) {
            const T xj = xc[e0[32 * k]];
            a0 = add_rn(a0, xj);
            n0 += negbit(xj);
          }
          if (k < len1) {
            const T xj = xc[e1[32 * k]];
            a1 = add_rn(a1, xj);
            n1 += negbit(xj);
          }
        }
        row_done(i0, mul_rn(a0, scale), typename EsAcc<VK>::type(int(len0) - 2 * int(n0)));
        if (i1 < n) row_done(i1, mul_rn(a1, scale), typename EsAcc<VK>::type(int(len1) - 2 * int(n1)));
      }
    } else {
      for (int base = w * rpw; base < n; base += nwarps * rpw) {
        const int i = base + lane / V;
        T acc;
        typename EsAcc<VK>::type es;
        rowdot(i, xc, nullptr, T(0), false, acc, es);
        row_done(i, acc, es);
      }
    }
    if (trc) g_small_trace[(p - 10) * 4 + 1] = clock64();
    block_reduce(v, red, tot);
    if (trc) g_small_trace[(p - 10) * 4 + 2] = clock64();
    if (threadIdx.x == 0) {
      const double now = double(globaltimer() - a.g->t0) * 1e-9;
      double t2[NQ];
      for (int q = 0; q < NQ; ++q) t2[q] = tot[q];
      bool stopped = control_after_pass(c, a.cfg, r, t2, p, now);
      if (!adoch) c.step = t2[Q_STEP];
      else if (!stopped && !exact) adoch_decide(c, a.cfg, r, t2, p);
      flag_stop = stopped ? 1 : 0;
    }
    __syncthreads();
    if (adoch) {
      if (!flag_stop && exact) {
        // ---- exact window: (J + aI) y with y formed on the fly
        for (int q = 0; q < NQ; ++q) v[q] = 0.0;
        if (p > 0) {
          for (int base = w * rpw; base < n; base += nwarps * rpw) {
            const int i = base + lane / V;
            T acc;
            typename EsAcc<VK>::type es;
            rowdot(i, xc, xo, cm, true, acc, es);
            if (i < n && sub == 0) {
              const T yi = extrap(xc[i], xo[i], cm);
              const T ayi = shifted(acc, alpha, yi);
              ayb[i] = ayi;
              double y2 = double(mul_rn(yi, yi));
              v[Q_SY4] += y2 * y2;
              v[Q_SYAY] += double(yi) * double(ayi);
            }
          }
        }
        block_reduce(v, red, tot);
        if (threadIdx.x == 0) {
          double t2[NQ];
          for (int q = 0; q < NQ; ++q) t2[q] = tot[q];
          adoch_decide(c, a.cfg, r, t2, p);
        }
        __syncthreads();
      }
      // ---- finalize: x_{p+1} = cbrt(Av / beta) into the x_{p-1} slot
      const bool acc_y = p > 0 && c.accept;
      double st = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const T xi = xc[i];
        if (c.pend == p) a.best[(int64_t)i * R + r] = xi >= T(0) ? 1 : -1;
        if (flag_stop) continue;
        const T av = acc_y ? (exact ? ayb[i] : extrap(ac[i], ao[i], cm)) : ac[i];
        const T xn = tmap_pass(av, beta, inv_beta(beta));
        st = fmax(st, double(fabs(xn - xi)));
        xo[i] = xn;
        if (states && p < a.cfg.max_iters) states[((int64_t)(p + 1) * n + i) * R + r] = xn;
      }
      double vv[NQ] = {0, 0, 0, st, 0, 0};
      block_reduce(vv, red, tot);
      if (threadIdx.x == 0) c.step = tot[Q_STEP];
      __syncthreads();
    } else if (flag_stop) {
      // DOCH: the pending copy for x_p happens here (no further pass)
      if (c.pend == p)
        for (int i = threadIdx.x; i < n; i += blockDim.x) a.best[(int64_t)i * R + r] = xc[i] >= T(0) ? 1 : -1;
    }
    if (trc) g_small_trace[(p - 10) * 4 + 3] = clock64();
    ++p;
    if (flag_stop) break;
  }
  // ---- write back state and control
  {
    T* gx0 = reinterpret_cast<T*>(a.x[0]);
    T* gx1 = reinterpret_cast<T*>(a.x[1]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      gx0[(int64_t)i * R + r] = xb0[i];
      gx1[(int64_t)i * R + r] = xb1[i];
    }
    if (adoch) {
      T* ga0 = reinterpret_cast<T*>(a.ax[0]);
      T* ga1 = reinterpret_cast<T*>(a.ax[1]);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        ga0[(int64_t)i * R + r] = axb0[i];
        ga1[(int64_t)i * R + r] = axb1[i];
      }
    }
  }
  if (threadIdx.x == 0) {
    if (flag_stop) atomicSub(&a.g->running, 1);
    a.ctl[r] = c;
  }
}

SmallPlan plan_small(const CsrDev& J, int solver, int window_mode, bool f64) {
  SmallPlan sp;
  const bool adoch = solver == DCX_SOLVER_ADOCH;
  const bool ell = J.V == 1 && J.col16 != nullptr && J.ell > 0 && J.ell < (1ll << 31);
  const SmemLayout L = small_layout((int)J.n, (uint32_t)J.nnz, f64 ? 8 : 4, adoch,
                                    window_mode == DCX_WINDOW_EXACT, J.col16 != nullptr, val_bytes(J.vk),
                                    ell ? uint32_t(J.ell) : 0u);
  sp.ell = ell;
  sp.smem = L.total;
  sp.threads = SMALL_THREADS;
  sp.fits = L.total <= 200 * 1024 && J.n <= (1 << 20) && J.nnz < (1ll << 31);
  if (J.vk == VK_PROC) sp.fits = false;  // no stored pattern: the procedural pass generates J
  return sp;
}

template <typename T, int VK>
static void launch_small_t(const SmallArgs& s, const SmallPlan& sp, cudaStream_t st) {
  auto k = small_kernel<T, VK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.smem);
  k<<<s.a.cfg.R, SMALL_THREADS, sp.smem, st>>>(s);
}

void launch_small(const MultiPass& m, const CsrDev& J, const SmallPlan& sp, int p_end, cudaStream_t st) {
  SmallArgs s;
  s.a = m.args;
  s.col16 = J.col16;
  s.col_is16 = J.col16 != nullptr;
  s.V = J.V;
  s.p_end = p_end;
  s.ell = sp.ell ? int(J.ell) : 0;
  s.pow2 = J.pow2_uniform ? 1 : 0;
  s.trace = std::getenv("DCX_SMALL_TRACE") != nullptr;
  if (m.f64) {
    switch (J.vk) {
      case VK_UNIFORM: launch_small_t<double, VK_UNIFORM>(s, sp, st); break;
      case VK_I8: launch_small_t<double, VK_I8>(s, sp, st); break;
      case VK_I16: launch_small_t<double, VK_I16>(s, sp, st); break;
      case VK_F32: launch_small_t<double, VK_F32>(s, sp, st); break;
      default: launch_small_t<double, VK_F64>(s, sp, st); break;
    }
  } else {
    switch (J.vk) {
      case VK_UNIFORM: launch_small_t<float, VK_UNIFORM>(s, sp, st); break;
      case VK_I8: launch_small_t<float, VK_I8>(s, sp, st); break;
      case VK_I16: launch_small_t<float, VK_I16>(s, sp, st); break;
      case VK_F32: launch_small_t<float, VK_F32>(s, sp, st); break;
      default: launch_small_t<float, VK_F64>(s, sp, st); break;
    }
  }
  if (s.trace) {
    unsigned long long t[64 * 4];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(t, g_small_trace, sizeof(t));
    double ph[3] = {0, 0, 0};
    int cnt = 0;
    for (int k = 0; k < 63; ++k) {
      if (!t[k * 4] || !t[k * 4 + 3]) continue;
      ph[0] += double(t[k * 4 + 1] - t[k * 4]);
      ph[1] += double(t[k * 4 + 2] - t[k * 4 + 1]);
      ph[2] += double(t[k * 4 + 3] - t[k * 4 + 2]);
      ++cnt;
    }
    if (cnt)
      std::fprintf(stderr, "[dcx small trace] cycles per iteration: pass %.0f | reduce %.0f | control+rest %.0f\n",
                   ph[0] / cnt, ph[1] / cnt, ph[2] / cnt);
  }
}

}  // namespace dcx
