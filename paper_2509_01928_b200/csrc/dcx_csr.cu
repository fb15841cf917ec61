// Multi-pass CSR path: one fused SpMV/SpMM + DC-update pass per iteration,
// a per-replica reduce+control kernel, and (ADOCH) an elementwise finalize.
//
// Replaces, per iteration, dc/solvers/doch.py:199-232 (DOCH) / :294-342 (ADOCH)
// with scipy csr_matvec (dc/coupling.py:189-190) as the product. One pass
// reads the CSR stream once and gathers x once; from the same gather it forms
// (J+aI)x, the next iterate, and J*sign(x) for the spin energy (exact integer
// accumulation for integer couplings), plus the H / E / step partials.
#include "dcx_internal.h"

namespace dcx {



// ---------------------------------------------------------------------------
// Row epilogue shared by the R=1 and R>1 kernels. `acc` = (J v)_i in T,
// `es` = (J sign x_p)_i. `xi` = x_p[i]. Everything that is elementwise given
// the row product happens here.
template <typename T, int MODE>
struct RowOut {
  double s4 = 0, sxax = 0, es = 0, step = 0, sy4 = 0, syay = 0;
};

template <typename T, int MODE>
__device__ __forceinline__ void row_epilogue(const PassArgs& a, const RepCtl& c, int p, int64_t idx, T acc,
                                             double esrow, RowOut<T, MODE>& o) {
  const T* xcur = reinterpret_cast<const T*>(a.x[p & 1]);
  T* xnext = reinterpret_cast<T*>(a.x[(p + 1) & 1]);
  const T alpha = T(c.alpha), beta = T(c.beta);
  if constexpr (MODE == MODE_ADOCH_Y) {
    // acc = J y ; y recomputed identically to the gather
    const T* xprev = reinterpret_cast<const T*>(a.x[(p + 1) & 1]);
    const T cm = T(c.cm[p & 1]);
    T yi = extrap(xcur[idx], xprev[idx], cm);
    T ayi = shifted(acc, alpha, yi);
    reinterpret_cast<T*>(a.ay)[idx] = ayi;
    double y2 = double(yi) * double(yi);
    o.sy4 += y2 * y2;
    o.syay += double(yi) * double(ayi);
    return;
  } else {
    const T xi = xcur[idx];
    const T ax = shifted(acc, alpha, xi);
    double x2 = double(mul_rn(xi, xi));
    o.s4 += x2 * x2;
    o.sxax += double(xi) * double(ax);
    o.es += (xi >= T(0) ? esrow : -esrow);
    if constexpr (MODE == MODE_DOCH) {
      // pending best-spin copy of x_{p-1}, still held in the write buffer
      if (c.pend == p - 1 && p > 0) a.best[idx] = xnext[idx] >= T(0) ? 1 : -1;
      if (c.status == DCX_STOP_RUNNING) {
        T xn = tmap(ax, beta);
        xnext[idx] = xn;
        if (a.states) reinterpret_cast<T*>(a.states)[(int64_t)(p + 1) * a.cfg.n * a.cfg.R + idx] = xn;
        o.step = fmax(o.step, double(fabs(xn - xi)));
      }
    } else {  // MODE_ADOCH_X: store Ax_p, H(y_p) partials for the economy window test
      T* axb = reinterpret_cast<T*>(a.ax[p & 1]);
      axb[idx] = ax;
      if (p > 0 && a.cfg.window_mode == DCX_WINDOW_ECONOMY) {
        const T* xprev = reinterpret_cast<const T*>(a.x[(p + 1) & 1]);
        const T* axprev = reinterpret_cast<const T*>(a.ax[(p + 1) & 1]);
        const T cm = T(c.cm[p & 1]);
        T yi = extrap(xi, xprev[idx], cm);
        T ayi = extrap(ax, axprev[idx], cm);
        double y2 = double(mul_rn(yi, yi));
        o.sy4 += y2 * y2;
        o.syay += double(yi) * double(ayi);
      }
    }
  }
}

template <typename T, int MODE>
__device__ __forceinline__ void write_partials(const PassArgs& a, int r, int slot, const RowOut<T, MODE>& o) {
  double* base = a.part + (int64_t)r * NQ * a.slots + slot;
  base[Q_S4 * a.slots] = o.s4;
  base[Q_SXAX * a.slots] = o.sxax;
  base[Q_ES * a.slots] = o.es;
  base[Q_STEP * a.slots] = o.step;
  base[Q_SY4 * a.slots] = o.sy4;
  base[Q_SYAY * a.slots] = o.syay;
}

// ---------------------------------------------------------------------------
// R = 1: V lanes cooperate on a row (V = 1 in f64 mode: the canonical
// sequential column-order sum). Grid-stride over rows; one partial slot per warp.
template <typename T, int VK, int V, int MODE>
__global__ void __launch_bounds__(256) pass_r1(PassArgs a) {
  if (!a.g->live) return;
  const int p = a.g->p;
  if (MODE == MODE_ADOCH_Y && p == 0) return;  // no extrapolation at k = 0
  const RepCtl c = a.ctl[0];
  const bool running = c.status == DCX_STOP_RUNNING;
  if (!running && !(MODE == MODE_DOCH && c.pend == p - 1)) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // global warp
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  constexpr int RPW = 32 / V;  // rows per warp step
  const T* xg = reinterpret_cast<const T*>(MODE == MODE_ADOCH_Y ? nullptr : a.x[p & 1]);
  const T* xc = reinterpret_cast<const T*>(a.x[p & 1]);
  const T* xp = reinterpret_cast<const T*>(a.x[(p + 1) & 1]);
  const T cm = T(c.cm[p & 1]);
  const T scale = T(a.scale);
  RowOut<T, MODE> o;
  const int64_t n = a.cfg.n;
  for (int64_t base = gw * RPW; base < n; base += nwarps * RPW) {
    const int64_t i = base + lane / V;
    const bool ok = i < n;
    T acc = T(0);
    typename EsAcc<VK>::type es = 0;
    if (ok && running) {
      const uint32_t lo = __ldg(a.rp + i), hi = __ldg(a.rp + i + 1);
      for (uint32_t e = lo + sub; e < hi; e += V) {
        const int j = __ldg(a.col + e);
        T xj;
        if constexpr (MODE == MODE_ADOCH_Y) xj = extrap(xc[j], xp[j], cm);
        else xj = xg[j];
        int q;
        const T v = load_entry<VK, true, T>(a.val, e, scale, q);
        acc = madd(acc, v, xj);
        if constexpr (MODE != MODE_ADOCH_Y) es += es_term<VK, T>(q, v, xj);
      }
    }
#pragma unroll
    for (int off = V / 2; off > 0; off >>= 1) {
      acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
      es += __shfl_xor_sync(0xffffffffu, es, off);
    }
    if (ok && sub == 0) {
      if (running) row_epilogue<T, MODE>(a, c, p, i, acc, double(es), o);
      else if (MODE == MODE_DOCH) {  // stopped: only the pending copy
        a.best[i] = reinterpret_cast<const T*>(a.x[(p + 1) & 1])[i] >= T(0) ? 1 : -1;
      }
    }
  }
  o.s4 = warp_sum(o.s4);
  o.sxax = warp_sum(o.sxax);
  o.es = warp_sum(o.es);
  o.step = warp_max(o.step);
  o.sy4 = warp_sum(o.sy4);
  o.syay = warp_sum(o.syay);
  if (lane == 0) write_partials<T, MODE>(a, 0, (int)gw, o);
}

// ---------------------------------------------------------------------------
// R > 1: one warp per row, lanes over replicas (layout x[j][r], coalesced),
// RG groups of 32 replicas per lane held in registers so the row's index and
// value stream is read once per 32*RG replicas.
template <typename T, int VK, int RG, int MODE>
__global__ void __launch_bounds__(256) pass_rn(PassArgs a) {
  if (!a.g->live) return;
  const int p = a.g->p;
  if (MODE == MODE_ADOCH_Y && p == 0) return;  // no extrapolation at k = 0
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int R = a.cfg.R;
  const int64_t n = a.cfg.n;
  const T* xc = reinterpret_cast<const T*>(a.x[p & 1]);
  const T* xp = reinterpret_cast<const T*>(a.x[(p + 1) & 1]);
  const T scale = T(a.scale);
  for (int r0 = 0; r0 < R; r0 += 32 * RG) {
    RowOut<T, MODE> o[RG];
    RepCtl c[RG];
    bool run[RG], act[RG];
#pragma unroll
    for (int g = 0; g < RG; ++g) {
      const int r = r0 + g * 32 + lane;
      act[g] = r < R;
      if (act[g]) c[g] = a.ctl[r];
      run[g] = act[g] && c[g].status == DCX_STOP_RUNNING;
      if (act[g] && !run[g] && !(MODE == MODE_DOCH && c[g].pend == p - 1)) act[g] = false;
    }
    for (int64_t i = gw; i < n; i += nwarps) {
      T acc[RG];
      typename EsAcc<VK>::type es[RG];
#pragma unroll
      for (int g = 0; g < RG; ++g) { acc[g] = T(0); es[g] = 0; }
      const uint32_t lo = __ldg(a.rp + i), hi = __ldg(a.rp + i + 1);
      for (uint32_t e = lo; e < hi; ++e) {
        const int64_t j = __ldg(a.col + e);
        int q;
        const T v = load_entry<VK, true, T>(a.val, e, scale, q);
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          if (run[g]) {
            const int64_t o2 = j * R + r0 + g * 32 + lane;
            T xj;
            if constexpr (MODE == MODE_ADOCH_Y) xj = extrap(xc[o2], xp[o2], T(c[g].cm[p & 1]));
            else xj = xc[o2];
            acc[g] = madd(acc[g], v, xj);
            if constexpr (MODE != MODE_ADOCH_Y) es[g] += es_term<VK, T>(q, v, xj);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < RG; ++g) {
        const int64_t idx = i * R + r0 + g * 32 + lane;
        if (run[g]) row_epilogue<T, MODE>(a, c[g], p, idx, acc[g], double(es[g]), o[g]);
        else if (act[g] && MODE == MODE_DOCH)
          a.best[idx] = reinterpret_cast<const T*>(a.x[(p + 1) & 1])[idx] >= T(0) ? 1 : -1;
      }
    }
#pragma unroll
    for (int g = 0; g < RG; ++g) {
      const int r = r0 + g * 32 + lane;
      if (r < R) write_partials<T, MODE>(a, r, (int)gw, o[g]);
    }
  }
}

// ---------------------------------------------------------------------------
// ADOCH finalize (elementwise): x_{p+1} = cbrt(Av/beta) with v = y or x_p as
// decided by control p (doch.py:313-318); pending best copy of x_p; step
// partials. Buffer holding x_{p-1} receives x_{p+1}.
template <typename T>
__global__ void __launch_bounds__(256) adoch_finalize(PassArgs a, double* spart, int sslots) {
  if (!a.g->live) return;
  const int p = a.g->p;
  const int R = a.cfg.R;
  const int64_t total = a.cfg.n * R;
  const T* xc = reinterpret_cast<const T*>(a.x[p & 1]);
  T* xo = reinterpret_cast<T*>(a.x[(p + 1) & 1]);  // holds x_{p-1}
  const T* axc = reinterpret_cast<const T*>(a.ax[p & 1]);
  const T* axp = reinterpret_cast<const T*>(a.ax[(p + 1) & 1]);
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  // R=1 keeps one step max per thread; R>1 requires one per replica: use
  // replica-major striding so a thread always touches the same replica.
  if (R == 1) {
    const RepCtl c = a.ctl[0];
    double st = 0.0;
    const bool run = c.status == DCX_STOP_RUNNING;
    const bool copy = c.pend == p;
    const T beta = T(c.beta), cm = T(c.cm[p & 1]);
    for (int64_t i = tid; i < total; i += nth) {
      const T xi = xc[i];
      if (copy) a.best[i] = xi >= T(0) ? 1 : -1;
      if (!run) continue;
      T av;
      if (p > 0 && c.accept) {
        av = (a.cfg.window_mode == DCX_WINDOW_EXACT) ? reinterpret_cast<const T*>(a.ay)[i]
                                                     : extrap(axc[i], axp[i], cm);
      } else {
        av = axc[i];
      }
      const T xn = tmap(av, beta);
      xo[i] = xn;
      if (a.states) reinterpret_cast<T*>(a.states)[(int64_t)(p + 1) * total + i] = xn;
      st = fmax(st, double(fabs(xn - xi)));
    }
    st = warp_max(st);
    if ((threadIdx.x & 31) == 0) spart[tid >> 5] = st;
    return;
  }
  // R > 1: thread handles replica r = tid % R over rows tid / R stepping nth / R
  // (nth is a multiple of R by construction of the launch).
  const int64_t rstep = nth / R;
  if (tid >= rstep * R) return;
  const int r = int(tid % R);
  const RepCtl c = a.ctl[r];
  const bool run = c.status == DCX_STOP_RUNNING;
  const bool copy = c.pend == p;
  const T beta = T(c.beta), cm = T(c.cm[p & 1]);
  double st = 0.0;
  for (int64_t i = tid / R; i < a.cfg.n; i += rstep) {
    const int64_t idx = i * R + r;
    const T xi = xc[idx];
    if (copy) a.best[idx] = xi >= T(0) ? 1 : -1;
    if (!run) continue;
    T av;
    if (p > 0 && c.accept) {
      av = (a.cfg.window_mode == DCX_WINDOW_EXACT) ? reinterpret_cast<const T*>(a.ay)[idx]
                                                   : extrap(axc[idx], axp[idx], cm);
    } else {
      av = axc[idx];
    }
    const T xn = tmap(av, beta);
    xo[idx] = xn;
    if (a.states) reinterpret_cast<T*>(a.states)[(int64_t)(p + 1) * total + idx] = xn;
    st = fmax(st, double(fabs(xn - xi)));
  }
  spart[(tid / R) * R + r] = st;  // slot = tid / R, replica-minor
}

// ---------------------------------------------------------------------------
// Reduce + control: block r reduces replica r's partial slots in a fixed order
// (deterministic for a fixed launch shape), then thread 0 runs the control.
// phase: 0 = DOCH pass, 1 = ADOCH bookkeeping (+decision if economy),
//        2 = ADOCH exact decision only.
__global__ void __launch_bounds__(256) reduce_control(PassArgs a, const double* spart, int sslots, int phase,
                                                      int last_kernel) {
  if (!a.g->live) return;
  const int p = a.g->p;
  const int r = blockIdx.x;
  const int R = a.cfg.R;
  __shared__ double red[NQ][256];
  __shared__ double tot[NQ + 1];
  RepCtl* cp = a.ctl + r;
  const bool running = cp->status == DCX_STOP_RUNNING;
  if (running) {
    for (int q = 0; q < NQ; ++q) {
      double acc = 0.0;
      const bool ismax = q == Q_STEP;
      const double* src = a.part + ((int64_t)r * NQ + q) * a.slots;
      for (int s = threadIdx.x; s < a.slots; s += blockDim.x) acc = ismax ? fmax(acc, src[s]) : acc + src[s];
      red[q][threadIdx.x] = acc;
    }
    double st = 0.0;
    if (spart) {
      for (int s = threadIdx.x; s < sslots; s += blockDim.x) st = fmax(st, spart[(int64_t)s * R + r]);
    }
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        for (int q = 0; q < NQ; ++q)
          red[q][threadIdx.x] = (q == Q_STEP) ? fmax(red[q][threadIdx.x], red[q][threadIdx.x + w])
                                              : red[q][threadIdx.x] + red[q][threadIdx.x + w];
      }
      __syncthreads();
    }
    // step partials of the ADOCH finalize
    __shared__ double sred[256];
    sred[threadIdx.x] = st;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) sred[threadIdx.x] = fmax(sred[threadIdx.x], sred[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      for (int q = 0; q < NQ; ++q) tot[q] = red[q][0];
      tot[NQ] = sred[0];
      RepCtl c = *cp;
      const double now = double(globaltimer() - a.g->t0) * 1e-9;
      bool stopped = false;
      if (phase == 0) {
        stopped = control_after_pass(c, a.cfg, r, tot, p, now);
        c.step = tot[Q_STEP];
      } else if (phase == 1) {
        if (p > 0) c.step = tot[NQ];  // step of the update x_{p-1} -> x_p
        stopped = control_after_pass(c, a.cfg, r, tot, p, now);
        if (!stopped && a.cfg.window_mode == DCX_WINDOW_ECONOMY) adoch_decide(c, a.cfg, r, tot, p);
      } else {
        adoch_decide(c, a.cfg, r, tot, p);
      }
      *cp = c;
      if (stopped) atomicSub(&a.g->running, 1);
    }
  }
  if (last_kernel) {
    // last block to finish advances the global pass counter
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const uint32_t prev = atomicAdd(&a.g->arrive, 1u);
      if (prev == gridDim.x - 1) {
        __threadfence();
        a.g->arrive = 0;
        a.g->p = p + 1;
        if (atomicAdd(&a.g->running, 0) == 0) a.g->live = 0;
        __threadfence();
      }
    }
  }
}

// ADOCH: the finalize is the last kernel of the iteration; a 1-thread kernel
// advances the pass counter afterwards (keeps the finalize free of atomics).
__global__ void advance_pass(GState* g) {
  if (!g->live) return;
  g->p = g->p + 1;
  if (g->running == 0) g->live = 0;
}

// ADOCH: freeze the decision for stopped replicas and let the exact-mode
// y-pass / decision run only for p > 0.
__global__ void start_clock(GState* g) { g->t0 = globaltimer(); }

// DOCH: copy the pending best spins after the last pass.
template <typename T>
__global__ void flush_best(PassArgs a) {
  const int R = a.cfg.R;
  const int64_t total = a.cfg.n * R;
  const int P = a.g->p - 1;  // last executed pass
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % R);
    const int pe = a.ctl[r].pend;
    if (pe >= 0 && pe == P) a.best[idx] = reinterpret_cast<const T*>(a.x[pe & 1])[idx] >= T(0) ? 1 : -1;
  }
}

// ---------------------------------------------------------------- operators
// y = J v (+ alpha v, cbrt) for R vectors: the operator seam used by matvec,
// apply_T, hamiltonian and energy (dc/matvec.py:99-114,181-190). Same row sum
// order as the passes (V lanes per row; V = 1 in f64 mode).
template <typename T, int VK, int V>
__global__ void __launch_bounds__(256) csr_apply(const uint32_t* rp, const int32_t* col, const void* val,
                                                double scale_d, const T* v, int64_t n, int R, T* jv,
                                                double* es_rows) {
  const int lane = threadIdx.x & 31, sub = lane % V;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  constexpr int RPW = 32 / V;
  const T scale = T(scale_d);
  for (int r = 0; r < R; ++r) {
    for (int64_t base = gw * RPW; base < n; base += nwarps * RPW) {
      const int64_t i = base + lane / V;
      const bool ok = i < n;
      T acc = T(0);
      typename EsAcc<VK>::type es = 0;
      if (ok) {
        const uint32_t lo = rp[i], hi = rp[i + 1];
        for (uint32_t e = lo + sub; e < hi; e += V) {
          const int64_t j = col[e];
          const T xj = v[j * R + r];
          int q;
          const T vv = load_entry<VK, true, T>(val, e, scale, q);
          acc = madd(acc, vv, xj);
          es += es_term<VK, T>(q, vv, xj);
        }
      }
#pragma unroll
      for (int off = V / 2; off > 0; off >>= 1) {
        acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        es += __shfl_xor_sync(0xffffffffu, es, off);
      }
      if (ok && sub == 0) {
        jv[i * R + r] = acc;
        if (es_rows) es_rows[i * R + r] = double(es);
      }
    }
  }
}

// ------------------------------------------------------------------ launch
template <typename T, int VK, int V>
static void launch_r1(int mode, const PassArgs& a, int grid, cudaStream_t s) {
  switch (mode) {
    case MODE_DOCH: pass_r1<T, VK, V, MODE_DOCH><<<grid, 256, 0, s>>>(a); break;
    case MODE_ADOCH_X: pass_r1<T, VK, V, MODE_ADOCH_X><<<grid, 256, 0, s>>>(a); break;
    default: pass_r1<T, VK, V, MODE_ADOCH_Y><<<grid, 256, 0, s>>>(a); break;
  }
}
template <typename T, int VK, int RG>
static void launch_rn(int mode, const PassArgs& a, int grid, cudaStream_t s) {
  switch (mode) {
    case MODE_DOCH: pass_rn<T, VK, RG, MODE_DOCH><<<grid, 256, 0, s>>>(a); break;
    case MODE_ADOCH_X: pass_rn<T, VK, RG, MODE_ADOCH_X><<<grid, 256, 0, s>>>(a); break;
    default: pass_rn<T, VK, RG, MODE_ADOCH_Y><<<grid, 256, 0, s>>>(a); break;
  }
}

template <typename T, int VK>
static void launch_pass_vk(int mode, const PassArgs& a, int V, int grid, cudaStream_t s) {
  if (a.cfg.R == 1) {
    switch (V) {
      case 1: launch_r1<T, VK, 1>(mode, a, grid, s); break;
      case 2: launch_r1<T, VK, 2>(mode, a, grid, s); break;
      case 4: launch_r1<T, VK, 4>(mode, a, grid, s); break;
      case 8: launch_r1<T, VK, 8>(mode, a, grid, s); break;
      case 16: launch_r1<T, VK, 16>(mode, a, grid, s); break;
      default: launch_r1<T, VK, 32>(mode, a, grid, s); break;
    }
  } else {
    const int R = a.cfg.R;
    if (R <= 32) launch_rn<T, VK, 1>(mode, a, grid, s);
    else if (R <= 64) launch_rn<T, VK, 2>(mode, a, grid, s);
    else if (R <= 128) launch_rn<T, VK, 4>(mode, a, grid, s);
    else launch_rn<T, VK, 8>(mode, a, grid, s);
  }
}

template <typename T>
static void launch_pass_t(int mode, const PassArgs& a, int vk, int V, int grid, cudaStream_t s) {
  switch (vk) {
    case VK_UNIFORM: launch_pass_vk<T, VK_UNIFORM>(mode, a, V, grid, s); break;
    case VK_I8: launch_pass_vk<T, VK_I8>(mode, a, V, grid, s); break;
    case VK_I16: launch_pass_vk<T, VK_I16>(mode, a, V, grid, s); break;
    case VK_F32: launch_pass_vk<T, VK_F32>(mode, a, V, grid, s); break;
    default: launch_pass_vk<T, VK_F64>(mode, a, V, grid, s); break;
  }
}

template <typename T, int VK>
static void launch_apply_vk(const CsrDev& J, const T* v, int R, T* jv, double* es, cudaStream_t s) {
  const int grid = J.grid;
  switch (J.V) {
    case 1: csr_apply<T, VK, 1><<<grid, 256, 0, s>>>(J.rp, J.col, J.val, J.scale, v, J.n, R, jv, es); break;
    case 2: csr_apply<T, VK, 2><<<grid, 256, 0, s>>>(J.rp, J.col, J.val, J.scale, v, J.n, R, jv, es); break;
    case 4: csr_apply<T, VK, 4><<<grid, 256, 0, s>>>(J.rp, J.col, J.val, J.scale, v, J.n, R, jv, es); break;
    case 8: csr_apply<T, VK, 8><<<grid, 256, 0, s>>>(J.rp, J.col, J.val, J.scale, v, J.n, R, jv, es); break;
    case 16: csr_apply<T, VK, 16><<<grid, 256, 0, s>>>(J.rp, J.col, J.val, J.scale, v, J.n, R, jv, es); break;
    default: csr_apply<T, VK, 32><<<grid, 256, 0, s>>>(J.rp, J.col, J.val, J.scale, v, J.n, R, jv, es); break;
  }
}

template <typename T>
void launch_csr_apply(const CsrDev& J, const T* v, int R, T* jv, double* es, cudaStream_t s) {
  switch (J.vk) {
    case VK_UNIFORM: launch_apply_vk<T, VK_UNIFORM>(J, v, R, jv, es, s); break;
    case VK_I8: launch_apply_vk<T, VK_I8>(J, v, R, jv, es, s); break;
    case VK_I16: launch_apply_vk<T, VK_I16>(J, v, R, jv, es, s); break;
    case VK_F32: launch_apply_vk<T, VK_F32>(J, v, R, jv, es, s); break;
    default: launch_apply_vk<T, VK_F64>(J, v, R, jv, es, s); break;
  }
}
template void launch_csr_apply<double>(const CsrDev&, const double*, int, double*, double*, cudaStream_t);
template void launch_csr_apply<float>(const CsrDev&, const float*, int, float*, double*, cudaStream_t);

// One iteration of the multi-pass path (enqueued; no host sync).
void enqueue_iteration(const MultiPass& m, cudaStream_t s) {
  PassArgs a = m.args;
  const bool f64 = m.f64;
  const int sslots = m.sslots;
  if (m.solver == DCX_SOLVER_DOCH) {
    if (f64) launch_pass_t<double>(MODE_DOCH, a, m.vk, m.V, m.grid, s);
    else launch_pass_t<float>(MODE_DOCH, a, m.vk, m.V, m.grid, s);
    reduce_control<<<a.cfg.R, 256, 0, s>>>(a, nullptr, 0, 0, 1);
    return;
  }
  if (f64) launch_pass_t<double>(MODE_ADOCH_X, a, m.vk, m.V, m.grid, s);
  else launch_pass_t<float>(MODE_ADOCH_X, a, m.vk, m.V, m.grid, s);
  reduce_control<<<a.cfg.R, 256, 0, s>>>(a, m.spart, sslots, 1, 0);
  if (a.cfg.window_mode == DCX_WINDOW_EXACT) {
    if (f64) launch_pass_t<double>(MODE_ADOCH_Y, a, m.vk, m.V, m.grid, s);
    else launch_pass_t<float>(MODE_ADOCH_Y, a, m.vk, m.V, m.grid, s);
    reduce_control<<<a.cfg.R, 256, 0, s>>>(a, nullptr, 0, 2, 0);
  }
  if (f64) adoch_finalize<double><<<m.fgrid, 256, 0, s>>>(a, m.spart, sslots);
  else adoch_finalize<float><<<m.fgrid, 256, 0, s>>>(a, m.spart, sslots);
  advance_pass<<<1, 1, 0, s>>>(a.g);
}

// The dominant kernel alone (the fused SpMV/SpMM pass), for live profiling.
void enqueue_pass_only(const MultiPass& m, cudaStream_t s) {
  const int mode = m.solver == DCX_SOLVER_DOCH ? MODE_DOCH : MODE_ADOCH_X;
  if (m.f64) launch_pass_t<double>(mode, m.args, m.vk, m.V, m.grid, s);
  else launch_pass_t<float>(mode, m.args, m.vk, m.V, m.grid, s);
}

void enqueue_flush(const MultiPass& m, cudaStream_t s) {
  if (m.solver != DCX_SOLVER_DOCH) return;
  if (m.f64) flush_best<double><<<256, 256, 0, s>>>(m.args);
  else flush_best<float><<<256, 256, 0, s>>>(m.args);
}

void enqueue_start_clock(GState* g, cudaStream_t s) { start_clock<<<1, 1, 0, s>>>(g); }

}  // namespace dcx
