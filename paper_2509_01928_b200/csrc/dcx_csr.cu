// Multi-pass CSR path: one fused SpMV/SpMM + DC-update pass per iteration,
// a per-replica reduce+control kernel, and (ADOCH) an elementwise finalize.
//
// Replaces, per iteration, dc/solvers/doch.py:199-232 (DOCH) / :294-342 (ADOCH)
// with scipy csr_matvec (dc/coupling.py:189-190) as the product. One pass
// reads the CSR stream once and gathers x once; from the same gather it forms
// (J+aI)x, the next iterate, and J*sign(x) for the spin energy (exact integer
// accumulation for integer couplings), plus the H / E / step partials.
#include <cstdlib>

#include "dcx_internal.h"
#include "dcx_rows.cuh"

namespace dcx {



// ---------------------------------------------------------------------------
// R = 1: V lanes cooperate on a row (V = 1 in f64 mode: the canonical
// sequential column-order sum). Grid-stride over rows; one partial slot per warp.
template <typename T, int VK, int V, int MODE>
__global__ void __launch_bounds__(256) pass_r1(PassArgs a) {
  if (!a.g->live) return;
  const int p = a.g->p;
  if (MODE == MODE_ADOCH_Y && p == 0) return;  // no extrapolation at k = 0
  const RowCtl<T> c = row_ctl<T>(a.ctl[0], p);
  const bool running = c.running;
  if (!running && !(MODE == MODE_DOCH && c.pend == copy_iter(a, p) && c.pend >= 0)) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // global warp
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  constexpr int RPW = 32 / V;  // rows per warp step
  const T* xc = reinterpret_cast<const T*>(a.gx[xslot(a, p)]);  // gather source (all spins)
  const T* xp = reinterpret_cast<const T*>(a.gx[xslot(a, p + a.nbuf - 1)]);  // x_{p-1}
  const T cm = c.cm;
  const T scale = T(a.scale);
  RowOut<T, MODE> o;
  const int64_t n = a.cfg.n;
  // Software pipeline over this warp's row batches b, b+S, b+2S: while batch b
  // gathers, the first two column entries of each lane's row in batch b+S and
  // the row pointers of batch b+2S are in flight, so a row's gathers issue
  // without waiting for its index loads.
  const int64_t S = nwarps * RPW;
  const uint32_t* rp = a.rp;  // locals: a lambda must not take the address of the kernel parameter
  const int32_t* colp = a.col;
  auto load_rp = [rp, running, n, lane](int64_t b, uint32_t& lo, uint32_t& hi) {
    const int64_t i = b + lane / V;
    lo = hi = 0;
    if (running && i < n) { lo = __ldg(rp + i); hi = __ldg(rp + i + 1); }
  };
  auto load_cols = [colp, sub](uint32_t lo, uint32_t hi, int& c0, int& c1) {
    c0 = c1 = 0;
    if (lo + sub < hi) c0 = __ldg(colp + lo + sub);
    if (lo + sub + V < hi) c1 = __ldg(colp + lo + sub + V);
  };
  auto gather = [xc, xp, cm](int j) -> T {
    if constexpr (MODE == MODE_ADOCH_Y) return extrap(xc[j], xp[j], cm);
    else return xc[j];
  };
  uint32_t c_lo, c_hi, n_lo, n_hi;
  int c_c0, c_c1;
  int64_t base = gw * RPW;
  load_rp(base, c_lo, c_hi);
  load_cols(c_lo, c_hi, c_c0, c_c1);
  load_rp(base + S, n_lo, n_hi);
  for (; base < n; base += S) {
    int f_c0, f_c1;
    uint32_t f_lo, f_hi;
    load_cols(n_lo, n_hi, f_c0, f_c1);  // batch b+S
    load_rp(base + 2 * S, f_lo, f_hi);  // batch b+2S
    const int64_t i = base + lane / V;
    const bool ok = i < n;
    T acc = T(0);
    typename EsAcc<VK>::type es = 0;
    if (ok && running) {
      // the first two entries of this lane (prefetched columns): both gathers in flight together
      const uint32_t e0 = c_lo + sub, e1 = e0 + V;
      const bool h0 = e0 < c_hi, h1 = e1 < c_hi;
      const T x0 = h0 ? gather(c_c0) : T(0);
      const T x1 = h1 ? gather(c_c1) : T(0);
      if (h0) {
        int q;
        const T v = load_entry<VK, true, T>(a.val, e0, scale, q);
        acc = madd(acc, v, x0);
        if constexpr (MODE != MODE_ADOCH_Y) es += es_term<VK, T>(q, v, x0);
      }
      if (h1) {
        int q;
        const T v = load_entry<VK, true, T>(a.val, e1, scale, q);
        acc = madd(acc, v, x1);
        if constexpr (MODE != MODE_ADOCH_Y) es += es_term<VK, T>(q, v, x1);
      }
      for (uint32_t e = e1 + V; e < c_hi; e += V) {  // longer rows: the rest in column order
        const int j = __ldg(a.col + e);
        const T xj = gather(j);
        int q;
        const T v = load_entry<VK, true, T>(a.val, e, scale, q);
        acc = madd(acc, v, xj);
        if constexpr (MODE != MODE_ADOCH_Y) es += es_term<VK, T>(q, v, xj);
      }
    }
    c_lo = n_lo; c_hi = n_hi; c_c0 = f_c0; c_c1 = f_c1;
    n_lo = f_lo; n_hi = f_hi;
#pragma unroll
    for (int off = V / 2; off > 0; off >>= 1) {
      acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
      es += __shfl_xor_sync(0xffffffffu, es, off);
    }
    if (ok && sub == 0) {
      if (running) row_epilogue<T, MODE>(a, c, p, i, acc, double(es), o);
      else if (MODE == MODE_DOCH) {  // stopped: only the pending copy
        a.best[i] = reinterpret_cast<const T*>(a.x[xslot(a, p + 1)])[i] >= T(0) ? 1 : -1;
      }
    }
  }
  o.s4 = warp_sum(o.s4);
  o.sxax = warp_sum(o.sxax);
  o.es = warp_sum(o.es);
  o.step = warp_max(o.step);
  o.sy4 = warp_sum(o.sy4);
  o.syay = warp_sum(o.syay);
  // one partial slot per block: the 8 warp sums in warp order (deterministic)
  __shared__ double red[8][NQ];
  const int warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[warp][Q_S4] = o.s4;
    red[warp][Q_SXAX] = o.sxax;
    red[warp][Q_ES] = o.es;
    red[warp][Q_STEP] = o.step;
    red[warp][Q_SY4] = o.sy4;
    red[warp][Q_SYAY] = o.syay;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    RowOut<T, MODE> b;
    b.s4 = red[0][Q_S4]; b.sxax = red[0][Q_SXAX]; b.es = red[0][Q_ES];
    b.step = red[0][Q_STEP]; b.sy4 = red[0][Q_SY4]; b.syay = red[0][Q_SYAY];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      b.s4 += red[w][Q_S4]; b.sxax += red[w][Q_SXAX]; b.es += red[w][Q_ES];
      b.step = fmax(b.step, red[w][Q_STEP]); b.sy4 += red[w][Q_SY4]; b.syay += red[w][Q_SYAY];
    }
    write_partials<T, MODE>(a, 0, (int)blockIdx.x, b);
  }
}

// ---------------------------------------------------------------------------
// R = 1, f32, integer couplings (UNIFORM / I8): entry-parallel pass. A warp owns
// 32 consecutive rows (one per lane) and walks their contiguous CSR entries in
// rounds of 32 x EPL: every lane loads EPL consecutive column indices with
// 16-byte vector loads (coalesced across the warp) and issues all EPL gathers of
// x before the first one is consumed, so a lane keeps EPL random loads in flight
// (the degree-8 graphs of E7 / R8 are bound by the L1 wavefronts of these
// gathers: one 32-byte sector per 4-byte load). The gathered values go to a
// per-warp shared-memory tile, entry k of lane l at k * 33 + l (each store
// instruction writes 32 consecutive words; the rows' reads below spread over the
// banks by the pad), then every lane sums ITS row's entries in column order (f32
// FMA, the order of the V = 1 kernel) with the exact integer spin-energy
// accumulator, and runs the shared row epilogue. Rows longer than a round
// continue into the next one.
constexpr int R1W_EPL = 12;                    // entries per lane per round
constexpr int R1W_ROUND = 32 * R1W_EPL;        // 384 entries per warp per round
constexpr int R1W_SLOT = R1W_EPL * 33;
// shared-memory slot of the round's entry e_rel = R1W_EPL * lane + k
__device__ __forceinline__ int r1w_pos(int e_rel) {
  const int l = e_rel / R1W_EPL;
  return (e_rel - l * R1W_EPL) * 33 + l;
}

template <int VK, int MODE>
__global__ void __launch_bounds__(256) pass_r1w(PassArgs a) {
  using T = float;
  static_assert(VK == VK_UNIFORM || VK == VK_I8, "integer couplings");
  if (!a.g->live) return;
  const int p = a.g->p;
  if (MODE == MODE_ADOCH_Y && p == 0) return;  // no extrapolation at k = 0
  const RowCtl<T> c = row_ctl<T>(a.ctl[0], p);
  const bool running = c.running;
  if (!running && !(MODE == MODE_DOCH && c.pend == copy_iter(a, p) && c.pend >= 0)) return;
  __shared__ float sx[8][R1W_SLOT];
  __shared__ int8_t sq[VK == VK_I8 ? 8 : 1][VK == VK_I8 ? R1W_SLOT : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const T* xc = reinterpret_cast<const T*>(a.gx[xslot(a, p)]);
  const T* xp = reinterpret_cast<const T*>(a.gx[xslot(a, p + a.nbuf - 1)]);  // x_{p-1}
  const T cm = c.cm;
  const T scale = T(a.scale);
  const int64_t n = a.cfg.n;
  const int32_t* colp = a.col;
  const int8_t* valp = reinterpret_cast<const int8_t*>(a.val);
  float* my = sx[warp];
  RowOut<T, MODE> o;
  for (int64_t i0 = gw * 32; i0 < n; i0 += nwarps * 32) {
    const int64_t i = i0 + lane;
    const bool ok = i < n;
    uint32_t lo = 0, hi = 0;
    if (ok) {
      lo = __ldg(a.rp + i);
      hi = __ldg(a.rp + i + 1);
    }
    const int last = int(n - 1 - i0 < 31 ? n - 1 - i0 : 31);
    const uint32_t E0 = __shfl_sync(0xffffffffu, lo, 0), E1 = __shfl_sync(0xffffffffu, hi, last);
    T acc = T(0);
    int es = 0;
    if (running) {
      for (uint32_t base = E0 & ~3u; base < E1; base += R1W_ROUND) {
        const uint32_t eb = base + uint32_t(R1W_EPL) * lane;  // 16-byte aligned
        int cj[R1W_EPL];
        if (eb < E1) {
#pragma unroll
          for (int v = 0; v < R1W_EPL / 4; ++v) {
            const int4 q4 = __ldg(reinterpret_cast<const int4*>(colp + eb) + v);
            cj[4 * v] = q4.x; cj[4 * v + 1] = q4.y; cj[4 * v + 2] = q4.z; cj[4 * v + 3] = q4.w;
          }
        }
        T xv[R1W_EPL];
#pragma unroll
        for (int k = 0; k < R1W_EPL; ++k) {  // every gather of the lane in flight
          const uint32_t e = eb + k;
          xv[k] = T(0);
          if (e >= E0 && e < E1) {
            if constexpr (MODE == MODE_ADOCH_Y) xv[k] = extrap(xc[cj[k]], xp[cj[k]], cm);
            else xv[k] = xc[cj[k]];
          }
        }
#pragma unroll
        for (int k = 0; k < R1W_EPL; ++k) my[k * 33 + lane] = xv[k];
        if constexpr (VK == VK_I8) {
          if (eb < E1) {
            // 12 bytes at a 4-byte aligned offset (eb % 4 == 0): three word loads
            int qw[3];
#pragma unroll
            for (int v = 0; v < 3; ++v) qw[v] = __ldg(reinterpret_cast<const int*>(valp + eb) + v);
            const int8_t* b = reinterpret_cast<const int8_t*>(qw);
#pragma unroll
            for (int k = 0; k < 12; ++k) sq[warp][k * 33 + lane] = b[k];
          }
        }
        __syncwarp();
        if (ok) {
          const uint32_t a0 = max(lo, base), a1 = min(hi, base + uint32_t(R1W_ROUND));
          for (uint32_t e = a0; e < a1; ++e) {  // this row's entries, column order
            const int k = r1w_pos(int(e - base));
            const T xj = my[k];
            if constexpr (VK == VK_UNIFORM) {
              acc = madd(acc, scale, xj);
              es += negbit(xj) ? -1 : 1;
            } else {
              const int q = sq[warp][k];
              acc = madd(acc, scale * T(q), xj);
              es += negbit(xj) ? -q : q;
            }
          }
        }
        __syncwarp();
      }
    }
    if (ok) {
      if (running) row_epilogue<T, MODE>(a, c, p, i, acc, double(es), o);
      else if (MODE == MODE_DOCH) {  // stopped: only the pending copy
        a.best[i] = reinterpret_cast<const T*>(a.x[xslot(a, p + 1)])[i] >= T(0) ? 1 : -1;
      }
    }
  }
  o.s4 = warp_sum(o.s4);
  o.sxax = warp_sum(o.sxax);
  o.es = warp_sum(o.es);
  o.step = warp_max(o.step);
  o.sy4 = warp_sum(o.sy4);
  o.syay = warp_sum(o.syay);
  __shared__ double red[8][NQ];
  if (lane == 0) {
    red[warp][Q_S4] = o.s4;
    red[warp][Q_SXAX] = o.sxax;
    red[warp][Q_ES] = o.es;
    red[warp][Q_STEP] = o.step;
    red[warp][Q_SY4] = o.sy4;
    red[warp][Q_SYAY] = o.syay;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    RowOut<T, MODE> b;
    b.s4 = red[0][Q_S4]; b.sxax = red[0][Q_SXAX]; b.es = red[0][Q_ES];
    b.step = red[0][Q_STEP]; b.sy4 = red[0][Q_SY4]; b.syay = red[0][Q_SYAY];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      b.s4 += red[w][Q_S4]; b.sxax += red[w][Q_SXAX]; b.es += red[w][Q_ES];
      b.step = fmax(b.step, red[w][Q_STEP]); b.sy4 += red[w][Q_SY4]; b.syay += red[w][Q_SYAY];
    }
    write_partials<T, MODE>(a, 0, (int)blockIdx.x, b);
  }
}

// ---------------------------------------------------------------------------
// R > 1: replica-vector kernel. Layout x[j][r] (replicas contiguous per spin).
// blockIdx.y selects a chunk of 32*VW replicas; each lane owns VW consecutive
// replicas and moves them with one 16-byte load/store (VW = 16 / sizeof(T)
// when R is a multiple of it, else 1). A warp walks one row at a time: the
// row's column/value entries are fetched 32 at a time with one coalesced load
// and broadcast by shuffle, and neighbour rows are gathered UNROLL at a time so
// several independent 16-byte loads are in flight per lane. Per-replica sums
// stay in column order (the scipy order, bit-exact in f64).
// Partials: one slot per block (blockIdx.x), reduced across the block's warps
// in a fixed order, so slots = gridDim.x.
template <typename T, int VW>
struct VecT;
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<double, 1> { using type = double; };
template <> struct VecT<double, 2> { using type = double2; };

template <typename T, int VW>
__device__ __forceinline__ void vload(const T* p, T (&out)[VW]) {
  using V = typename VecT<T, VW>::type;
  const V v = *reinterpret_cast<const V*>(p);
  memcpy(out, &v, sizeof(V));
}
template <typename T, int VW>
__device__ __forceinline__ void vstore(T* p, const T (&in)[VW]) {
  using V = typename VecT<T, VW>::type;
  V v;
  memcpy(&v, in, sizeof(V));
  *reinterpret_cast<V*>(p) = v;
}

// Per-row spin-energy accumulator (J sign x_p)_i of the replica kernel, by
// value kind; padding edges carry q = 0 / v = 0 / x = +0 and add nothing.
template <int VK, typename T>
struct EsRow {  // real values: double sum of +-v
  double s = 0.0;
  __device__ __forceinline__ void add(int, float, T v, T x) { s += negbit(x) ? -double(v) : double(v); }
  __device__ __forceinline__ double value(uint32_t) const { return s; }
};
template <typename T>
struct EsRowF {  // q in {0, 1} (UNIFORM) or |q| <= 127 (I8), row sum of |q| < 2^24 (enforced on upload): exact in f32
  float s = 0.0f;
  __device__ __forceinline__ void add(int, float qf, T, T x) { s = fmaf(qf, sgnf_bits(x), s); }
  __device__ __forceinline__ double value(uint32_t) const { return double(s); }
  __device__ __forceinline__ float value_f() const { return s; }
};
template <typename T>
struct EsRow<VK_UNIFORM, T> : EsRowF<T> {};
template <typename T>
struct EsRow<VK_I8, T> : EsRowF<T> {};
template <typename T>
struct EsRow<VK_I16, T> {
  int s = 0;
  __device__ __forceinline__ void add(int q, float, T, T x) {
    const int m = -int(negbit(x));
    s += (q ^ m) - m;
  }
  __device__ __forceinline__ double value(uint32_t) const { return double(s); }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int B>
__device__ __forceinline__ void cp_async(uint32_t dst, const void* src) {
  if constexpr (B == 16) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  else if constexpr (B == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// edges per row staged through shared memory by cp.async (0: gather directly)
template <int MODE>
constexpr int rv_staged_edges() { return MODE == MODE_ADOCH_Y ? 0 : 8; }
template <typename T, int VW, int MODE>
constexpr size_t rv_smem_bytes() { return size_t(2) * 8 * rv_staged_edges<MODE>() * 32 * VW * sizeof(T); }

template <typename T, int VK, int VW, int MODE>
__global__ void __launch_bounds__(256, (VW * sizeof(T) >= 16) ? 2 : 3) pass_rv(PassArgs a) {
  constexpr int UNROLL = 4;
  constexpr int G = rv_staged_edges<MODE>();
  constexpr int CB = VW * int(sizeof(T));  // bytes per lane per spin row
  extern __shared__ __align__(16) unsigned char stage_mem[];
  if (!a.g->live) return;
  const int p = a.g->p;
  if (MODE == MODE_ADOCH_Y && p == 0) return;  // no extrapolation at k = 0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = a.cfg.R;
  const int64_t n = a.cfg.n;
  const int r0 = blockIdx.y * 32 * VW + lane * VW;  // this lane's first replica
  const bool lane_on = r0 < R;                      // all VW replicas in or all out
  T alpha[VW], beta[VW], ibeta[VW], cm[VW];
  bool run[VW], copy[VW];
  bool any_run = false, all_run = true, any_copy = false;
#pragma unroll
  for (int v = 0; v < VW; ++v) {
    run[v] = copy[v] = false;
    alpha[v] = beta[v] = cm[v] = T(0);
    ibeta[v] = T(1);
    if (lane_on) {
      const RepCtl& c = a.ctl[r0 + v];
      run[v] = c.status == DCX_STOP_RUNNING;
      copy[v] = MODE == MODE_DOCH && c.pend >= 0 && c.pend == copy_iter(a, p);
      alpha[v] = T(c.alpha);
      beta[v] = T(c.beta);
      ibeta[v] = inv_beta(beta[v]);
      cm[v] = T(c.cm[p & 1]);
    }
    any_run |= run[v];
    all_run &= run[v];
    any_copy |= copy[v];
  }
  // nothing to do for this replica chunk (block-uniform: the chunk is per block)
  if (!__syncthreads_or(any_run || any_copy)) return;
  const bool warp_run = __any_sync(0xffffffffu, any_run);
  const T* xc = reinterpret_cast<const T*>(a.x[xslot(a, p)]);
  const T* xp = reinterpret_cast<const T*>(a.x[xslot(a, p + a.nbuf - 1)]);  // x_{p-1}
  T* xn_buf = reinterpret_cast<T*>(a.x[xslot(a, p + 1)]);  // x_{p+1} (holds the copy iterate)
  const T scale = T(a.scale);
  // per-replica partials over this warp's rows, in T (f32 mode: a few hundred
  // rows per lane, summed in double across warps and blocks); the step max is
  // exact in T; the spin-energy sum stays in double (exact for integer J)
  T s4[VW], sxax[VW], sy4[VW], syay[VW], step[VW];
  double esum[VW];
  float esf[VW];  // exact f32 spin-energy sums (a.es_f32, integer kinds)
  const bool es32 = (VK == VK_UNIFORM || VK == VK_I8 || VK == VK_I16) && a.es_f32;
#pragma unroll
  for (int v = 0; v < VW; ++v) {
    s4[v] = sxax[v] = sy4[v] = syay[v] = step[v] = T(0);
    esum[v] = 0.0;
    esf[v] = 0.0f;
  }

  // Pipeline over this warp's rows A = i, B = i+S, C = i+2S, D = i+3S. While
  // row A is computed, the neighbour-row chunks of B's first G edges are in
  // flight into shared memory (cp.async), C's first column batch and D's row
  // pointers are in flight into registers.
  const int64_t S = int64_t(gridDim.x) * 8;
  int64_t i = int64_t(blockIdx.x) * 8 + warp;
  const uint32_t rowb = uint32_t(R) * uint32_t(sizeof(T));  // bytes per spin row of x
  const char* xcb = reinterpret_cast<const char*>(reinterpret_cast<const T*>(a.gx[xslot(a, p)]) + r0);  // gathers
  const char* xpb = reinterpret_cast<const char*>(reinterpret_cast<const T*>(a.gx[xslot(a, p + a.nbuf - 1)]) + r0);
  // stage s of this warp, edge e, this lane: stage_mem + ((s*8 + warp)*G + e)*32*CB + lane*CB
  const uint32_t st_base = smem_u32(stage_mem) + uint32_t((warp * G * 32 + lane) * CB);
  constexpr uint32_t ST_STRIDE = 8u * G * 32 * CB;  // between stages
  auto load_rp = [&](int64_t r, uint32_t& lo, uint32_t& hi) {
    lo = hi = 0;
    if (warp_run && r < n) { lo = __ldg(a.rp + r); hi = __ldg(a.rp + r + 1); }
  };
  auto load_batch = [&](uint32_t base, uint32_t hi, int& col, int& q, T& v) {
    col = 0; q = 0; v = T(0);
    if (base + lane < hi) {
      col = __ldg(a.col + base + lane);
      v = load_entry<VK, true, T>(a.val, base + lane, scale, q);
    }
  };
  // TMA staging (a.xmap set): one tile::gather4 per four staged edges, issued by
  // lane 0 with the columns the batch registers hold, completion on an mbarrier
  const bool tma = G > 0 && a.xmap[0] != nullptr;
  const void* xmap = a.xmap[xslot(a, p)];
  const int cb = int(blockIdx.y) * 32 * VW;  // first replica of this block's chunk
  constexpr uint32_t CHUNK = 32u * CB;
  __shared__ __align__(8) uint64_t stage_bar[8][2];
  const uint32_t mb0 = smem_u32(&stage_bar[warp][0]);
  uint32_t bar_par = 0;
  auto stage_row = [&](int s, uint32_t lo, uint32_t hi, int col) {
    if constexpr (G > 0) {
      const uint32_t deg = hi - lo;
      if (tma) {
        const uint32_t ne = min(deg, uint32_t(G));
        if (ne == 0) return;
        int jj[G];
#pragma unroll
        for (int e = 0; e < G; ++e) jj[e] = __shfl_sync(0xffffffffu, col, e);
        if (lane == 0) {
#pragma unroll
          for (int e = 1; e < G; ++e)
            if (uint32_t(e) >= ne) jj[e] = jj[0];  // padding rows: any valid row (weight 0)
          const uint32_t nq = (ne + 3) / 4;
          const uint32_t mb = mb0 + 8u * s;
          const uint32_t dst = smem_u32(stage_mem) + uint32_t((s * 8 + warp) * G) * CHUNK;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(nq * 4 * CHUNK)
                       : "memory");
#pragma unroll
          for (uint32_t g = 0; g < uint32_t(G) / 4; ++g)
            if (g < nq)
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes "
                  "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst + g * 4 * CHUNK),
                  "l"(reinterpret_cast<uint64_t>(xmap)), "r"(cb), "r"(jj[4 * g]), "r"(jj[4 * g + 1]),
                  "r"(jj[4 * g + 2]), "r"(jj[4 * g + 3]), "r"(mb)
                  : "memory");
        }
        return;
      }
#pragma unroll
      for (int e = 0; e < G; ++e) {
        if (e >= deg) break;  // warp-uniform
        const uint32_t j = uint32_t(__shfl_sync(0xffffffffu, col, e));
        if (lane_on) cp_async<CB>(st_base + s * ST_STRIDE + e * 32 * CB, xcb + size_t(j) * rowb);
      }
      cp_async_commit();
    }
  };
  if constexpr (G > 0) {
    // stage slots past a row's degree are read as padding (times a zero
    // weight): start them at +0 so stale contents are always finite values
    const T z[VW] = {};
    for (int e = 0; e < 2 * G; ++e)
      vstore<T, VW>(reinterpret_cast<T*>(stage_mem + ((e / G) * ST_STRIDE + (warp * G + e % G) * 32 * CB + lane * CB)), z);
    if (tma && lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8) : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero fill / inits before async-proxy writes
    __syncwarp();
  }
  // one edge's value / integer weight from the lane-distributed batch registers
  auto edge_value = [&](int kk, bool real, int myq, T myv, int& q, T& v) {
    if constexpr (VK == VK_UNIFORM) { q = real; v = real ? scale : T(0); }
    else if constexpr (VK == VK_F32 || VK == VK_F64) { q = 0; v = __shfl_sync(0xffffffffu, myv, kk & 31); }
    else { q = __shfl_sync(0xffffffffu, myq, kk & 31); v = scale * T(q); }
  };

  uint32_t a_lo, a_hi, b_lo, b_hi, c_lo, c_hi;
  int a_col, a_q, b_col, b_q;
  T a_v, b_v;
  load_rp(i, a_lo, a_hi);
  load_batch(a_lo, a_hi, a_col, a_q, a_v);
  load_rp(i + S, b_lo, b_hi);
  stage_row(0, a_lo, a_hi, a_col);
  load_batch(b_lo, b_hi, b_col, b_q, b_v);
  load_rp(i + 2 * S, c_lo, c_hi);
  int s = 0;
  for (; i < n; i += S, s ^= 1) {
    stage_row(s ^ 1, b_lo, b_hi, b_col);         // row B -> the other stage
    int c_col, c_q;
    T c_v;
    uint32_t d_lo, d_hi;
    load_batch(c_lo, c_hi, c_col, c_q, c_v);    // row C, first batch
    load_rp(i + 3 * S, d_lo, d_hi);             // row D
    const int64_t idx = i * R + r0;
    // own-row operands, issued before the gather
    T xi[VW], xn[VW];
    if constexpr (MODE == MODE_DOCH) {
      if (lane_on && any_run) vload<T, VW>(xc + idx, xi);
      if (lane_on && (any_copy || !all_run)) vload<T, VW>(xn_buf + idx, xn);  // x_{p-1} (still held)
    } else if constexpr (MODE == MODE_ADOCH_X) {
      if (lane_on && any_run) vload<T, VW>(xc + idx, xi);
    }
    T acc[VW];
    EsRow<VK, T> es[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) acc[v] = T(0);
    const uint32_t deg = a_hi - a_lo;
    if constexpr (G > 0) {
      if (!tma) {
        cp_async_wait1();  // row A's stage has landed (row B's may still be in flight)
      } else if (deg > 0) {
        const uint32_t mb = mb0 + 8u * s, par = (bar_par >> s) & 1u;
        asm volatile(
            "{\n.reg .pred P1;\nRVW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra RVW;\n}\n" ::"r"(mb),
            "r"(par)
            : "memory");
        bar_par ^= 1u << s;
      }
      const uint32_t sa = st_base + s * ST_STRIDE;
#pragma unroll
      for (int k = 0; k < G; k += UNROLL) {
        if (k >= deg) break;
        T xg[UNROLL][VW];
        T vv[UNROLL];
        int qq[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const int kk = k + u;
          const bool real = kk < deg;
          edge_value(kk, real, a_q, a_v, qq[u], vv[u]);  // padding: weight 0
          // padding slots hold finite stale values (zero-initialised above)
          vload<T, VW>(reinterpret_cast<const T*>(stage_mem + (sa + kk * 32 * CB - smem_u32(stage_mem))), xg[u]);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
          for (int v = 0; v < VW; ++v) {
            acc[v] = madd(acc[v], vv[u], xg[u][v]);
            es[v].add(qq[u], float(qq[u]), vv[u], xg[u][v]);
          }
        }
      }
    }
    // edges past the staged ones: gathered directly, UNROLL at a time
    for (uint32_t base = a_lo, k0 = G; base < a_hi; base += 32, k0 = 0) {
      const int cnt = int(min(32u, a_hi - base));
      if (int(k0) >= cnt) continue;
      int mycol = a_col, myq = a_q;
      T myv = a_v;
      if (base != a_lo) load_batch(base, a_hi, mycol, myq, myv);
      for (int k = k0; k < cnt; k += UNROLL) {
        T xg[UNROLL][VW];
        T vv[UNROLL];
        int qq[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const int kk = k + u;  // uniform across the warp
          const bool real = kk < cnt;
          const uint32_t j = uint32_t(__shfl_sync(0xffffffffu, mycol, kk & 31));
          edge_value(kk, real, myq, myv, qq[u], vv[u]);
#pragma unroll
          for (int v = 0; v < VW; ++v) xg[u][v] = T(0);
          if (real && lane_on) {
            const size_t off = size_t(j) * rowb;
            if constexpr (MODE == MODE_ADOCH_Y) {
              T a0[VW], a1[VW];
              vload<T, VW>(reinterpret_cast<const T*>(xcb + off), a0);
              vload<T, VW>(reinterpret_cast<const T*>(xpb + off), a1);
#pragma unroll
              for (int v = 0; v < VW; ++v) xg[u][v] = extrap(a0[v], a1[v], cm[v]);
            } else {
              vload<T, VW>(reinterpret_cast<const T*>(xcb + off), xg[u]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
          for (int v = 0; v < VW; ++v) {
            acc[v] = madd(acc[v], vv[u], xg[u][v]);
            if constexpr (MODE != MODE_ADOCH_Y) es[v].add(qq[u], float(qq[u]), vv[u], xg[u][v]);
          }
        }
      }
    }
    a_lo = b_lo; a_hi = b_hi; a_col = b_col; a_q = b_q; a_v = b_v;
    b_lo = c_lo; b_hi = c_hi; b_col = c_col; b_q = c_q; b_v = c_v;
    c_lo = d_lo; c_hi = d_hi;
    if (!lane_on) continue;
    if constexpr (MODE == MODE_DOCH) {
      if (!any_run) {  // stopped replicas: only the pending best-spin copy
        if (any_copy) {
#pragma unroll
          for (int v = 0; v < VW; ++v)
            if (copy[v]) a.best[idx + v] = xn[v] >= T(0) ? 1 : -1;
        }
        continue;
      }
      if (any_copy) {
#pragma unroll
        for (int v = 0; v < VW; ++v)
          if (copy[v]) a.best[idx + v] = xn[v] >= T(0) ? 1 : -1;
      }
      // branch-free over the lane's replicas (so they interleave); partials of
      // stopped replicas are accumulated but never read (reduce_control skips them)
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const T ax = shifted(acc[v], alpha[v], xi[v]);
        const T x2 = mul_rn(xi[v], xi[v]);
        s4[v] += x2 * x2;
        sxax[v] += xi[v] * ax;
        if (es32) {
          esf[v] += __uint_as_float(__float_as_uint(float(es[v].value(deg))) ^ (negbit(xi[v]) << 31));
        } else {
          const double e = es[v].value(deg);
          esum[v] += negbit(xi[v]) ? -e : e;
        }
        const T xnew = tmap_pass(ax, beta[v], ibeta[v]);
        step[v] = fmax(step[v], fabs(xnew - xi[v]));
        xn[v] = run[v] ? xnew : xn[v];
      }
      vstore<T, VW>(xn_buf + idx, xn);
      if (a.states && p < a.cfg.max_iters) vstore<T, VW>(reinterpret_cast<T*>(a.states) + (int64_t)(p + 1) * n * R + idx, xn);
    } else if constexpr (MODE == MODE_ADOCH_X) {
      if (!any_run) continue;
      T ax[VW];
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        ax[v] = shifted(acc[v], alpha[v], xi[v]);
        const T x2 = mul_rn(xi[v], xi[v]);
        s4[v] += x2 * x2;
        sxax[v] += xi[v] * ax[v];
        if (es32) {
          esf[v] += __uint_as_float(__float_as_uint(float(es[v].value(deg))) ^ (negbit(xi[v]) << 31));
        } else {
          const double e = es[v].value(deg);
          esum[v] += negbit(xi[v]) ? -e : e;
        }
      }
      vstore<T, VW>(reinterpret_cast<T*>(a.ax[p & 1]) + idx, ax);
      if (p > 0 && a.cfg.window_mode == DCX_WINDOW_ECONOMY) {
        T xq[VW], axq[VW];
        vload<T, VW>(xp + idx, xq);
        vload<T, VW>(reinterpret_cast<const T*>(a.ax[(p + 1) & 1]) + idx, axq);
#pragma unroll
        for (int v = 0; v < VW; ++v) {
          const T yi = extrap(xi[v], xq[v], cm[v]);
          const T ayi = extrap(ax[v], axq[v], cm[v]);
          const T y2 = mul_rn(yi, yi);
          sy4[v] += y2 * y2;
          syay[v] += yi * ayi;
        }
      }
    } else {  // MODE_ADOCH_Y: acc = J y
      if (!any_run) continue;
      T xq[VW], ay[VW];
      vload<T, VW>(xc + idx, xi);
      vload<T, VW>(xp + idx, xq);
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const T yi = extrap(xi[v], xq[v], cm[v]);
        ay[v] = shifted(acc[v], alpha[v], yi);
        const T y2 = yi * yi;
        sy4[v] += y2 * y2;
        syay[v] += yi * ay[v];
      }
      vstore<T, VW>(reinterpret_cast<T*>(a.ay) + idx, ay);
    }
  }
  if constexpr (G > 0) cp_async_wait0();

  // block reduction of the per-replica partials, warps in a fixed order
  __shared__ double red[NQ][32 * VW];
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const int c = lane * VW + v;
        const double q[NQ] = {double(s4[v]), double(sxax[v]), es32 ? double(esf[v]) : esum[v], double(step[v]),
                              double(sy4[v]), double(syay[v])};
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          if (w == 0) red[k][c] = q[k];
          else red[k][c] = (k == Q_STEP) ? fmax(red[k][c], q[k]) : red[k][c] + q[k];
        }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < NQ * 32 * VW; t += blockDim.x) {
    const int k = t / (32 * VW), c = t % (32 * VW);
    const int r = blockIdx.y * 32 * VW + c;
    if (r < R) a.part[((int64_t)r * NQ + k) * a.slots + blockIdx.x] = red[k][c];
  }
}

// ---------------------------------------------------------------------------
// 2-D periodic lattice (BASELINE configs[2], T6): stencil pass, R > 1, f32.
// Replaces pass_rv when the coupling was recognised at upload as the L x L torus
// of SURVEY.md Appendix A (every row i = (a, b) holds exactly its four lattice
// neighbours, +-q bonds): no row pointers, no column indices -- the neighbours
// are computed, the bonds come from two int8 arrays (q(i, right(i)), q(i, down(i))),
// and a warp moves whole 512-byte replica rows (32 lanes x float4) of the site
// and its four neighbours, for SITES sites at once so 5 * SITES 16-byte loads
// per lane are in flight. The row sum runs over the neighbours in ascending
// column order with the same FMA and epilogue as pass_rv, so the iterates are
// bit-identical to it. The spin energy of the pass is accumulated per replica
// over FORWARD edges only: sum_i s_i (J s)_i = 2 sum_i (q_r(i) s_i s_right + q_d(i)
// s_i s_down), exact as an integer count of negative products.


__device__ __forceinline__ void sort4_cols(int64_t (&c)[4], int (&k)[4]) {
  // 5-comparator network on (column, slot); columns are distinct for L >= 3
  auto cx = [&](int i, int j) {
    if (c[j] < c[i]) {
      const int64_t t = c[i]; c[i] = c[j]; c[j] = t;
      const int u = k[i]; k[i] = k[j]; k[j] = u;
    }
  };
  cx(0, 1); cx(2, 3); cx(0, 2); cx(1, 3); cx(1, 2);
}

template <int MODE>
#ifndef DCX_TORUS_MINB
#define DCX_TORUS_MINB 2
#endif
#ifndef DCX_TORUS_THREADS
#define DCX_TORUS_THREADS 256
#endif
__global__ void __launch_bounds__(DCX_TORUS_THREADS, DCX_TORUS_MINB) pass_torus(PassArgs a) {
  using T = float;
  constexpr int VW = 4;
  static_assert(MODE != MODE_ADOCH_Y, "exact-window ADOCH stays on pass_rv");
  if (!a.g->live) return;
  const int p = a.g->p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = a.cfg.R;
  const int n = int(a.cfg.n);  // L <= 46340 and n * R / 4 < 2^31 (checked at launch): 32-bit offsets
  const int L = a.torus_L;
  const int r0 = blockIdx.y * 32 * VW + lane * VW;
  const bool lane_on = r0 < R;
  T alpha[VW], beta[VW], ibeta[VW], cm[VW];
  bool run[VW], copy[VW];
  bool any_run = false, all_run = true, any_copy = false;
#pragma unroll
  for (int v = 0; v < VW; ++v) {
    run[v] = copy[v] = false;
    alpha[v] = beta[v] = cm[v] = T(0);
    ibeta[v] = T(1);
    if (lane_on) {
      const RepCtl& c = a.ctl[r0 + v];
      run[v] = c.status == DCX_STOP_RUNNING;
      copy[v] = MODE == MODE_DOCH && p > 0 && c.pend == p - 1;
      alpha[v] = T(c.alpha);
      beta[v] = T(c.beta);
      ibeta[v] = inv_beta(beta[v]);
      cm[v] = T(c.cm[p & 1]);
    }
    any_run |= run[v];
    all_run &= run[v];
    any_copy |= copy[v];
  }
  if (!__syncthreads_or(any_run || any_copy)) return;
  // float4 views: a spin's replica row is R / 4 float4; this lane's column is r0 / 4
  const int RV = R / VW, c4 = r0 / VW;
  const float4* xc = reinterpret_cast<const float4*>(a.x[p & 1]) + c4;
  const float4* xp = reinterpret_cast<const float4*>(a.x[(p + 1) & 1]) + c4;
  float4* xn_buf = reinterpret_cast<float4*>(a.x[(p + 1) & 1]) + c4;
  const T scale = T(a.scale);
  T s4[VW], sxax[VW], sy4[VW], syay[VW], step[VW];
  int neg[VW], nedge = 0;  // forward-edge products q s_i s_j < 0, and forward edges counted
#pragma unroll
  for (int v = 0; v < VW; ++v) {
    s4[v] = sxax[v] = sy4[v] = syay[v] = step[v] = T(0);
    neg[v] = 0;
  }
  // site (ar, b) of this warp, advanced by S = grid * 8 sites per step without divisions
  const int NW = int(blockDim.x >> 5);
  const int S = int(gridDim.x) * NW;
  const int Sa = S / L, Sb = S - Sa * L;
  int i_cur = int(blockIdx.x) * NW + warp;
  int a_cur = i_cur / L, b_cur = i_cur - a_cur * L;
  auto advance = [&](int& i, int& ar, int& b) {
    i += S;
    ar += Sa;
    b += Sb;
    if (b >= L) { b -= L; ++ar; }
  };
  auto f4 = [](const float4& q, int v) { return v == 0 ? q.x : v == 1 ? q.y : v == 2 ? q.z : q.w; };
  // two register stages: the loads of the next site are in flight while this one computes
  struct Stage {
    float4 xs[5];  // 0 = own row, 1..4 = neighbours in ascending column order
    float4 xo, axo;
    T qv[4];
    uint32_t qr, qd;
    int slot_r, slot_d, isite;
    bool on;
  };
  auto load_stage = [&](Stage& st, const int iu, const int au, const int bu) {
      st.on = iu < n;
      st.isite = iu;
      const int ii = st.on ? iu : 0, ar = st.on ? au : 0, b = st.on ? bu : 0;
      const int c_up = ar == 0 ? ii + (L - 1) * L : ii - L;
      const int c_left = b == 0 ? ii + L - 1 : ii - 1;
      const int c_right = b == L - 1 ? ii - L + 1 : ii + 1;
      const int c_down = ar == L - 1 ? ii - (L - 1) * L : ii + L;
      const int q_up = __ldg(a.bond_d + c_up), q_left = __ldg(a.bond_r + c_left), q_right = __ldg(a.bond_r + ii),
                q_down = __ldg(a.bond_d + ii);
      st.qr = q_right < 0 ? 0x80000000u : 0u;
      st.qd = q_down < 0 ? 0x80000000u : 0u;
      int col[4];
      // ascending column order: interior (and most border) sites up < left < right < down;
      // the wrapped ones are sorted (warp-uniform branch)
      if (c_up < c_left && c_left < c_right && c_right < c_down) {
        col[0] = c_up; col[1] = c_left; col[2] = c_right; col[3] = c_down;
        st.qv[0] = scale * T(q_up); st.qv[1] = scale * T(q_left); st.qv[2] = scale * T(q_right);
        st.qv[3] = scale * T(q_down);
        st.slot_r = 2;
        st.slot_d = 3;
      } else {
        int64_t cc[4] = {c_up, c_left, c_right, c_down};
        int k[4] = {0, 1, 2, 3};
        sort4_cols(cc, k);
        const int qs[4] = {q_up, q_left, q_right, q_down};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          col[m] = int(cc[m]);
          const int km = k[m];
          st.qv[m] = scale * T(km == 0 ? qs[0] : km == 1 ? qs[1] : km == 2 ? qs[2] : qs[3]);
          if (km == 2) st.slot_r = m;
          if (km == 3) st.slot_d = m;
        }
      }
      const bool ld = st.on && lane_on;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      st.xs[0] = (ld && any_run) ? __ldg(xc + ii * RV) : z;
#pragma unroll
      for (int m = 0; m < 4; ++m) st.xs[1 + m] = (ld && any_run) ? __ldg(xc + col[m] * RV) : z;
      st.xo = st.axo = z;
      if constexpr (MODE == MODE_DOCH) {
        // the pending copy reads the sign words of x_{p-1} (1 bit per replica), not x_{p-1}
        if (ld && any_copy) {
          const uint32_t* sw = a.sgnw[(p + 1) & 1] + int64_t(ii) * (4 * gridDim.y) + blockIdx.y * 4;
          st.xo = make_float4(__uint_as_float(__ldg(sw)), __uint_as_float(__ldg(sw + 1)),
                              __uint_as_float(__ldg(sw + 2)), __uint_as_float(__ldg(sw + 3)));
        }
      } else {
        if (ld && any_run && p > 0 && a.cfg.window_mode == DCX_WINDOW_ECONOMY) {
          st.xo = __ldg(xp + ii * RV);
          st.axo = __ldg(reinterpret_cast<const float4*>(a.ax[(p + 1) & 1]) + c4 + ii * RV);
        }
      }
  };
  auto compute_stage = [&](const Stage& st) {
      if (!st.on || !lane_on) return;
      const int ofs = st.isite * RV;
      if constexpr (MODE == MODE_DOCH) {
        if (any_copy) {  // pending best copy: sign(x_{p-1}) of the copying replicas, one 32-bit store
          uint32_t* bp = reinterpret_cast<uint32_t*>(a.best + int64_t(st.isite) * R + r0);
          uint32_t w = *bp;
#pragma unroll
          for (int v = 0; v < VW; ++v)
            if (copy[v]) {
              const uint32_t negb = (__float_as_uint(f4(st.xo, v)) >> lane) & 1u;  // word v, bit lane
              w = (w & ~(0xffu << (8 * v))) | ((negb ? 0xffu : 0x01u) << (8 * v));
            }
          *bp = w;
        }
        // sign words of x_p for the copy of pass p + 1 (x is never -0.0: sign bit <=> x < 0)
        const unsigned am = __activemask();
        uint32_t bw[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) bw[v] = __ballot_sync(am, __float_as_uint(f4(st.xs[0], v)) >> 31);
        const bool wany = __any_sync(am, any_run);  // every lane of am votes (no short-circuit)
        if (lane < VW && wany)
          a.sgnw[p & 1][int64_t(st.isite) * (4 * gridDim.y) + blockIdx.y * 4 + lane] =
              lane == 0 ? bw[0] : lane == 1 ? bw[1] : lane == 2 ? bw[2] : bw[3];
      }
      if (!any_run) return;
      T xi[VW], acc[VW];
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        xi[v] = f4(st.xs[0], v);
        acc[v] = T(0);
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[v] = madd(acc[v], st.qv[m], f4(st.xs[1 + m], v));
      }
      nedge += 2;
      const float4 xr = st.slot_r == 2 ? st.xs[3] : st.slot_r == 0 ? st.xs[1] : st.slot_r == 1 ? st.xs[2] : st.xs[4];
      const float4 xd = st.slot_d == 3 ? st.xs[4] : st.slot_d == 0 ? st.xs[1] : st.slot_d == 1 ? st.xs[2] : st.xs[3];
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const uint32_t xb = __float_as_uint(xi[v]);
        neg[v] += int((xb ^ __float_as_uint(f4(xr, v)) ^ st.qr) >> 31) + int((xb ^ __float_as_uint(f4(xd, v)) ^ st.qd) >> 31);
      }
      if constexpr (MODE == MODE_DOCH) {
        T xn[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) {
          const T ax = shifted(acc[v], alpha[v], xi[v]);
          const T x2 = mul_rn(xi[v], xi[v]);
          s4[v] += x2 * x2;
          sxax[v] += xi[v] * ax;
          const T xnew = tmap_pass(ax, beta[v], ibeta[v]);
          step[v] = fmax(step[v], fabs(xnew - xi[v]));
          xn[v] = xnew;
        }
        const float4 o4 = make_float4(xn[0], xn[1], xn[2], xn[3]);
        if (all_run) {
          xn_buf[ofs] = o4;
        } else {  // stopped replicas keep their x_{p-1} in this buffer: store the running ones only
          float* e = reinterpret_cast<float*>(xn_buf + ofs);
#pragma unroll
          for (int v = 0; v < VW; ++v)
            if (run[v]) e[v] = xn[v];
        }
        if (a.states && p < a.cfg.max_iters) {
          float* st = reinterpret_cast<float*>(reinterpret_cast<float4*>(a.states) + (int64_t)(p + 1) * n * RV + c4 + ofs);
#pragma unroll
          for (int v = 0; v < VW; ++v) st[v] = run[v] ? xn[v] : reinterpret_cast<const float*>(xn_buf + ofs)[v];
        }
      } else {  // MODE_ADOCH_X
        T ax[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) {
          ax[v] = shifted(acc[v], alpha[v], xi[v]);
          const T x2 = mul_rn(xi[v], xi[v]);
          s4[v] += x2 * x2;
          sxax[v] += xi[v] * ax[v];
        }
        reinterpret_cast<float4*>(a.ax[p & 1])[c4 + ofs] = make_float4(ax[0], ax[1], ax[2], ax[3]);
        if (p > 0 && a.cfg.window_mode == DCX_WINDOW_ECONOMY) {
#pragma unroll
          for (int v = 0; v < VW; ++v) {
            const T yi = extrap(xi[v], f4(st.xo, v), cm[v]);
            const T ayi = extrap(ax[v], f4(st.axo, v), cm[v]);
            const T y2 = mul_rn(yi, yi);
            sy4[v] += y2 * y2;
            syay[v] += yi * ayi;
          }
        }
      }
  };
#if DCX_TORUS_MINB > 2 || DCX_TORUS_THREADS > 256
  // one register stage, more resident warps (latency hidden across warps)
  for (;;) {
    Stage sa;
    load_stage(sa, i_cur, a_cur, b_cur);
    if (!sa.on) break;
    compute_stage(sa);
    advance(i_cur, a_cur, b_cur);
  }
#else
  Stage sa, sb;
  load_stage(sa, i_cur, a_cur, b_cur);
  while (sa.on) {
    advance(i_cur, a_cur, b_cur);
    load_stage(sb, i_cur, a_cur, b_cur);
    compute_stage(sa);
    if (!sb.on) break;
    advance(i_cur, a_cur, b_cur);
    load_stage(sa, i_cur, a_cur, b_cur);
    compute_stage(sb);
  }
#endif
  // block reduction of the per-replica partials, warps in a fixed order (as pass_rv)
  __shared__ double red[NQ][32 * VW];
  for (int w = 0; w < NW; ++w) {
    if (warp == w) {
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const int c = lane * VW + v;
        // sum over this warp's sites of s_i (J s)_i = 2 * (forward edges - 2 * negative ones)
        const double es = 2.0 * double(nedge - 2 * neg[v]);
        const double q[NQ] = {double(s4[v]), double(sxax[v]), es, double(step[v]), double(sy4[v]), double(syay[v])};
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          if (w == 0) red[k][c] = q[k];
          else red[k][c] = (k == Q_STEP) ? fmax(red[k][c], q[k]) : red[k][c] + q[k];
        }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < NQ * 32 * VW; t += blockDim.x) {
    const int k = t / (32 * VW), c = t % (32 * VW);
    const int r = blockIdx.y * 32 * VW + c;
    if (r < R) a.part[((int64_t)r * NQ + k) * a.slots + blockIdx.x] = red[k][c];
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
      const T xn = tmap_pass(av, beta, inv_beta(beta));
      xo[i] = xn;
      if (a.states && p < a.cfg.max_iters) reinterpret_cast<T*>(a.states)[(int64_t)(p + 1) * total + i] = xn;
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
    const T xn = tmap_pass(av, beta, inv_beta(beta));
    xo[idx] = xn;
    if (a.states && p < a.cfg.max_iters) reinterpret_cast<T*>(a.states)[(int64_t)(p + 1) * total + idx] = xn;
    st = fmax(st, double(fabs(xn - xi)));
  }
  spart[(tid / R) * R + r] = st;  // slot = tid / R, replica-minor
}

// ---------------------------------------------------------------------------
// Reduce + control: block r reduces replica r's partial slots in a fixed order
// (deterministic for a fixed launch shape), then thread 0 runs the control.
// phase: 0 = DOCH pass, 1 = ADOCH bookkeeping (+decision if economy),
//        2 = ADOCH exact decision only.
// dist: 0 = single context; 1 = reduce only, totals to qs (sums) / qm (maxima and
// elapsed time) for the caller's all-reduce; 2 = control only, from the reduced
// qs / qm (every rank then takes identical decisions, including the time budget:
// the elapsed time is the maximum over ranks).
__global__ void __launch_bounds__(256) reduce_control(PassArgs a, const double* spart, int sslots, int phase,
                                                      int last_kernel, int dist, double* qs, double* qm) {
  if (!a.g->live) return;
  const int p = a.g->p;
  const int r = blockIdx.x;
  const int R = a.cfg.R;
  __shared__ double red[NQ][256];
  __shared__ double tot[NQ + 1];
  RepCtl* cp = a.ctl + r;
  const bool running = cp->status == DCX_STOP_RUNNING;
  if (running && dist == 2) {
    if (threadIdx.x == 0) {
      const double* s = qs + (int64_t)r * DCX_QSUM;
      const double* m = qm + (int64_t)r * DCX_QMAX;
      tot[Q_S4] = s[0];
      tot[Q_SXAX] = s[1];
      tot[Q_ES] = s[2];
      tot[Q_SY4] = s[3];
      tot[Q_SYAY] = s[4];
      tot[Q_STEP] = m[0];
      tot[NQ] = m[1];
      RepCtl c = *cp;
      const double now = m[2];
      bool stopped = false;
      if (phase == 0) {
        stopped = control_after_pass(c, a.cfg, r, tot, p, now);
        c.step = tot[Q_STEP];
      } else {
        if (p > 0) c.step = tot[NQ];
        stopped = control_after_pass(c, a.cfg, r, tot, p, now);
        if (!stopped && a.cfg.window_mode == DCX_WINDOW_ECONOMY) adoch_decide(c, a.cfg, r, tot, p);
      }
      *cp = c;
      if (stopped) atomicSub(&a.g->running, 1);
    }
  } else if (running) {
    // each thread folds slots t, t + 256, ... in increasing order; the loads of
    // eight slots and all NQ quantities are issued before the folds (one L2
    // round trip per 8 x NQ slots instead of one per slot; same order, same bits)
    constexpr int U = 8;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    const double* src = a.part + (int64_t)r * NQ * a.slots;
    for (int s0 = threadIdx.x; s0 < a.slots; s0 += U * blockDim.x) {
      double v[NQ][U];
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int s = s0 + u * blockDim.x;
          v[q][u] = s < a.slots ? src[(int64_t)q * a.slots + s] : 0.0;  // 0: identity of + and of the step max
        }
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (s0 + u * blockDim.x >= a.slots) break;
          acc[q] = (q == Q_STEP) ? fmax(acc[q], v[q][u]) : acc[q] + v[q][u];
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) red[q][threadIdx.x] = acc[q];
    double st = 0.0;
    if (spart) {
      for (int s0 = threadIdx.x; s0 < sslots; s0 += 8 * blockDim.x) {  // eight loads in flight (max: any order)
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int s = s0 + u * blockDim.x;
          v[u] = s < sslots ? spart[(int64_t)s * R + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) st = fmax(st, v[u]);
      }
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
    if (threadIdx.x == 0 && dist == 1) {
      double* s = qs + (int64_t)r * DCX_QSUM;
      double* m = qm + (int64_t)r * DCX_QMAX;
      s[0] = red[Q_S4][0];
      s[1] = red[Q_SXAX][0];
      s[2] = red[Q_ES][0];
      s[3] = red[Q_SY4][0];
      s[4] = red[Q_SYAY][0];
      m[0] = red[Q_STEP][0];
      m[1] = sred[0];
      m[2] = double(globaltimer() - a.g->t0) * 1e-9;
    } else if (threadIdx.x == 0) {
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
    // not yet copied by a pass: pend > the copy iterate of the last pass (x_P; with three
    // buffers also x_{P-1}), both still in their buffers
    if (pe >= 0 && pe > copy_iter(a, P)) a.best[idx] = reinterpret_cast<const T*>(a.x[xslot(a, pe)])[idx] >= T(0) ? 1 : -1;
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
template <typename T, int VK, int VW, int MODE>
static void launch_rv_mode(const PassArgs& a, dim3 grid, cudaStream_t s) {
  constexpr size_t smem = rv_smem_bytes<T, VW, MODE>();
  static unsigned long long opted = 0;  // devices this instantiation opted in on
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && !((opted >> (dev & 63)) & 1ull)) {
    cudaFuncSetAttribute(pass_rv<T, VK, VW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    opted |= 1ull << (dev & 63);
  }
  pass_rv<T, VK, VW, MODE><<<grid, 256, smem, s>>>(a);
}
template <typename T, int VK, int VW>
static void launch_rv(int mode, const PassArgs& a, dim3 grid, cudaStream_t s) {
  switch (mode) {
    case MODE_DOCH: launch_rv_mode<T, VK, VW, MODE_DOCH>(a, grid, s); break;
    case MODE_ADOCH_X: launch_rv_mode<T, VK, VW, MODE_ADOCH_X>(a, grid, s); break;
    default: launch_rv_mode<T, VK, VW, MODE_ADOCH_Y>(a, grid, s); break;
  }
}

// replicas per lane of the R > 1 kernel
// f32 replica vector width (4, or 2 with DCX_RV_VW=2: fewer registers per lane,
// three resident blocks per SM)
static int rv_vw_f32() {
  static const int w = [] {
    const char* e = std::getenv("DCX_RV_VW");
    return (e && std::atoi(e) == 2) ? 2 : 4;
  }();
  return w;
}

int replica_vector_width(int R, bool f64) {
  const int w = f64 ? 2 : rv_vw_f32();
  return R % w == 0 ? w : 1;
}

// the lattice stencil pass for recognised tori: opt-in (DCX_TORUS=1). It is bit-identical
// to pass_rv but measured slower on T6 (1.59 vs 1.41 ms per iteration):
// register-staged neighbour rows hide less latency than pass_rv's TMA staging into
// shared memory. Read per launch so one process can A/B both kernels (tests).
static bool use_torus() {
  const char* e = std::getenv("DCX_TORUS");
  return e && std::atoi(e) == 1;
}

// the entry-parallel R = 1 pass for f32 integer couplings (DCX_R1W=0 falls back to pass_r1)
static bool use_r1w() {
  static const bool on = [] {
    const char* e = std::getenv("DCX_R1W");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

template <typename T, int VK>
static void launch_pass_vk(int mode, const PassArgs& a, int V, int grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4 && (VK == VK_UNIFORM || VK == VK_I8)) {
    if (a.cfg.R == 1 && a.chunks.C > 0 && mode != MODE_ADOCH_Y) {
      launch_chunked_pass(mode, VK, a, grid, s);
      return;
    }
    if (a.cfg.R == 1 && use_r1w()) {
      switch (mode) {
        case MODE_DOCH: pass_r1w<VK, MODE_DOCH><<<grid, 256, 0, s>>>(a); break;
        case MODE_ADOCH_X: pass_r1w<VK, MODE_ADOCH_X><<<grid, 256, 0, s>>>(a); break;
        default: pass_r1w<VK, MODE_ADOCH_Y><<<grid, 256, 0, s>>>(a); break;
      }
      return;
    }
  }
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
    const int W = replica_vector_width(R, sizeof(T) == 8);
    if constexpr (sizeof(T) == 4 && VK == VK_I8) {
      if (a.torus_L > 0 && W == 4 && mode != MODE_ADOCH_Y && use_torus() && a.cfg.n * R / 4 < (int64_t(1) << 31)) {
        const dim3 g(grid, (R + 127) / 128);
        if (mode == MODE_DOCH) pass_torus<MODE_DOCH><<<g, DCX_TORUS_THREADS, 0, s>>>(a);
        else pass_torus<MODE_ADOCH_X><<<g, DCX_TORUS_THREADS, 0, s>>>(a);
        return;
      }
    }
    if constexpr (sizeof(T) == 8) {
      if (W == 2) launch_rv<T, VK, 2>(mode, a, dim3(grid, (R + 63) / 64), s);
      else launch_rv<T, VK, 1>(mode, a, dim3(grid, (R + 31) / 32), s);
    } else {
      if (W == 4) launch_rv<T, VK, 4>(mode, a, dim3(grid, (R + 127) / 128), s);
      else if (W == 2) launch_rv<T, VK, 2>(mode, a, dim3(grid, (R + 63) / 64), s);
      else launch_rv<T, VK, 1>(mode, a, dim3(grid, (R + 31) / 32), s);
    }
  }
}

template <typename T>
static void launch_pass_t(int mode, const PassArgs& a, int vk, int V, int grid, cudaStream_t s) {
  if (vk == VK_PROC) {
    launch_proc_pass<T>(mode, a, grid, s);
    return;
  }
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
  if (J.vk == VK_PROC) {
    launch_proc_apply<T>(J.n, J.proc_seed, v, R, jv, es, s);
    return;
  }
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
    reduce_control<<<a.cfg.R, 256, 0, s>>>(a, nullptr, 0, 0, 1, 0, nullptr, nullptr);
    return;
  }
  if (f64) launch_pass_t<double>(MODE_ADOCH_X, a, m.vk, m.V, m.grid, s);
  else launch_pass_t<float>(MODE_ADOCH_X, a, m.vk, m.V, m.grid, s);
  reduce_control<<<a.cfg.R, 256, 0, s>>>(a, m.spart, sslots, 1, 0, 0, nullptr, nullptr);
  if (a.cfg.window_mode == DCX_WINDOW_EXACT) {
    if (f64) launch_pass_t<double>(MODE_ADOCH_Y, a, m.vk, m.V, m.grid, s);
    else launch_pass_t<float>(MODE_ADOCH_Y, a, m.vk, m.V, m.grid, s);
    reduce_control<<<a.cfg.R, 256, 0, s>>>(a, nullptr, 0, 2, 0, 0, nullptr, nullptr);
  }
  if (f64) adoch_finalize<double><<<m.fgrid, 256, 0, s>>>(a, m.spart, sslots);
  else adoch_finalize<float><<<m.fgrid, 256, 0, s>>>(a, m.spart, sslots);
  advance_pass<<<1, 1, 0, s>>>(a.g);
}

void enqueue_dist_pass(const MultiPass& m, double* qs, double* qm, cudaStream_t s) {
  const PassArgs& a = m.args;
  const bool doch = m.solver == DCX_SOLVER_DOCH;
  const int mode = doch ? MODE_DOCH : MODE_ADOCH_X;
  if (m.f64) launch_pass_t<double>(mode, a, m.vk, m.V, m.grid, s);
  else launch_pass_t<float>(mode, a, m.vk, m.V, m.grid, s);
  reduce_control<<<a.cfg.R, 256, 0, s>>>(a, doch ? nullptr : m.spart, doch ? 0 : m.sslots, doch ? 0 : 1, 0, 1, qs, qm);
}

// The pass over own rows [lo, hi) only (the interior / boundary split of the exchange
// overlap): every row-indexed pointer moves to row lo; the gather source
// (gx, the whole local + halo space) does not. Partials go to slot half `half` of the 2 x grid
// slots a row-partitioned run allocates; enqueue_dist_reduce folds both halves.
void enqueue_dist_pass_rows(const MultiPass& m, int64_t lo, int64_t hi, int half, cudaStream_t s) {
  PassArgs a = m.args;
  const int64_t R = a.cfg.R;
  const size_t tb = m.f64 ? 8 : 4;
  auto shift = [&](void* p) { return p ? static_cast<void*>(static_cast<char*>(p) + size_t(lo) * R * tb) : p; };
  a.rp += lo;
  a.x[0] = shift(a.x[0]);
  a.x[1] = shift(a.x[1]);
  a.ax[0] = shift(a.ax[0]);
  a.ax[1] = shift(a.ax[1]);
  a.ay = shift(a.ay);
  a.best += lo * R;
  a.cfg.n = hi - lo;
  a.part += int64_t(half) * (a.slots / 2);
  const int mode = m.solver == DCX_SOLVER_DOCH ? MODE_DOCH : MODE_ADOCH_X;
  if (m.f64) launch_pass_t<double>(mode, a, m.vk, m.V, m.grid, s);
  else launch_pass_t<float>(mode, a, m.vk, m.V, m.grid, s);
}

void enqueue_dist_reduce(const MultiPass& m, double* qs, double* qm, cudaStream_t s) {
  const PassArgs& a = m.args;
  const bool doch = m.solver == DCX_SOLVER_DOCH;
  reduce_control<<<a.cfg.R, 256, 0, s>>>(a, doch ? nullptr : m.spart, doch ? 0 : m.sslots, doch ? 0 : 1, 0, 1, qs, qm);
}

void enqueue_dist_control(const MultiPass& m, const double* qs, const double* qm, cudaStream_t s) {
  const PassArgs& a = m.args;
  double* q0 = const_cast<double*>(qs);
  double* q1 = const_cast<double*>(qm);
  if (m.solver == DCX_SOLVER_DOCH) {
    reduce_control<<<a.cfg.R, 256, 0, s>>>(a, nullptr, 0, 0, 1, 2, q0, q1);
    return;
  }
  reduce_control<<<a.cfg.R, 256, 0, s>>>(a, nullptr, 0, 1, 0, 2, q0, q1);
  if (m.f64) adoch_finalize<double><<<m.fgrid, 256, 0, s>>>(a, m.spart, m.sslots);
  else adoch_finalize<float><<<m.fgrid, 256, 0, s>>>(a, m.spart, m.sslots);
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
