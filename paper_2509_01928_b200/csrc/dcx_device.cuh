// Device-side building blocks shared by every DOCH/ADOCH kernel.
//
// The per-replica control logic (`control_after_pass`, `adoch_decide`) is the
// single device restatement of the reference loop bookkeeping
// (dc/solvers/doch.py:199-232 for DOCH, :294-342 for ADOCH; best tracking
// dc/solvers/common.py:70-91). The multi-pass CSR path, the persistent small-n
// kernel and the dense path all call it, so the semantics live in one place.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/dcx.h"

namespace dcx {

// ---------------------------------------------------------------- value kinds
// Coupling values are stored in the narrowest exact form.
// VK_PROC: procedural J_ij = sin(i*j + seed), generated on the fly (dcx_proc.cu)
enum ValueKind : int { VK_UNIFORM = 0, VK_I8 = 1, VK_I16 = 2, VK_F32 = 3, VK_F64 = 4, VK_PROC = 5 };

// partial-sum slots (per warp slot, per replica)
enum : int { Q_S4 = 0, Q_SXAX = 1, Q_ES = 2, Q_STEP = 3, Q_SY4 = 4, Q_SYAY = 5, NQ = 6 };

enum Mode : int { MODE_DOCH = 0, MODE_ADOCH_X = 1, MODE_ADOCH_Y = 2 };

struct RepCtl {
  double alpha, beta;
  double h;        // H(x_k)
  double best;     // best recorded energy
  double step;     // ||x_{k+1} - x_k||_inf produced by the last update
  double t;        // ADOCH Nesterov t_k
  double cm[2];    // ADOCH momentum coefficient c_p, indexed by pass parity
  double wmax;     // max over the whole window while it has not evicted
  int32_t k;       // iterations completed
  int32_t status;  // DCX_STOP_*
  int32_t best_iter;
  int32_t pend;    // iteration whose sign(x) must become the best spins (-1: none)
  int32_t accept;  // ADOCH decision for the pending update (1: v = y)
  int32_t label;   // DCX_EV_ACCEPTED / DCX_EV_REJECTED for the next record
  int32_t warned;  // first descent-violation iteration, -1 if none
  int32_t wlen;    // ADOCH window fill
};

struct HistRec {
  double h, e, t;
  int32_t ev, pad;
};

struct RunCfg {
  int64_t n;
  int32_t R;
  int32_t solver, window_mode, lookback_q;
  int64_t max_iters, stride;
  double budget;  // < 0: none
  double conv_tol, descent_tol;
  int32_t hist_cap, wcap;
  double es_scale;  // Es partials are multiplied by this (integer kinds)
  HistRec* hist;    // [R][hist_cap]
  double* window;   // [R][wcap]
  double momentum_floor;  // ADOCH in f32 / tensor-core precision: no extrapolation once the step is
                          // <= momentum_floor * sqrt(alpha / beta) (the state's scale; 0: off)
};

struct GState {
  int32_t p;       // passes executed
  int32_t live;    // 0 once every replica has stopped
  int32_t running; // replicas still running
  uint32_t arrive; // last-block-done counter
  unsigned long long t0;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// --------------------------------------------------------------- arithmetic
// Expressions that mirror numpy statements are evaluated with explicit
// round-to-nearest intrinsics so nvcc cannot contract them into FMAs; that is
// what makes apply_T / states / replay bitwise self-consistent (the reference
// tests pkg/tests/test_doch.py:318-342 rely on it).
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double cbrt_t(double a) { return cbrt(a); }
__device__ __forceinline__ float cbrt_t(float a) { return cbrtf(a); }

// SpMV accumulation. f64: multiply then add, row entries in column order
// (the order of scipy's csr_matvec, dc/coupling.py:189-190). f32: FMA.
__device__ __forceinline__ double madd(double acc, double v, double x) { return __dadd_rn(acc, __dmul_rn(v, x)); }
__device__ __forceinline__ float madd(float acc, float v, float x) { return fmaf(v, x, acc); }

template <typename T>
__device__ __forceinline__ T sgn(T x) { return x >= T(0) ? T(1) : T(-1); }  // dc/model.py:31-33

// (J + alpha I) x = Jx + alpha*x   (dc/solvers/doch.py:66-68)
template <typename T>
__device__ __forceinline__ T shifted(T jx, T alpha, T xi) { return add_rn(jx, mul_rn(alpha, xi)); }
// cbrt(Ax / beta)   (dc/solvers/doch.py:90-91)
// f64: the numpy expression exactly (IEEE division, correctly rounded cbrt).
// f32: Ax * (1/beta) and a cube root from the MUFU log2/exp2 estimate plus one
// Newton step (<= 1 ulp from cbrtf, about half the instructions of
// __fdiv_rn + cbrtf); zero maps to +0 so no iterate is ever -0.0 (the spin of
// x = -0.0 is +1, and the sign-bit energy accumulation relies on that).
__device__ __forceinline__ float cbrt_fast(float t) {
  const float a = fabsf(t);
  // branch-free: tiny inputs (denormals) are scaled by 2^96 exactly, the root by 2^-32
  const bool tiny = a < 1.0e-30f;
  const float as = tiny ? a * 0x1p96f : a;
  float l, r, rc;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(as));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * (1.0f / 3.0f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(r * r));
  r = fmaf(fmaf(as, rc, -r), 1.0f / 3.0f, r);  // Newton: r + (a / r^2 - r) / 3
  r = tiny ? r * 0x1p-32f : r;
  r = a == __int_as_float(0x7f800000) ? a : r;  // inf
  return a == 0.0f ? 0.0f : copysignf(r, t);
}
// Cube root for the solver iterations, whose arguments are normal floats or zero
// (t = (J + aI)x / beta ~ x^3 with x ~ sqrt(alpha / beta), far above the denormal range): MUFU
// log2 / exp2 estimate and one Newton step with the reciprocal of r^2 + 1e-37,
// so t = 0 gives +0 without a branch or select (the offset is a normal float: a
// denormal one would be flushed by rcp.approx.ftz and turn t = 0 into NaN; it is
// below 2e-12 of r^2 for every normal t, so <= 1 ulp from cbrtf on normal
// arguments). Denormal arguments flush to zero explicitly: lg2.approx.ftz would see 0,
// leave r = 0 and the Newton step would return a * 1e37 / 3.
__device__ __forceinline__ float cbrt_lean(float t) {
  const float a = fabsf(t);
  float l, r, rc;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(a));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * (1.0f / 3.0f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(fmaf(r, r, 1e-37f)));
  r = fmaf(fmaf(a, rc, -r), 1.0f / 3.0f, r);
  r = a < 1.17549435e-38f ? 0.0f : r;
  return __uint_as_float((__float_as_uint(r) & 0x7fffffffu) | (__float_as_uint(t) & 0x80000000u)) + 0.0f;
}
// Cube root from the inverse cube root: y = 2^(-log2|t| / 3) (2 MUFU), one FMA-only Newton
// step y(4 - |t| y^3)/3 (relative error ~1e-13 before rounding), then |t| y^2: <= ~1 ulp
// like cbrt_lean with one MUFU (the reciprocal) fewer. Zero and denormal arguments give +0.
__device__ __forceinline__ float cbrt_inv(float t) {
  const float a = fabsf(t);
  float l, y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(a));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(l * (-1.0f / 3.0f)));
  const float y3 = y * y * y;
  y = fmaf(y * fmaf(-a, y3, 1.0f), 1.0f / 3.0f, y);
  float r = (a * y) * y;
  r = a < 1.17549435e-38f ? 0.0f : r;
  return __uint_as_float((__float_as_uint(r) & 0x7fffffffu) | (__float_as_uint(t) & 0x80000000u)) + 0.0f;
}
// Cube root of the tensor-core DOCH update: t |t|^(-2/3) from the MUFU log2 / exp2 estimates
// alone (2 MUFU + 3 FP ops; no Newton step, so ~1e-7 relative instead of <= 1 ulp). The
// delta iteration rounds each step to e4m3 / f16 anyway and converges to the fixed point of
// this (deterministic) map; zero and denormal arguments give +0.
__device__ __forceinline__ float cbrt_mufu(float t) {
  const float a = fabsf(t);
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(a));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * (-2.0f / 3.0f)));
  return a < 1.17549435e-38f ? 0.0f : t * r;
}
__device__ __forceinline__ double inv_beta(double beta) { return beta; }  // unused in f64
__device__ __forceinline__ float inv_beta(float beta) { return __frcp_rn(beta); }
__device__ __forceinline__ double tmap(double ax, double beta, double) { return cbrt(__ddiv_rn(ax, beta)); }
__device__ __forceinline__ float tmap(float ax, float, float ibeta) { return cbrt_fast(__fmul_rn(ax, ibeta)); }
// inside the solver iterations (arguments never denormal / infinite): the lean cube root
__device__ __forceinline__ double tmap_pass(double ax, double beta, double ib) { return tmap(ax, beta, ib); }
__device__ __forceinline__ float tmap_pass(float ax, float, float ibeta) { return cbrt_lean(__fmul_rn(ax, ibeta)); }

// Sign-bit helpers for the spin-energy accumulation: x < 0 <=> sign bit set,
// valid because iterates are never -0.0 (see tmap; initial states are
// canonicalised on upload).
__device__ __forceinline__ uint32_t negbit(float x) { return __float_as_uint(x) >> 31; }
__device__ __forceinline__ uint32_t negbit(double x) { return uint32_t(__double_as_longlong(x) >> 63) & 1u; }
__device__ __forceinline__ float sgnf_bits(float x) {
  return __uint_as_float((__float_as_uint(x) & 0x80000000u) | 0x3f800000u);
}
__device__ __forceinline__ float sgnf_bits(double x) {
  return __uint_as_float((uint32_t(__double_as_longlong(x) >> 32) & 0x80000000u) | 0x3f800000u);
}
// y = x + c (x - xp)   (dc/solvers/doch.py:299, :301)
template <typename T>
__device__ __forceinline__ T extrap(T x, T xp, T c) { return add_rn(x, mul_rn(c, sub_rn(x, xp))); }

// -------------------------------------------------------------- value loads
template <int VK>
struct EsAcc { using type = double; };
template <> struct EsAcc<VK_UNIFORM> { using type = int32_t; };
template <> struct EsAcc<VK_I8> { using type = int32_t; };
template <> struct EsAcc<VK_I16> { using type = int32_t; };

// One coupling entry: the value in T and, for integer kinds, the exact integer
// q with value = scale * q. NC selects the read-only global path (not usable
// on shared memory).
template <int VK, bool NC, typename T>
__device__ __forceinline__ T load_entry(const void* vals, int64_t e, T scale, int& q) {
  if constexpr (VK == VK_UNIFORM) { q = 1; return scale; }
  else if constexpr (VK == VK_I8) {
    const int8_t* p = reinterpret_cast<const int8_t*>(vals) + e;
    q = NC ? int(__ldg(p)) : int(*p);
    return scale * T(q);
  } else if constexpr (VK == VK_I16) {
    const int16_t* p = reinterpret_cast<const int16_t*>(vals) + e;
    q = NC ? int(__ldg(p)) : int(*p);
    return scale * T(q);
  } else if constexpr (VK == VK_F32) {
    const float* p = reinterpret_cast<const float*>(vals) + e;
    q = 0;
    return T(NC ? __ldg(p) : *p);
  } else {
    const double* p = reinterpret_cast<const double*>(vals) + e;
    q = 0;
    return T(NC ? __ldg(p) : *p);
  }
}

// contribution of one entry to the spin-energy accumulator (J sign x)_i
template <int VK, typename T>
__device__ __forceinline__ typename EsAcc<VK>::type es_term(int q, T v, T xj) {
  if constexpr (VK == VK_UNIFORM || VK == VK_I8 || VK == VK_I16) return xj >= T(0) ? q : -q;
  else return xj >= T(0) ? double(v) : -double(v);
}

// ------------------------------------------------------------ warp helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------- control logic
// Window of the last q+1 Hamiltonian values (dc/solvers/doch.py:282,305,322).
__device__ __forceinline__ void window_push(RepCtl& c, const RunCfg& cfg, int r, double h) {
  double* w = cfg.window + (int64_t)r * cfg.wcap;
  int q1 = cfg.lookback_q + 1;
  int cap = cfg.wcap;  // == min(q+1, max_iters+1)
  // position of this value: count so far
  w[c.wlen % cap] = h;
  c.wlen += 1;
  if (c.wlen <= q1) c.wmax = (c.wlen == 1) ? h : fmax(c.wmax, h);
}
__device__ __forceinline__ double window_max(const RepCtl& c, const RunCfg& cfg, int r) {
  int q1 = cfg.lookback_q + 1;
  if (c.wlen <= q1) return c.wmax;  // nothing evicted yet
  const double* w = cfg.window + (int64_t)r * cfg.wcap;
  double m = w[0];
  for (int i = 1; i < cfg.wcap; ++i) m = fmax(m, w[i]);
  return m;
}

__device__ __forceinline__ double nesterov_next(double t) {  // dc/solvers/doch.py:295
  return __dmul_rn(0.5, __dadd_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(__dmul_rn(4.0, t), t)))));
}

// Bookkeeping after the pass that evaluated x_p: H(x_p), E(sign x_p), and the
// step ||x_p - x_{p-1}|| stored in c.step by the previous update.
// `tot` holds reduced partials. Returns true if the replica stopped now.
__device__ inline bool control_after_pass(RepCtl& c, const RunCfg& cfg, int r, const double* tot, int p,
                                          double now_s) {
  const double h = __dsub_rn(__dmul_rn(__dmul_rn(0.25, c.beta), tot[Q_S4]), __dmul_rn(0.5, tot[Q_SXAX]));
  const double E = __dmul_rn(-0.5, __dmul_rn(cfg.es_scale, tot[Q_ES]));
  // cfg.hist == nullptr: redundant evaluation (dense path), no history writes
  HistRec* hr = cfg.hist ? cfg.hist + (int64_t)r * cfg.hist_cap + (p % cfg.hist_cap) : nullptr;
  bool stopped = false;
  if (p == 0) {
    c.h = h;
    c.k = 0;
    c.best = E;  // first record always improves on +inf (dc/solvers/common.py:70-73)
    c.best_iter = 0;
    c.pend = 0;
    if (hr) { hr->h = h; hr->e = E; hr->t = now_s; hr->ev = DCX_EV_RECORDED; }
    if (cfg.solver == DCX_SOLVER_ADOCH) { c.wlen = 0; window_push(c, cfg, r, h); }
    if (cfg.max_iters <= 0) { c.status = DCX_STOP_MAX_ITERS; stopped = true; }
    return stopped;
  }
  const int k = p;
  int ev = 0;
  bool force = false;
  if (cfg.solver == DCX_SOLVER_DOCH) {
    if (__dsub_rn(h, c.h) > cfg.descent_tol) {  // dc/solvers/doch.py:206-213
      ev |= DCX_EV_DESCENT;
      force = true;
      if (c.warned < 0) c.warned = k;
    }
  } else {
    ev |= c.label;  // label of the decision that produced x_k (doch.py:308,312)
    window_push(c, cfg, r, h);
  }
  c.h = h;
  c.k = k;
  const bool converged = c.step <= cfg.conv_tol;                 // doch.py:220
  const bool late = cfg.budget >= 0.0 && now_s >= cfg.budget;    // doch.py:221-223
  const bool record = (k % cfg.stride == 0) || converged || late || (k == cfg.max_iters) || force;
  if (record) {
    ev |= DCX_EV_RECORDED;
    if (E < c.best) { c.best = E; c.best_iter = k; c.pend = k; }
  }
  if (hr) { hr->h = h; hr->e = record ? E : __longlong_as_double(0x7ff8000000000000ll); hr->t = now_s; hr->ev = ev; }
  if (converged) { c.status = DCX_STOP_CONVERGED; stopped = true; }
  else if (late) { c.status = DCX_STOP_TIME_BUDGET; stopped = true; }
  else if (k >= cfg.max_iters) { c.status = DCX_STOP_MAX_ITERS; stopped = true; }
  return stopped;
}

// ADOCH acceptance decision for loop index k = p (doch.py:294-315). Pass p used
// c.cm[p&1]; the partials Q_SY4/Q_SYAY hold H(y_p) terms.
__device__ inline void adoch_decide(RepCtl& c, const RunCfg& cfg, int r, const double* tot, int p) {
  const double t_next = nesterov_next(c.t);
  if (p == 0) {
    c.accept = 1;
    c.label = 0;
  } else {
    const double hy = __dsub_rn(__dmul_rn(__dmul_rn(0.25, c.beta), tot[Q_SY4]), __dmul_rn(0.5, tot[Q_SYAY]));
    bool ok = hy <= window_max(c, cfg, r);
    // f32 / tensor-core endgame: once the step is below the state's resolution the extrapolated
    // point y carries only rounding noise, which the momentum amplifies ~ k/3, so
    // the iteration never settles; the plain step T(x) lets it reach its discrete fixed point
    if (cfg.momentum_floor > 0.0 && c.step <= cfg.momentum_floor * sqrt(__ddiv_rn(c.alpha, c.beta))) ok = false;
    c.accept = ok ? 1 : 0;
    c.label = ok ? DCX_EV_ACCEPTED : DCX_EV_REJECTED;
  }
  c.t = t_next;
  // coefficient for the next extrapolation: c_{p+1} = (t_{p+1} - 1) / t_{p+2}
  c.cm[(p + 1) & 1] = __ddiv_rn(__dsub_rn(c.t, 1.0), nesterov_next(c.t));
}

}  // namespace dcx
