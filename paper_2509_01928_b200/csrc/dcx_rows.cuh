// Row epilogue shared by the pass kernels (dcx_csr.cu, dcx_proc.cu): everything
// that is elementwise once a row product (J v)_i is known.
#pragma once
#include "dcx_internal.h"

namespace dcx {

// ---------------------------------------------------------------------------
// Row epilogue shared by the pass kernels. `acc` = (J v)_i in T,
// `es` = (J sign x_p)_i. `xi` = x_p[i]. Everything that is elementwise given
// the row product happens here.
template <typename T, int MODE>
struct RowOut {
  double s4 = 0, sxax = 0, es = 0, step = 0, sy4 = 0, syay = 0;
};

// The replica's control values the epilogue needs, in registers.
template <typename T>
struct RowCtl {
  T alpha, beta, ibeta, cm;
  int pend;
  bool running;
};
template <typename T>
__device__ __forceinline__ RowCtl<T> row_ctl(const RepCtl& c, int p) {
  RowCtl<T> k;
  k.alpha = T(c.alpha);
  k.beta = T(c.beta);
  k.ibeta = inv_beta(k.beta);
  k.cm = T(p & 1 ? c.cm[1] : c.cm[0]);
  k.pend = c.pend;
  k.running = c.status == DCX_STOP_RUNNING;
  return k;
}

template <typename T, int MODE>
__device__ __forceinline__ void row_epilogue(const PassArgs& a, const RowCtl<T>& c, int p, int64_t idx, T acc,
                                             double esrow, RowOut<T, MODE>& o) {
  const T* xcur = reinterpret_cast<const T*>(a.x[xslot(a, p)]);
  T* xnext = reinterpret_cast<T*>(a.x[xslot(a, p + 1)]);
  const T alpha = c.alpha;
  if constexpr (MODE == MODE_ADOCH_Y) {
    // acc = J y ; y recomputed identically to the gather
    const T* xprev = reinterpret_cast<const T*>(a.x[xslot(a, p + a.nbuf - 1)]);
    T yi = extrap(xcur[idx], xprev[idx], c.cm);
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
      // pending best-spin copy (x_{p-1}, or x_{p-2} with three buffers), still held in the write buffer
      if (c.pend == copy_iter(a, p) && c.pend >= 0) a.best[idx] = xnext[idx] >= T(0) ? 1 : -1;
      if (c.running) {
        T xn = tmap_pass(ax, c.beta, c.ibeta);
        xnext[idx] = xn;
        // slots 0..max_iters: the pass at p = max_iters computes an x that is never kept
        if (a.states && p < a.cfg.max_iters) reinterpret_cast<T*>(a.states)[(int64_t)(p + 1) * a.cfg.n * a.cfg.R + idx] = xn;
        o.step = fmax(o.step, double(fabs(xn - xi)));
      }
    } else {  // MODE_ADOCH_X: store Ax_p, H(y_p) partials for the economy window test
      T* axb = reinterpret_cast<T*>(a.ax[p & 1]);
      axb[idx] = ax;
      if (p > 0 && a.cfg.window_mode == DCX_WINDOW_ECONOMY) {
        const T* xprev = reinterpret_cast<const T*>(a.x[xslot(a, p + a.nbuf - 1)]);
        const T* axprev = reinterpret_cast<const T*>(a.ax[(p + 1) & 1]);
        T yi = extrap(xi, xprev[idx], c.cm);
        T ayi = extrap(ax, axprev[idx], c.cm);
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

}  // namespace dcx
