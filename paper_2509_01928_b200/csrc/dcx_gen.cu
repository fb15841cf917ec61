// Instance generation and ingest on the device.
//
// gen_sparse_9bit (dc/generate.py:80-112). The reference draws, for every row
// i = 1..n-1 of the lower triangle, i integers z in [1, n_p] from its own
// Philox stream keyed (seed, i) (dc/generate.py:53-55) with numpy's
// Generator.integers, keeps z < 1023 as the coupling z - 511 at column j (the
// draw's index), and closes the pattern symmetrically through scipy's COO ->
// CSR. numpy's draw for a range below 2^32 is Lemire's bounded rule on the
// bit generator's 32-bit outputs: m = u * n_p, accept when (m mod 2^32) >=
// (2^32 - n_p) mod n_p, value m >> 32 (+1); Philox4x64-10's 32-bit outputs
// are the low then the high half of each 64-bit word, four words per counter
// value, counters 1, 2, ... A rejection only skips a 32-bit output, so the
// accepted outputs of a row are its draws in order: each warp evaluates 32
// counter blocks (256 outputs) at once, ranks the accepted ones with a
// ballot-free lane scan, and keeps going until the row has i draws. The same
// pass runs twice (count, then fill at the scanned offsets); the transposed
// half comes from a stable radix sort of the lower entries by column, so each
// row's columns end up strictly increasing exactly as scipy orders them.
//
// validate_csr: the CsrCoupling invariants of dc/coupling.py:153-176 checked
// by one warp per row (offsets, column range, strictly increasing columns, no
// diagonal, finite values, symmetry by binary search of the transposed entry:
// a stored value must equal its mirror, or be zero when the mirror is absent,
// which is what `(sp != sp.T).nnz == 0` accepts). The host reports the first
// failing check in the reference's order.
#include <cub/cub.cuh>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "dcx_internal.h"

namespace dcx {

namespace {

#define GCK(call)                                                                                       \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr uint64_t PH_M0 = 0xD2E7470EE14C6C93ull, PH_M1 = 0xCA5A826395121157ull;
constexpr uint64_t PH_W0 = 0x9E3779B97F4A7C15ull, PH_W1 = 0xBB67AE8584CAA73Bull;

// Philox4x64-10 of counter (c0, 0, 0, 0) under key (k0, k1) (Random123 / numpy)
__device__ __forceinline__ void philox4x64(uint64_t c0, uint64_t k0, uint64_t k1, uint64_t (&o)[4]) {
  uint64_t a = c0, b = 0, c = 0, d = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += PH_W0;
      k1 += PH_W1;
    }
    const uint64_t hi0 = __umul64hi(PH_M0, a), lo0 = PH_M0 * a;
    const uint64_t hi1 = __umul64hi(PH_M1, c), lo1 = PH_M1 * c;
    const uint64_t na = hi1 ^ b ^ k0, nc = hi0 ^ d ^ k1;
    a = na;
    b = lo1;
    c = nc;
    d = lo0;
  }
  o[0] = a;
  o[1] = b;
  o[2] = c;
  o[3] = d;
}

__device__ __forceinline__ int64_t clamp64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane, uint32_t& total) {
  uint32_t s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += t;
  }
  total = __shfl_sync(0xffffffffu, s, 31);
  return s - v;
}

// FILL = false: lower-triangle kept count of every row; true: write the entries
// (column j, row i, value z - 511) at loff[i] in draw order (increasing j)
template <bool FILL>
__global__ void __launch_bounds__(256) rows_9bit(int64_t n, uint32_t n_p, uint32_t thr, uint64_t seed, int64_t* cnt,
                                                 const int64_t* loff, uint32_t* lcol, uint32_t* lrow, int16_t* lval) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = 1 + w; i < n; i += nw) {
    int64_t done = 0, kept = 0;
    uint64_t blk = 0;
    const int64_t pos0 = FILL ? loff[i] : 0;
    while (done < i) {
      uint64_t o[4];
      philox4x64(blk + uint64_t(lane) + 1, seed, uint64_t(i), o);
      uint32_t z[8];
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t u = (k & 1) ? uint32_t(o[k >> 1] >> 32) : uint32_t(o[k >> 1]);
        const uint64_t m = uint64_t(u) * n_p;
        z[k] = uint32_t(m >> 32) + 1u;
        if (uint32_t(m) >= thr) acc |= 1u << k;
      }
      uint32_t total;
      const uint32_t before = warp_excl_scan(__popc(acc), lane, total);
      // this lane's accepted outputs are draws done + before, done + before + 1, ...
      uint32_t keepm = 0;
      int rank = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if ((acc >> k) & 1u) {
          const int64_t d = done + before + rank++;
          if (d < i && z[k] < 1023u) keepm |= 1u << k;
        }
      uint32_t ktot;
      const uint32_t kbefore = warp_excl_scan(__popc(keepm), lane, ktot);
      if (FILL && keepm) {
        int64_t pos = pos0 + kept + kbefore;
        int r2 = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if ((acc >> k) & 1u) {
            const int64_t d = done + before + r2++;
            if ((keepm >> k) & 1u) {
              lcol[pos] = uint32_t(d);
              lrow[pos] = uint32_t(i);
              lval[pos] = int16_t(int(z[k]) - 511);
              ++pos;
            }
          }
        }
      }
      kept += ktot;
      done += total;
      blk += 32;
    }
    if (!FILL && lane == 0) cnt[i] = kept;
  }
}

__global__ void column_counts(const uint32_t* lcol, int64_t L, unsigned long long* ucnt) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < L; t += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(ucnt + lcol[t], 1ull);
}

__global__ void row_totals(int64_t n, const int64_t* lcnt, const unsigned long long* ucnt, int64_t* tot) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= n; r += int64_t(gridDim.x) * blockDim.x)
    tot[r] = r < n ? lcnt[r] + int64_t(ucnt[r]) : 0;
}

__global__ void iota_u32(uint32_t* v, int64_t L) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < L; t += int64_t(gridDim.x) * blockDim.x)
    v[t] = uint32_t(t);
}

// row r of the symmetric CSR: its lower entries (columns < r, in order), then the
// transposed ones (columns > r: rows of the lower triangle that kept column r, in
// increasing row order by the stable sort)
__global__ void __launch_bounds__(256) assemble_rows(int64_t n, const int64_t* loff, const int64_t* uoff,
                                                     const int64_t* ro, const uint32_t* lcol, const uint32_t* lrow,
                                                     const int16_t* lval, const uint32_t* sorted_idx, int64_t* col,
                                                     double* val) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w; r < n; r += nw) {
    const int64_t a0 = loff[r], a1 = loff[r + 1], b0 = uoff[r], b1 = uoff[r + 1], o = ro[r];
    for (int64_t t = a0 + lane; t < a1; t += 32) {
      col[o + (t - a0)] = lcol[t];
      val[o + (t - a0)] = double(lval[t]);
    }
    const int64_t o2 = o + (a1 - a0);
    for (int64_t t = b0 + lane; t < b1; t += 32) {
      const uint32_t k = sorted_idx[t];
      col[o2 + (t - b0)] = lrow[k];
      val[o2 + (t - b0)] = double(lval[k]);
    }
  }
}

template <typename T>
T* dmalloc(size_t count) {
  void* p = nullptr;
  GCK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

struct Scratch {  // frees every allocation on scope exit (exceptions included)
  std::vector<void*> ptrs;
  template <typename T>
  T* get(size_t count) {
    T* p = dmalloc<T>(count);
    ptrs.push_back(p);
    return p;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

void excl_scan_i64(const int64_t* in, int64_t* out, int64_t count, Scratch& sc, cudaStream_t s) {
  size_t tb = 0;
  GCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, count, s));
  void* tmp = sc.get<unsigned char>(tb);
  GCK(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, count, s));
}

int grid_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + per_block - 1) / per_block;
  return int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * 16)));
}

// ------------------------------------------------------------------ validation
struct VFlags {
  unsigned long long inc_row, diag_row;  // first row with a non-increasing column / a stored diagonal
  int offsets_bad, range_bad, nonfinite, nonint, asym;
};

__global__ void __launch_bounds__(256) validate_rows(int64_t n, int64_t nnz, const int64_t* ro, const int64_t* col,
                                                     const double* val, VFlags* f) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw) {
    int64_t lo = ro[i], hi = ro[i + 1];
    if (lane == 0 && (hi < lo || (i == 0 && lo != 0))) f->offsets_bad = 1;
    lo = clamp64(lo, 0, nnz);
    hi = clamp64(hi, lo, nnz);
    bool inc = false, diag = false;
    for (int64_t e = lo + lane; e < hi; e += 32) {
      const int64_t j = col[e];
      const double v = val[e];
      if (j < 0 || j >= n) {
        f->range_bad = 1;
        continue;
      }
      if (e > lo && col[e - 1] >= j) inc = true;
      if (j == i) diag = true;
      if (!isfinite(v)) f->nonfinite = 1;
      if (v != rint(v)) f->nonint = 1;
      // mirror (j, i): binary search in row j (columns sorted where the other checks pass)
      int64_t a = clamp64(ro[j], 0, nnz), b = clamp64(ro[j + 1], a, nnz);
      bool found = false;
      double mv = 0.0;
      while (a < b) {
        const int64_t m = (a + b) >> 1;
        const int64_t c = col[m];
        if (c == i) {
          found = true;
          mv = val[m];
          break;
        }
        if (c < i) a = m + 1;
        else b = m;
      }
      if (found ? !(mv == v) : (v != 0.0)) f->asym = 1;
    }
    if (__any_sync(0xffffffffu, inc) && lane == 0) atomicMin(&f->inc_row, (unsigned long long)i);
    if (__any_sync(0xffffffffu, diag) && lane == 0) atomicMin(&f->diag_row, (unsigned long long)i);
  }
}

}  // namespace

void GenCsr::release() {
  if (ro) cudaFree(ro);
  if (col) cudaFree(col);
  if (val) cudaFree(val);
  ro = col = nullptr;
  val = nullptr;
  n = nnz = 0;
}

void gen_sparse_9bit(int64_t n, int64_t n_p, uint64_t seed, GenCsr& out, cudaStream_t s) {
  if (n < 2) throw std::invalid_argument("n must be >= 2");
  if (n >= (int64_t(1) << 31)) throw std::invalid_argument("n >= 2^31 is not supported");
  if (n_p < 1 || n_p > 0xFFFFFFFFll) throw std::invalid_argument("n_p out of range");
  out.release();
  Scratch sc;
  const uint32_t np32 = uint32_t(n_p);
  // numpy's Lemire threshold (2^32 - n_p) mod n_p, i.e. (UINT32_MAX - rng) % (rng + 1), rng = n_p - 1
  const uint32_t thr = uint32_t((0xFFFFFFFFull - uint64_t(n_p - 1)) % uint64_t(n_p));
  int64_t* lcnt = sc.get<int64_t>(n + 1);
  GCK(cudaMemsetAsync(lcnt, 0, sizeof(int64_t) * (n + 1), s));
  const int gr = grid_for(n * 32, 256);
  if (n_p > 1) rows_9bit<false><<<gr, 256, 0, s>>>(n, np32, thr, seed, lcnt, nullptr, nullptr, nullptr, nullptr);
  GCK(cudaGetLastError());
  int64_t* loff = sc.get<int64_t>(n + 1);
  excl_scan_i64(lcnt, loff, n + 1, sc, s);
  int64_t L = 0;
  GCK(cudaMemcpyAsync(&L, loff + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GCK(cudaStreamSynchronize(s));
  if (2 * L >= (int64_t(1) << 31)) throw std::invalid_argument("more than 2^31 stored couplings are not supported");
  uint32_t* lcol = sc.get<uint32_t>(L);
  uint32_t* lrow = sc.get<uint32_t>(L);
  int16_t* lval = sc.get<int16_t>(L);
  if (L > 0) rows_9bit<true><<<gr, 256, 0, s>>>(n, np32, thr, seed, nullptr, loff, lcol, lrow, lval);
  GCK(cudaGetLastError());
  // transposed half: stable sort of the lower entries by column
  unsigned long long* ucnt = sc.get<unsigned long long>(n + 1);
  GCK(cudaMemsetAsync(ucnt, 0, sizeof(unsigned long long) * (n + 1), s));
  uint32_t* idx_in = sc.get<uint32_t>(L);
  uint32_t* idx_out = sc.get<uint32_t>(L);
  uint32_t* keys_out = sc.get<uint32_t>(L);
  if (L > 0) {
    const int g2 = grid_for(L, 256);
    column_counts<<<g2, 256, 0, s>>>(lcol, L, ucnt);
    iota_u32<<<g2, 256, 0, s>>>(idx_in, L);
    int bits = 1;
    while ((int64_t(1) << bits) < n) ++bits;
    size_t tb = 0;
    GCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, lcol, keys_out, idx_in, idx_out, int(L), 0, bits, s));
    void* tmp = sc.get<unsigned char>(tb);
    GCK(cub::DeviceRadixSort::SortPairs(tmp, tb, lcol, keys_out, idx_in, idx_out, int(L), 0, bits, s));
  }
  int64_t* ucnt64 = reinterpret_cast<int64_t*>(ucnt);  // counts < 2^63: same bits
  int64_t* uoff = sc.get<int64_t>(n + 1);
  excl_scan_i64(ucnt64, uoff, n + 1, sc, s);
  int64_t* tot = sc.get<int64_t>(n + 1);
  row_totals<<<grid_for(n + 1, 256), 256, 0, s>>>(n, lcnt, ucnt, tot);
  out.ro = dmalloc<int64_t>(n + 1);
  out.n = n;
  excl_scan_i64(tot, out.ro, n + 1, sc, s);
  out.nnz = 2 * L;
  out.col = dmalloc<int64_t>(out.nnz);
  out.val = dmalloc<double>(out.nnz);
  if (L > 0)
    assemble_rows<<<grid_for(n * 32, 256), 256, 0, s>>>(n, loff, uoff, out.ro, lcol, lrow, lval, idx_out, out.col,
                                                         out.val);
  GCK(cudaGetLastError());
  GCK(cudaStreamSynchronize(s));
}

int validate_csr_device(int64_t n, int64_t nnz, const int64_t* ro_h, const int64_t* col_h, const double* val_h,
                        int64_t* row, int* all_int, cudaStream_t s) {
  // returns 0 = valid, 2 offsets, 3 lengths, 4 column range, 5 non-increasing row, 6 diagonal, 7 non-finite,
  // 8 asymmetric (the order of dc/coupling.py:153-176)
  *row = -1;
  *all_int = 0;
  if (ro_h[0] != 0) return 2;
  if (ro_h[n] != nnz) {
    // a decreasing offset sequence is reported first, as the reference does
    for (int64_t i = 0; i < n; ++i)
      if (ro_h[i + 1] < ro_h[i]) return 2;
    return 3;
  }
  Scratch sc;
  int64_t* ro = sc.get<int64_t>(n + 1);
  int64_t* col = sc.get<int64_t>(nnz);
  double* val = sc.get<double>(nnz);
  VFlags* f = sc.get<VFlags>(1);
  GCK(cudaMemcpyAsync(ro, ro_h, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  if (nnz) {
    GCK(cudaMemcpyAsync(col, col_h, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
    GCK(cudaMemcpyAsync(val, val_h, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
  }
  VFlags h{};
  h.inc_row = h.diag_row = ~0ull;
  GCK(cudaMemcpyAsync(f, &h, sizeof(VFlags), cudaMemcpyHostToDevice, s));
  validate_rows<<<grid_for(n * 32, 256), 256, 0, s>>>(n, nnz, ro, col, val, f);
  GCK(cudaGetLastError());
  GCK(cudaMemcpyAsync(&h, f, sizeof(VFlags), cudaMemcpyDeviceToHost, s));
  GCK(cudaStreamSynchronize(s));
  *all_int = (nnz > 0 && !h.nonint) ? 1 : 0;
  if (h.offsets_bad) return 2;
  if (h.range_bad) return 4;
  if (h.inc_row != ~0ull || h.diag_row != ~0ull) {
    const unsigned long long first = std::min(h.inc_row, h.diag_row);
    *row = int64_t(first);
    return h.inc_row == first ? 5 : 6;
  }
  if (h.nonfinite) return 7;
  if (h.asym) return 8;
  return 0;
}

}  // namespace dcx
