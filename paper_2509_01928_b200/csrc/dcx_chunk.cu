// Column-chunked R = 1 pass for states larger than L2 (BASELINE configs[4], R8).
//
// The R8 state x is 400 MB; the 126 MB L2 cannot hold it, so every one of the
// 3e8 random 4-byte gathers of pass_r1w is a random DRAM access (ncu: 33 GB of
// DRAM reads per pass, profiles/r2_ncu_r8_pass_r1w.txt). Here the column space
// is cut into C chunks of at most CHUNK_BYTES of x each, and a pass becomes C
// sweeps, sweep c visiting exactly the entries whose column lies in chunk c --
// while it runs, the chunk of x it gathers from stays in L2. The entries of a
// chunk are stored once per coupling, regrouped into row segments (a row's
// consecutive entries with columns in that chunk), ordered by row; each
// segment continues its row's running sum, kept between sweeps in an 8-byte
// (f32 sum, int32 spin-energy sum) pair per row. A row's entries are sorted by
// column, so sweeping the chunks in order applies exactly the FMA sequence of
// the row kernels (column order): the iterates are bit-identical to pass_r1w.
// A last per-row kernel applies the shared row epilogue (dcx_rows.cuh) to the
// finished sums and clears them for the next pass.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "dcx_internal.h"
#include "dcx_rows.cuh"

namespace dcx {

namespace {

#define KCK(call)                                                                                       \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int ROW_BITS = 27;  // key = chunk << 27 | row: n < 2^27, C < 32

__global__ void entry_keys(const uint32_t* rp, const int32_t* col, int64_t n, int64_t width, uint32_t* keys,
                           uint32_t* idx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
      keys[e] = (uint32_t(col[e] / width) << ROW_BITS) | uint32_t(i);
      idx[e] = e;
    }
}

__global__ void gather_entries(const uint32_t* order, const int32_t* col, const int8_t* q, int64_t nnz, int32_t* ecol,
                               int8_t* eq) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = order[k];
    ecol[k] = col[e];
    if (q) eq[k] = q[e];
  }
}

// segment s of the run-length encoding: its row, and the first segment of every chunk
__global__ void segment_index(const uint32_t* ukeys, const uint32_t* counts, int64_t nseg, uint32_t* seg_row,
                              uint8_t* seg_cnt, int64_t* chunk_begin, int C, unsigned* too_long) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nseg; s += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t k = ukeys[s];
    seg_row[s] = k & ((1u << ROW_BITS) - 1u);
    if (counts[s] > 255u) *too_long = 1;
    seg_cnt[s] = uint8_t(counts[s]);
    const int c = int(k >> ROW_BITS);
    const int cp = s == 0 ? -1 : int(ukeys[s - 1] >> ROW_BITS);
    for (int q = cp + 1; q <= c; ++q) chunk_begin[q] = s;  // chunks without segments start here too
    if (s == nseg - 1)
      for (int q = c + 1; q <= C; ++q) chunk_begin[q] = nseg;
  }
}

// one sweep: the segments of chunk c, each continuing its row's running sums.
// A thread takes CK_U segments at a time and issues their independent loads
// (segment words, running sums, first column, first gather) before using any:
// most R8 segments hold one entry, so the loop is a chain of dependent loads.
constexpr int CK_U = 4;
// x gathers: keep the chunk in L2 against the streams (which load with evict-first .cs)
__device__ __forceinline__ float ld_keep(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
template <int VK, int MODE>
__global__ void __launch_bounds__(256) chunk_sweep(PassArgs a, int c) {
  using T = float;
  if (!a.g->live) return;
  const int p = a.g->p;
  const RowCtl<T> rc = row_ctl<T>(a.ctl[0], p);
  if (!rc.running) return;
  const ChunkArgs& k = a.chunks;
  const int64_t s0 = k.chunk_begin[c], s1 = k.chunk_begin[c + 1];
  const T* xc = reinterpret_cast<const T*>(a.gx[p & 1]);
  const T scale = T(a.scale);
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  uint64_t keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  for (int64_t sb = s0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; sb < s1; sb += CK_U * nt) {
    uint32_t row[CK_U], e0[CK_U];
    int cnt[CK_U];
    float2 acc2[CK_U];
    int32_t j0[CK_U];
#pragma unroll
    for (int u = 0; u < CK_U; ++u) {
      const int64_t s = sb + u * nt;
      cnt[u] = 0;
      if (s < s1) {
        row[u] = __ldcs(k.seg_row + s);
        cnt[u] = __ldcs(k.seg_cnt + s);
        e0[u] = __ldcs(k.seg_start + s);
      }
    }
#pragma unroll
    for (int u = 0; u < CK_U; ++u)
      if (cnt[u]) {
        acc2[u] = __ldcs(k.acc + row[u]);
        j0[u] = __ldcs(k.ecol + e0[u]);
      }
    T x0[CK_U];
#pragma unroll
    for (int u = 0; u < CK_U; ++u)
      if (cnt[u]) x0[u] = ld_keep(xc + j0[u], keep);
#pragma unroll
    for (int u = 0; u < CK_U; ++u) {
      if (!cnt[u]) continue;
      T acc = acc2[u].x;
      int es = __float_as_int(acc2[u].y);
      for (int t = 0; t < cnt[u]; ++t) {  // the row's entries of this chunk, column order
        const T xj = t == 0 ? x0[u] : ld_keep(xc + __ldcs(k.ecol + e0[u] + t), keep);
        if constexpr (VK == VK_UNIFORM) {
          acc = madd(acc, scale, xj);
          es += negbit(xj) ? -1 : 1;
        } else {
          const int q = k.eq[e0[u] + t];
          acc = madd(acc, scale * T(q), xj);
          es += negbit(xj) ? -q : q;
        }
      }
      __stcs(k.acc + row[u], make_float2(acc, __int_as_float(es)));
    }
  }
}

// the row epilogue over the finished sums (which it clears for the next pass)
template <int MODE>
__global__ void __launch_bounds__(256) chunk_epilogue(PassArgs a) {
  using T = float;
  if (!a.g->live) return;
  const int p = a.g->p;
  const RowCtl<T> c = row_ctl<T>(a.ctl[0], p);
  const bool running = c.running;
  if (!running && !(MODE == MODE_DOCH && c.pend == p - 1)) return;
  const int64_t n = a.cfg.n;
  RowOut<T, MODE> o;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if (running) {
      const float2 s = a.chunks.acc[i];
      a.chunks.acc[i] = make_float2(0.f, 0.f);
      row_epilogue<T, MODE>(a, c, p, i, s.x, double(__float_as_int(s.y)), o);
    } else if (MODE == MODE_DOCH) {  // stopped: only the pending copy
      a.best[i] = reinterpret_cast<const T*>(a.x[(p + 1) & 1])[i] >= T(0) ? 1 : -1;
    }
  }
  o.s4 = warp_sum(o.s4);
  o.sxax = warp_sum(o.sxax);
  o.es = warp_sum(o.es);
  o.step = warp_max(o.step);
  o.sy4 = warp_sum(o.sy4);
  o.syay = warp_sum(o.syay);
  __shared__ double red[8][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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

template <typename T>
T* kalloc(size_t count) {
  T* p = nullptr;
  KCK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return p;
}

}  // namespace

void ChunkPlan::release() {
  for (const void* p : {static_cast<const void*>(seg_row), static_cast<const void*>(seg_cnt),
                        static_cast<const void*>(seg_start), static_cast<const void*>(ecol),
                        static_cast<const void*>(eq), static_cast<const void*>(acc),
                        static_cast<const void*>(chunk_begin)})
    if (p) cudaFree(const_cast<void*>(p));
  static_cast<ChunkArgs&>(*this) = ChunkArgs{};
}

// Chunks for R = 1 f32 runs: DCX_CHUNKS=C (0 = off); DCX_CHUNKS=auto sizes them to CHUNK_BYTES of x
// when x exceeds it. Opt-in: measured slower than pass_r1w on R8.
int chunk_count(int64_t n) {
  const char* e = std::getenv("DCX_CHUNKS");
  if (!e) return 0;
  if (std::string(e) != "auto") return std::max(0, std::min(31, std::atoi(e)));
  const int64_t bytes = n * 4;
  if (bytes <= CHUNK_BYTES) return 0;
  return int(std::min<int64_t>(31, (bytes + CHUNK_BYTES - 1) / CHUNK_BYTES));
}

void build_chunk_plan(ChunkPlan& k, const uint32_t* rp, const int32_t* col, const int8_t* q, int64_t n, int64_t nnz,
                      int C, cudaStream_t s) {
  k.release();
  if (C <= 0) return;
  if (n >= (int64_t(1) << ROW_BITS)) throw std::invalid_argument("chunked pass: n >= 2^27");
  const int64_t width = (n + C - 1) / C;
  uint32_t *keys = kalloc<uint32_t>(nnz), *keys2 = kalloc<uint32_t>(nnz), *idx = kalloc<uint32_t>(nnz),
           *idx2 = kalloc<uint32_t>(nnz);
  const int grid = int(std::min<int64_t>(148 * 32, (n + 255) / 256 + 1));
  entry_keys<<<grid, 256, 0, s>>>(rp, col, n, width, keys, idx);
  KCK(cudaGetLastError());
  size_t tb = 0;
  const int bits = ROW_BITS + 5;
  KCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, idx2, nnz, 0, bits, s));
  void* tmp = nullptr;
  KCK(cudaMalloc(&tmp, tb));
  KCK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, idx, idx2, nnz, 0, bits, s));  // stable
  cudaFree(tmp);
  int32_t* ecol = kalloc<int32_t>(nnz);
  int8_t* eq = q ? kalloc<int8_t>(nnz) : nullptr;
  k.ecol = ecol;
  k.eq = eq;
  gather_entries<<<grid, 256, 0, s>>>(idx2, col, q, nnz, ecol, eq);
  KCK(cudaGetLastError());
  // run-length encode the sorted keys: one segment per (chunk, row)
  uint32_t* ukeys = keys;  // reuse
  uint32_t* counts = idx;
  int64_t* nseg_d = kalloc<int64_t>(1);
  tb = 0;
  KCK(cub::DeviceRunLengthEncode::Encode(nullptr, tb, keys2, ukeys, counts, nseg_d, nnz, s));
  KCK(cudaMalloc(&tmp, tb));
  KCK(cub::DeviceRunLengthEncode::Encode(tmp, tb, keys2, ukeys, counts, nseg_d, nnz, s));
  cudaFree(tmp);
  int64_t nseg = 0;
  KCK(cudaMemcpyAsync(&nseg, nseg_d, 8, cudaMemcpyDeviceToHost, s));
  KCK(cudaStreamSynchronize(s));
  k.nseg = nseg;
  uint32_t* seg_row = kalloc<uint32_t>(nseg);
  uint8_t* seg_cnt = kalloc<uint8_t>(nseg);
  uint32_t* seg_start = kalloc<uint32_t>(nseg);
  int64_t* chunk_begin = kalloc<int64_t>(C + 1);
  k.seg_row = seg_row;
  k.seg_cnt = seg_cnt;
  k.seg_start = seg_start;
  k.chunk_begin = chunk_begin;
  unsigned* too_long = reinterpret_cast<unsigned*>(nseg_d);
  KCK(cudaMemsetAsync(too_long, 0, 4, s));
  segment_index<<<grid, 256, 0, s>>>(ukeys, counts, nseg, seg_row, seg_cnt, chunk_begin, C, too_long);
  KCK(cudaGetLastError());
  tb = 0;
  KCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, seg_start, nseg, s));
  KCK(cudaMalloc(&tmp, tb));
  KCK(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, seg_start, nseg, s));
  cudaFree(tmp);
  unsigned tl = 0;
  KCK(cudaMemcpyAsync(&tl, too_long, 4, cudaMemcpyDeviceToHost, s));
  KCK(cudaStreamSynchronize(s));
  cudaFree(keys);
  cudaFree(keys2);
  cudaFree(idx);
  cudaFree(idx2);
  cudaFree(nseg_d);
  if (tl) {  // a row with more than 255 entries in one chunk: keep the row kernels
    k.release();
    return;
  }
  k.acc = kalloc<float2>(n);
  KCK(cudaMemsetAsync(k.acc, 0, n * sizeof(float2), s));
  KCK(cudaStreamSynchronize(s));
  k.C = C;
}

// C sweeps + the epilogue (R = 1, f32, integer couplings, DOCH / ADOCH x-pass)
void launch_chunked_pass(int mode, int vk, const PassArgs& a, int grid, cudaStream_t s) {
  const ChunkArgs& k = a.chunks;
  const int sg = 148 * 8;
  for (int c = 0; c < k.C; ++c) {
    if (vk == VK_UNIFORM) {
      if (mode == MODE_DOCH) chunk_sweep<VK_UNIFORM, MODE_DOCH><<<sg, 256, 0, s>>>(a, c);
      else chunk_sweep<VK_UNIFORM, MODE_ADOCH_X><<<sg, 256, 0, s>>>(a, c);
    } else {
      if (mode == MODE_DOCH) chunk_sweep<VK_I8, MODE_DOCH><<<sg, 256, 0, s>>>(a, c);
      else chunk_sweep<VK_I8, MODE_ADOCH_X><<<sg, 256, 0, s>>>(a, c);
    }
  }
  if (mode == MODE_DOCH) chunk_epilogue<MODE_DOCH><<<grid, 256, 0, s>>>(a);
  else chunk_epilogue<MODE_ADOCH_X><<<grid, 256, 0, s>>>(a);
}

}  // namespace dcx
