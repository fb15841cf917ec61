// Internal declarations shared by the .cu translation units of libdcx.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "dcx_device.cuh"

namespace dcx {

// Device CSR in its compressed form for one precision.
struct CsrDev {
  int64_t n = 0, nnz = 0;
  const uint32_t* rp = nullptr;
  const int32_t* col = nullptr;
  const uint16_t* col16 = nullptr;  // present when n <= 65536 (persistent kernel)
  const void* val = nullptr;
  int vk = VK_F64;
  double scale = 1.0;
  int V = 1;     // lanes per row (R = 1 kernels and the operator seam)
  int64_t ell = 0;  // entries of the 32-row sliced-ELL form of the pattern (persistent kernel, n <= 65536)
  bool pow2_uniform = false;  // uniform values with a power-of-two scale (sum x, then scale: exact)
  int grid = 1;  // grid of the R = 1 pass / apply kernels
  long long proc_seed = 0;  // VK_PROC: seed of sin(i*j + seed)
};

// Column-chunked R = 1 pass (dcx_chunk.cu): a coupling's entries regrouped by
// column chunk into row segments, and the per-row running sums carried between
// the chunk sweeps of one pass. Non-owning view (kernel argument).
struct ChunkArgs {
  int C = 0;                        // chunks; 0 = no plan (row kernels)
  int64_t nseg = 0;
  const int64_t* chunk_begin = nullptr;  // [C + 1] first segment of each chunk
  const uint32_t* seg_row = nullptr;     // [nseg] row of the segment
  const uint8_t* seg_cnt = nullptr;      // [nseg] entries (<= 255)
  const uint32_t* seg_start = nullptr;   // [nseg] first entry in ecol / eq
  const int32_t* ecol = nullptr;         // [nnz] columns, segment order
  const int8_t* eq = nullptr;            // [nnz] int8 values (VK_I8), segment order
  float2* acc = nullptr;                 // [n] (f32 row sum, int32 spin-energy sum as bits)
};
// owning form, kept by the context next to its coupling
struct ChunkPlan : ChunkArgs {
  void release();
  ~ChunkPlan() { release(); }
};
constexpr int64_t CHUNK_BYTES = int64_t(48) << 20;  // x per chunk: leaves L2 room for the streams
int chunk_count(int64_t n);
void build_chunk_plan(ChunkPlan& k, const uint32_t* rp, const int32_t* col, const int8_t* q, int64_t n, int64_t nnz,
                      int C, cudaStream_t s);

// Kernel argument block of one multi-pass iteration (passed by value).
struct PassArgs {
  const uint32_t* rp;
  const int32_t* col;
  const void* val;
  double scale;
  RepCtl* ctl;
  GState* g;
  void* x[4];      // iterate buffers (xslot below), layout [n][R], at this context's own rows
  void* gx[4];     // the same buffers at spin 0: the gather source (== x unless row-partitioned)
  void* ax[2];     // ADOCH (J+aI)x_p by parity
  void* ay;        // ADOCH exact (J+aI)y
  int8_t* best;    // best spins [n][R]
  void* states;    // optional [(max_iters+1)][n][R]
  double* part;    // pass partials [R][NQ][slots]
  int32_t slots;
  int32_t es_f32;  // pass_rv: per-lane spin-energy sums exact in f32 (integer couplings, bounded rows)
  const void* xmap[4];  // pass_rv: tile::gather4 maps over gx[0..nbuf) (device copies), or null (cp.async staging)
  long long proc_seed;  // procedural coupling (vk == VK_PROC): seed of sin(i*j + seed)
  // 2-D periodic L x L lattice detected at upload (dcx_api.cu detect_torus): the stencil
  // pass reads the bonds instead of the CSR. torus_L = 0: not a lattice
  int32_t torus_L;
  const int8_t* bond_r;  // q(i, right(i))  [n]
  const int8_t* bond_d;  // q(i, down(i))   [n]
  // pass_torus: sign bits of x_p written by pass p into sgnw[p & 1], [n][R / 32] words
  // (word 4c + v of a site: bit l = replica 128c + 4l + v); the pending best copy of
  // pass p + 1 reads them instead of x_p
  uint32_t* sgnw[2];
  ChunkArgs chunks;  // C > 0: the R = 1 pass runs as C column-chunk sweeps + a row epilogue
  // iterate buffers in rotation: 2 (by pass parity), or 3 / 4 (DOCH multipass: x_{p-nbuf+1} survives
  // pass p, so the best-spin copy of x_q is made only when none of the next nbuf - 2 iterates improves on it)
  int32_t nbuf;
  RunCfg cfg;
};

// the buffer holding x_q (q >= 0)
__host__ __device__ __forceinline__ int xslot(const PassArgs& a, int q) {
  return a.nbuf == 2 ? (q & 1) : (a.nbuf == 4 ? (q & 3) : q % 3);
}
// pass p copies sign(x_q) into the best spins when q = pend is this pass's copy iterate x_{p-nbuf+1}
// (x_{p-1} with two buffers), the buffer pass p overwrites (xslot(a, p + 1))
__host__ __device__ __forceinline__ int copy_iter(const PassArgs& a, int p) { return p - a.nbuf + 1; }

struct MultiPass {
  PassArgs args;
  bool f64 = true;
  int solver = DCX_SOLVER_DOCH;
  int vk = VK_F64, V = 1, grid = 1, fgrid = 1, sslots = 1;
  double* spart = nullptr;  // ADOCH finalize step partials [sslots][R]
};

// dcx_csr.cu
void enqueue_iteration(const MultiPass& m, cudaStream_t s);
// row-partitioned (multi-GPU) iteration, split around the caller's all-reduce of
// the per-replica partials: pass + per-rank reduction into qs/qm, then control
void enqueue_dist_pass(const MultiPass& m, double* qs, double* qm, cudaStream_t s);
void enqueue_dist_control(const MultiPass& m, const double* qs, const double* qm, cudaStream_t s);
// the pass over own rows [lo, hi) into slot half `half`, and the fold of both halves into qs / qm
void enqueue_dist_pass_rows(const MultiPass& m, int64_t lo, int64_t hi, int half, cudaStream_t s);
void enqueue_dist_reduce(const MultiPass& m, double* qs, double* qm, cudaStream_t s);
void enqueue_flush(const MultiPass& m, cudaStream_t s);
void enqueue_pass_only(const MultiPass& m, cudaStream_t s);
void enqueue_start_clock(GState* g, cudaStream_t s);
int replica_vector_width(int R, bool f64);
// dcx_chunk.cu
void launch_chunked_pass(int mode, int vk, const PassArgs& a, int grid, cudaStream_t s);
// dcx_dense.cu: row-gather TMA map ([rows][cols], box = one row of box_cols elements)
void encode_row_gather_map(void* map_out, void* base, uint64_t cols, uint64_t rows, bool f64, uint32_t box_cols);
// dcx_power.cu
void launch_power(const CsrDev& J, int use_shift, double shift, double tol, int64_t max_iters, double* v, double* w,
                  const double* restart, double* part, double* part2, unsigned* bar, double* out, int grid,
                  cudaStream_t s);
template <typename T>
void launch_csr_apply(const CsrDev& J, const T* v, int R, T* jv, double* es_rows, cudaStream_t s);

// dcx_proc.cu: procedural couplings (VK_PROC)
template <typename T>
void launch_proc_pass(int mode, const PassArgs& a, int grid, cudaStream_t s);
int proc_pass_grid(int64_t n);
int proc_replica_chunk(int R);
template <typename T>
void launch_proc_apply(int64_t n, long long seed, const T* v, int R, T* jv, double* es_rows, cudaStream_t s);
void launch_proc_row_stats(int64_t n, long long seed, double* out, cudaStream_t s);

// dcx_gen.cu: instance generation and ingest on the device
struct GenCsr {  // a generated CSR in the reference's host layout (int64 offsets / columns, f64 values)
  int64_t n = 0, nnz = 0;
  int64_t* ro = nullptr;
  int64_t* col = nullptr;
  double* val = nullptr;
  void release();
  ~GenCsr() { release(); }
};
void gen_sparse_9bit(int64_t n, int64_t n_p, uint64_t seed, GenCsr& out, cudaStream_t s);
int validate_csr_device(int64_t n, int64_t nnz, const int64_t* ro, const int64_t* col, const double* val,
                        int64_t* row, int* all_int, cudaStream_t s);

// dcx_small.cu: persistent one-CTA-per-replica kernel (whole CSR in smem)
struct SmallPlan {
  size_t smem = 0;
  int threads = 256;
  bool fits = false;
  bool ell = false;  // sliced-ELL column layout in shared memory
};
SmallPlan plan_small(const CsrDev& J, int solver, int window_mode, bool f64);
void launch_small(const MultiPass& m, const CsrDev& J, const SmallPlan& sp, int p_end, cudaStream_t s);

}  // namespace dcx
