// libdcx C ABI (include/dcx.h): context, coupling upload, operator seam and
// the chunked solve driver. No exception crosses the ABI.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <emmintrin.h>
#include <pthread.h>

#include "dcx_internal.h"
#include "dcx_dense.h"

using namespace dcx;

namespace {

thread_local std::string g_last_error;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t b) {
    if (b == bytes && p) return;
    release();
    if (b == 0) return;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      throw std::runtime_error(std::string("OOM: cudaMalloc(") + std::to_string(b) + "): " + cudaGetErrorString(e));
    }
    bytes = b;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

}  // namespace

// A pinned history buffer, shared between the context that drains a run into it and the
// detached result that reads it later (the context takes a free one for its next run).
struct PinnedRing {
  HistRec* p = nullptr;
  size_t n = 0;
  // the last run's history copy is left in flight (the host returns to the caller while
  // it lands); readers wait on `ready` first
  cudaEvent_t ready = nullptr;
  bool pending = false;
  void mark_pending(cudaStream_t s) {
    if (!ready && cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) {
      ready = nullptr;
      cudaStreamSynchronize(s);
      return;
    }
    cudaEventRecord(ready, s);
    pending = true;
  }
  void wait() {
    if (pending) cudaEventSynchronize(ready);
    pending = false;
  }
  ~PinnedRing() {
    if (ready) {
      cudaEventSynchronize(ready);
      cudaEventDestroy(ready);
    }
    if (p) cudaFreeHost(p);
  }
};
// Device buffer owned by a detached result (gathered states / best spins).
struct SharedDev {
  void* p = nullptr;
  size_t bytes = 0;
  ~SharedDev() {
    if (p) cudaFree(p);
  }
};

// DCX_TIMING=1: wall-clock phases of the host entry points on stderr (e2e analysis)
static bool timing_on() {
  static const bool on = std::getenv("DCX_TIMING") != nullptr;
  return on;
}
struct PhaseClock {
  const char* what;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  explicit PhaseClock(const char* w) : what(w) {}
  void mark(const char* phase) {
    if (!timing_on()) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dcx timing] %s %-18s %8.3f ms\n", what, phase,
                 std::chrono::duration<double, std::milli>(t - last).count());
    last = t;
  }
};

struct dcx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // ---------------------------------------------------------- coupling
  bool have = false, dense = false, csr_ready = false;
  bool proc = false;         // procedural J_ij = sin(i*j + proc_seed) (dcx_set_procedural)
  long long proc_seed = 0;
  std::vector<double> dense_host;  // dense couplings: host copy for the lazily built CSR form (filled on first use
                                   // from the device copy the dense upload keeps, dn.scratch)
  int64_t n = 0, nnz = 0;
  int64_t n_cols = 0, row_base = 0;  // row block of a row-partitioned coupling (n_cols == n, 0 otherwise)
  int vk_int = -1;  // VK_UNIFORM / VK_I8 / VK_I16, or -1 for real values
  double scale = 1.0;
  int V32 = 1;
  int64_t ell_entries = 0;  // 32-row sliced ELL size of the pattern (n <= 65536)
  double es_row_bound = 0;  // max over rows of sum_j |q_ij| (integer kinds; bound)
  DevBuf rp, col, col16, vint, v64, v32;
  int64_t torus_L = 0;     // > 0: the coupling is the periodic torus_L x torus_L lattice (detect_torus)
  DevBuf bond_r, bond_d;   // its bonds q(i, right(i)), q(i, down(i)) as int8
  DenseDev dn;  // dense tensor-core operands (dcx_dense.cu)
  ChunkPlan chunks;  // column-chunked R = 1 pass plan (dcx_chunk.cu), built on first use per coupling
  // ---------------------------------------------------------- run state
  dcx_params prm{};
  int R = 0;
  bool begun = false, finished = false, f64 = true;
  int path = DCX_PATH_MULTIPASS;
  int cap = 0, wcap = 0, chunk = 0, p_host = 0;
  DevBuf ctl, g, hist, window, xb0, xb1, xb2, xb3, ax0, ax1, ay, best, states, part, spart;
  DevBuf scratch;  // grow-only staging (x0 upload, result gathers): no cudaMalloc / cudaFree per call
  DevBuf xmaps;    // pass_rv row-gather TMA maps over the two iterate buffers
  DevBuf sgn0, sgn1;  // pass_torus sign words of x_p by pass parity
  MultiPass mp;
  CsrDev J;
  SmallPlan sp;
  cudaGraphExec_t graph = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // the final history copy of a run goes out on its own stream (copy_hist defer): syncs of
  // `stream` (result gathers, the next upload) do not wait for it; the next run's first
  // write of `hist` waits for hist_copied
  cudaStream_t hstream = nullptr;
  cudaEvent_t hist_go = nullptr, hist_copied = nullptr;
  bool hist_inflight = false;
  double* wdelta = nullptr;  // mapped pinned [R]: descent-warning deltas written by a kernel
  size_t wdelta_n = 0;       // (no copy queued behind the in-flight history copy)
  double dev_seconds = 0.0;
  bool dist = false;              // dcx_dist_begin run: external iterate buffers, caller's collectives
  double *qs = nullptr, *qm = nullptr;
  std::vector<std::vector<HistRec>> hh;  // drained history (used when the ring can wrap)
  bool ring_direct = false;              // the ring holds every record: results read it in place
  std::vector<int64_t> hcnt;             // records per replica (ring_direct)
  int64_t nhist(int r) const { return ring_direct ? hcnt[r] : (int64_t)hh[r].size(); }
  const HistRec& rec(int r, int64_t k) const { return ring_direct ? ring[size_t(r) * cap + k] : hh[r][k]; }
  std::vector<RepCtl> hctl;
  float prof_ms = 0.f;  // dcx_profile_kernel: summed event time of the timed dense launches
  HistRec* ring = nullptr;  // pinned host copy of the device history ring (ringp->p)
  size_t ring_n = 0;
  std::shared_ptr<PinnedRing> ringp;                 // the current run's ring
  std::vector<std::shared_ptr<PinnedRing>> spare;    // rings no detached result holds any more
  std::vector<std::shared_ptr<SharedDev>> dspare;    // result device buffers free for reuse
  GState hg{};
  GenCsr gen;  // dcx_gen_sparse_9bit result until dcx_gen_result
  unsigned char* pin = nullptr;  // grow-only pinned staging of CSR uploads (row offsets + columns)
  size_t pin_bytes = 0;

  ~dcx_ctx() {
    if (pin) cudaFreeHost(pin);
    if (graph) cudaGraphExecDestroy(graph);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (hstream) cudaStreamSynchronize(hstream);
    if (wdelta) cudaFreeHost(wdelta);
    if (hist_go) cudaEventDestroy(hist_go);
    if (hist_copied) cudaEventDestroy(hist_copied);
    if (hstream) cudaStreamDestroy(hstream);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

int fail(dcx_ctx* ctx, int code, const std::string& msg) {
  g_last_error = msg;
  if (ctx) ctx->err = msg;
  return code;
}

template <typename F>
int guarded(dcx_ctx* ctx, F&& f) {
  try {
    if (ctx) CK(cudaSetDevice(ctx->device));
    f();
    return DCX_OK;
  } catch (const InvalidArg& e) {
    return fail(ctx, DCX_E_INVALID, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(ctx, DCX_E_INVALID, e.what());
  } catch (const CudaError& e) {
    return fail(ctx, DCX_E_CUDA, e.what());
  } catch (const std::bad_alloc& e) {
    return fail(ctx, DCX_E_OOM, "host allocation failed");
  } catch (const std::runtime_error& e) {
    const std::string m = e.what();
    return fail(ctx, m.rfind("OOM", 0) == 0 ? DCX_E_OOM : DCX_E_CUDA, m);
  } catch (...) {
    return fail(ctx, DCX_E_CUDA, "unknown error");
  }
}

int lanes_for_degree(double d) {
  if (d < 3) return 1;
  if (d < 6) return 2;
  if (d < 12) return 4;
  if (d < 24) return 8;
  if (d < 48) return 16;
  return 32;
}

// Host passes over the uploaded arrays (10^8 entries at R8) run on all host threads.
// Host worker pool for par_for: spawning 16 threads per call cost 0.2-0.3 ms, paid
// several times per solve (classify J, convert x0, CSR staging). Workers spin for a few
// milliseconds after a job (the calls come in bursts) and then block.
struct HostPool {
  // A parallel loop is a set of blocks taken from a shared counter by the calling thread and by
  // whichever workers are awake: a worker whose virtual CPU the host does not schedule for a
  // while (measured: single uploads stalled 0.5-0.9 s when the loop waited for every worker's
  // fixed share) only misses the blocks the others took. The loop is done when every block is;
  // a worker that wakes after that finds the loop closed and never touches it.
  std::mutex run_mu;  // one parallel loop at a time
  std::mutex mu;
  std::condition_variable cv, cv_done;
  std::atomic<uint64_t> gen{0};
  std::atomic<int> next{0}, done{0};
  int nblk = 0, active = 0;
  bool open = false;
  const std::function<void(int)>* job = nullptr;
  std::vector<std::thread> th;
  explicit HostPool(int n) {
    for (int i = 1; i < n; ++i) th.emplace_back([this] { loop(); });
  }
  int size() const { return int(th.size()) + 1; }
  void work() {  // blocks until none is left
    for (int b; (b = next.fetch_add(1, std::memory_order_acq_rel)) < nblk;) {
      (*job)(b);
      done.fetch_add(1, std::memory_order_acq_rel);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // spin up to 3 ms: waking a blocked worker on these hosts (KVM guests) cost ~0.4 ms
      // per parallel loop, more than the loops themselves
      const auto t0 = std::chrono::steady_clock::now();
      while (gen.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(3))
        for (int s = 0; s < 64; ++s) _mm_pause();
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return gen.load(std::memory_order_acquire) != seen; });
        seen = gen.load(std::memory_order_acquire);
        if (!open) continue;  // that loop finished without this worker
        ++active;
      }
      work();
      std::lock_guard<std::mutex> lk(mu);
      if (--active == 0) cv_done.notify_one();
    }
  }
  // f(b) for every block b in [0, blocks)
  void run(int blocks, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> g(run_mu);
    {
      std::lock_guard<std::mutex> lk(mu);
      job = &f;
      nblk = blocks;
      next.store(0, std::memory_order_relaxed);
      done.store(0, std::memory_order_relaxed);
      open = true;
      gen.fetch_add(1, std::memory_order_acq_rel);
    }
    cv.notify_all();
    work();
    while (done.load(std::memory_order_acquire) < blocks) _mm_pause();  // blocks other threads hold
    std::unique_lock<std::mutex> lk(mu);
    open = false;  // late workers skip this loop
    cv_done.wait(lk, [&] { return active == 0; });  // workers still inside finished their last block
  }
};

HostPool* g_pool = nullptr;
std::mutex g_pool_mu;

HostPool& host_pool() {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool) {
    // a forked child has none of the parent's workers: it builds its own pool
    static bool hooked = [] { return pthread_atfork(nullptr, nullptr, [] { g_pool = nullptr; }) == 0; }();
    (void)hooked;
    unsigned hw = std::min(32u, std::max(1u, std::thread::hardware_concurrency()));
    if (const char* e = std::getenv("DCX_HOST_THREADS"))
      hw = unsigned(std::max(1, std::min(32, std::atoi(e))));
    else if (const char* l = std::getenv("LOCAL_WORLD_SIZE"))  // torchrun: ranks on this node share the cores
      hw = std::max(1u, hw / unsigned(std::max(1, std::atoi(l))));
    g_pool = new HostPool(int(hw));  // never freed: workers live as long as the process
  }
  return *g_pool;
}

// f(lo, hi, t) over contiguous blocks [lo, hi) of [0, n), block t < 32 (callers keep one result
// slot per block); block starts are multiples of 64 elements so streaming stores (stream_fill)
// cover whole cache lines
template <class F>
static void par_for(int64_t n, F&& f, int max_threads = 32) {
  if (n < (int64_t(1) << 16)) {
    f(int64_t(0), n, 0);
    return;
  }
  HostPool& pool = host_pool();
  // up to 32 blocks (callers keep one result slot per block), two per thread
  const int T = std::max(1, std::min({pool.size(), max_threads, 16}));
  const int blocks = std::min(32, 2 * T);
  const int64_t chunk = ((n + blocks - 1) / blocks + 63) / 64 * 64;
  const std::function<void(int)> body = [&](int t) {
    const int64_t lo = std::min(n, t * chunk), hi = std::min(n, lo + chunk);
    if (lo < hi) f(lo, hi, t);
  };
  pool.run(blocks, body);
}

// dst[k] = f(k) for k in [lo, hi) with streaming (non-temporal) stores: the pinned staging
// a DMA reads next must not sit dirty in 16 cores' private caches. Measured on the B200
// hosts (KVM guests): 8 MB written by 16 threads then copied H2D at 6.6 GB/s with plain
// stores, 51 GB/s with streaming stores.
template <class T, class F>
static inline void stream_fill(T* dst, int64_t lo, int64_t hi, F&& f) {
  static_assert(16 % sizeof(T) == 0, "element size must divide 16");
  constexpr int V = int(16 / sizeof(T));
  int64_t k = lo;
  for (; k < hi && (reinterpret_cast<uintptr_t>(dst + k) & 15); ++k) dst[k] = f(k);
  for (; k + V <= hi; k += V) {
    alignas(16) T tmp[V];
    for (int j = 0; j < V; ++j) tmp[j] = f(k + j);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k), _mm_load_si128(reinterpret_cast<const __m128i*>(tmp)));
  }
  for (; k < hi; ++k) dst[k] = f(k);
  _mm_sfence();
}
// Round to nearest even without a libm call (std::nearbyint is one on the x86-64 baseline,
// a call per entry): exact for |x| < 2^51; larger or non-finite x fail every caller's
// |q| <= 127 / 32767 or q * scale == v check, as with nearbyint.
static inline double rne(double x) {
  const double m = 6755399441055744.0;  // 1.5 * 2^52
  return (x + m) - m;
}

// dst[k] = int32(ci[k]) for k in [lo, hi), streamed; true if some index is outside [0, n_cols)
// (SSE2: low and high 32-bit halves of four indices per step, n_cols < 2^31)
static bool stage_columns(const int64_t* ci, int32_t* dst, int64_t lo, int64_t hi, int64_t n_cols) {
  bool bad = false;
  int64_t k = lo;
  for (; k < hi && (reinterpret_cast<uintptr_t>(dst + k) & 15); ++k) {
    bad |= uint64_t(ci[k]) >= uint64_t(n_cols);
    dst[k] = int32_t(ci[k]);
  }
  const __m128i zero = _mm_setzero_si128(), last = _mm_set1_epi32(int32_t(n_cols - 1));
  __m128i acc = zero;
  for (; k + 4 <= hi; k += 4) {
    const __m128 a = _mm_castsi128_ps(_mm_loadu_si128(reinterpret_cast<const __m128i*>(ci + k)));
    const __m128 b = _mm_castsi128_ps(_mm_loadu_si128(reinterpret_cast<const __m128i*>(ci + k + 2)));
    const __m128i l = _mm_castps_si128(_mm_shuffle_ps(a, b, _MM_SHUFFLE(2, 0, 2, 0)));
    const __m128i h = _mm_castps_si128(_mm_shuffle_ps(a, b, _MM_SHUFFLE(3, 1, 3, 1)));
    acc = _mm_or_si128(acc, _mm_or_si128(h, _mm_or_si128(_mm_cmplt_epi32(l, zero), _mm_cmpgt_epi32(l, last))));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k), l);
  }
  bad |= _mm_movemask_epi8(_mm_cmpeq_epi8(acc, zero)) != 0xFFFF;
  for (; k < hi; ++k) {
    bad |= uint64_t(ci[k]) >= uint64_t(n_cols);
    dst[k] = int32_t(ci[k]);
  }
  _mm_sfence();
  return bad;
}

// one pass over v[lo, hi): all finite, all equal to v0, min |nonzero| (SSE2, four
// independent accumulators: a scalar min chain ran at a third of the memory rate)
static void value_stats(const double* v, int64_t lo, int64_t hi, double v0, bool& fin, bool& uni, double& mn) {
  const double inf = std::numeric_limits<double>::infinity();
  const __m128d absm = _mm_castsi128_pd(_mm_set1_epi64x(0x7fffffffffffffffLL));
  const __m128d big = _mm_set1_pd(std::numeric_limits<double>::max()), vinf = _mm_set1_pd(inf);
  const __m128d z = _mm_setzero_pd(), w0 = _mm_set1_pd(v0);
  __m128d m[4] = {vinf, vinf, vinf, vinf};
  __m128d ok = _mm_cmpeq_pd(z, z), eq = ok;
  int64_t k = lo;
  for (; k + 8 <= hi; k += 8) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __m128d x = _mm_loadu_pd(v + k + 2 * j), a = _mm_and_pd(x, absm);
      ok = _mm_and_pd(ok, _mm_cmple_pd(a, big));
      eq = _mm_and_pd(eq, _mm_cmpeq_pd(x, w0));
      const __m128d isz = _mm_cmpeq_pd(a, z);
      m[j] = _mm_min_pd(m[j], _mm_or_pd(_mm_and_pd(isz, vinf), _mm_andnot_pd(isz, a)));
    }
  }
  const __m128d mm = _mm_min_pd(_mm_min_pd(m[0], m[1]), _mm_min_pd(m[2], m[3]));
  alignas(16) double t[2];
  _mm_store_pd(t, mm);
  double mnv = std::min(t[0], t[1]);
  bool f = _mm_movemask_pd(ok) == 3, u = _mm_movemask_pd(eq) == 3;
  for (; k < hi; ++k) {
    const double x = v[k], a = std::fabs(x);
    f &= a <= std::numeric_limits<double>::max();
    u &= x == v0;
    mnv = std::min(mnv, a == 0.0 ? inf : a);
  }
  fin = f;
  uni = u;
  mn = mnv;
}

// Detect the narrowest exact storage of the coupling values.
void classify_values(const double* v, int64_t nnz, int& vk, double& scale) {
  if (nnz == 0) { vk = VK_UNIFORM; scale = 0.0; return; }
  std::vector<unsigned char> uni(32, 1), fin(32, 1);
  std::vector<double> mns(32, std::numeric_limits<double>::infinity());
  par_for(nnz, [&](int64_t lo, int64_t hi, int t) {
    bool u = true, f = true;
    double mn = std::numeric_limits<double>::infinity();
    value_stats(v, lo, hi, v[0], f, u, mn);
    uni[t] = u;
    fin[t] = f;
    mns[t] = mn;
  });
  bool uniform = true;
  double mn = std::numeric_limits<double>::infinity();
  for (int t = 0; t < 32; ++t) {
    if (!fin[t]) throw InvalidArg("couplings must be finite");
    uniform = uniform && uni[t];
    mn = std::min(mn, mns[t]);
  }
  if (uniform) { vk = VK_UNIFORM; scale = v[0]; return; }
  if (!std::isfinite(mn)) { vk = VK_UNIFORM; scale = 0.0; return; }
  for (double s : {mn, 1.0, 0.5, 0.25}) {
    std::vector<unsigned char> oks(32, 1);
    std::vector<double> amaxs(32, 0.0);
    par_for(nnz, [&](int64_t lo, int64_t hi, int t) {
      bool okt = true;
      double am = 0.0;
      for (int64_t e = lo; e < hi && okt; ++e) {
        const double q = v[e] / s;
        if (q != rne(q) || s * rne(q) != v[e]) okt = false;
        am = std::max(am, std::fabs(q));
      }
      oks[t] = okt;
      amaxs[t] = am;
    });
    bool ok = true;
    double amax = 0.0;
    for (int t = 0; t < 32; ++t) {
      ok = ok && oks[t];
      amax = std::max(amax, amaxs[t]);
    }
    if (!ok) continue;
    if (amax <= 127) { vk = VK_I8; scale = s; return; }
    if (amax <= 32767) { vk = VK_I16; scale = s; return; }
  }
  vk = -1;
  scale = 1.0;
}

CsrDev csr_view(const dcx_ctx* c, bool f64) {
  CsrDev J;
  J.n = c->n;
  J.nnz = c->nnz;
  if (c->proc) {  // nothing stored: the procedural kernels generate every entry
    J.vk = VK_PROC;
    J.proc_seed = c->proc_seed;
    J.V = 1;
    J.grid = proc_pass_grid(c->n);
    return J;
  }
  J.rp = c->rp.as<uint32_t>();
  J.col = c->col.as<int32_t>();
  J.col16 = c->col16.as<uint16_t>();
  if (c->vk_int >= 0) {
    J.vk = c->vk_int;
    J.val = c->vint.p;
    J.scale = c->scale;
  } else if (f64) {
    J.vk = VK_F64;
    J.val = c->v64.p;
  } else {
    J.vk = VK_F32;
    J.val = c->v32.p;
  }
  J.V = f64 ? 1 : c->V32;
  J.ell = c->ell_entries;
  if (J.vk == VK_UNIFORM && J.scale != 0.0) {
    int ex = 0;
    J.pow2_uniform = std::frexp(std::fabs(J.scale), &ex) == 0.5;
  }
  const int64_t rows_per_warp = 32 / J.V;
  const int64_t warps = (c->n + rows_per_warp - 1) / rows_per_warp;
  J.grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 16));
  return J;
}

void require_coupling(const dcx_ctx* c) {
  if (!c->have) throw InvalidArg("no coupling set");
}

// ------------------------------------------------------------ small kernels
template <typename T, typename S = double>
__global__ void to_device_layout_s(const S* src, T* dst, int64_t n, int R) {
  // src [R][n] -> dst [n][R]
  const int64_t total = n * R;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx / R;
    const int r = int(idx % R);
    dst[idx] = T(src[(int64_t)r * n + i]) + T(0);  // + 0 turns -0.0 into +0.0 (same spin, see tmap)
  }
}

template <typename T>
__global__ void to_device_layout(const double* src, T* dst, int64_t n, int R) {
  // src [R][n] -> dst [n][R]
  const int64_t total = n * R;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx / R;
    const int r = int(idx % R);
    dst[idx] = T(src[(int64_t)r * n + i]) + T(0);  // + 0 turns -0.0 into +0.0 (same spin, see tmap)
  }
}
template <typename T>
__global__ void from_device_layout(const T* src, double* dst, int64_t n, int R) {
  const int64_t total = n * R;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx / R;
    const int r = int(idx % R);
    dst[(int64_t)r * n + i] = double(src[idx]);
  }
}
// final state of each replica (buffer by the parity of its last iteration),
// [n][R] -> [R][n] f64, written coalesced for one device-to-host copy
template <typename T>
__global__ void gather_final_state(const T* x0, const T* x1, const T* x2, const T* x3, int nbuf, const RepCtl* ctl,
                                   int64_t n, int R, double* out) {
  const int64_t total = n * R;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total; o += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(o / n);
    const int64_t i = o % n;
    const int k = max(0, ctl[r].k);
    const int slot = nbuf == 2 ? (k & 1) : (nbuf == 4 ? (k & 3) : k % 3);  // the buffer of x_k (xslot)
    out[o] = double((slot == 0 ? x0 : (slot == 1 ? x1 : (slot == 2 ? x2 : x3)))[i * R + r]);
  }
}
// h_k - h_(k-1) at each replica's first descent violation k, NaN if none (the records sit
// in place: record k of replica r at r * cap + k)
__global__ void gather_warn_delta(const HistRec* hist, const RepCtl* ctl, int64_t cap, int R, double* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int k = ctl[r].warned;
  out[r] = (k >= 1 && k <= ctl[r].k) ? hist[r * cap + k].h - hist[r * cap + k - 1].h
                                     : __longlong_as_double(0x7ff8000000000000LL);
}
__global__ void gather_best(const int8_t* best, int64_t n, int R, int8_t* out) {
  const int64_t total = n * R;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total; o += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(o / n);
    const int64_t i = o % n;
    out[o] = best[i * R + r];
  }
}

// mode 0: tx = cbrt((jv + a v)/b), h = H(v); mode 1: E = -1/2 scale sum s_i es_i
template <typename T>
__global__ void rows_epilogue(int mode, const T* v, const T* jv, const double* es, const double* alpha,
                              const double* beta, double es_scale, int64_t n, int R, T* tx, double* out) {
  const int r = blockIdx.x;
  __shared__ double sa[256], sb[256];
  double a = 0.0, b = 0.0;
  const T al = mode == 0 ? T(alpha[r]) : T(0), be = mode == 0 ? T(beta[r]) : T(1);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t idx = i * R + r;
    if (mode == 0) {
      const T xi = v[idx];
      const T ax = shifted(jv[idx], al, xi);
      if (tx) tx[idx] = tmap(ax, be, inv_beta(be));
      const double x2 = double(mul_rn(xi, xi));
      a += x2 * x2;
      b += double(xi) * double(ax);
    } else {
      a += (v[idx] >= T(0) ? es[idx] : -es[idx]);
    }
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sa[threadIdx.x] += sa[threadIdx.x + w];
      sb[threadIdx.x] += sb[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (mode == 0) out[r] = __dsub_rn(__dmul_rn(__dmul_rn(0.25, beta[r]), sa[0]), __dmul_rn(0.5, sb[0]));
    else out[r] = __dmul_rn(-0.5, __dmul_rn(es_scale, sa[0]));
  }
}
__global__ void spins_to_device(const int8_t* s, double* dst, int64_t n, int R) {
  const int64_t total = n * R;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx / R;
    const int r = int(idx % R);
    dst[idx] = s[(int64_t)r * n + i] >= 0 ? 1.0 : -1.0;
  }
}

int grid_for(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 32)); }

}  // namespace

// -------------------------------------------------------------- operators
template <typename T>
static void apply_impl(dcx_ctx* c, int R, const double* alpha, const double* beta, const double* v, double* jv_out,
                       double* tx_out, double* h_out, const int8_t* spins, double* e_out) {
  const int64_t n = c->n;
  const bool f64 = sizeof(T) == 8;
  CsrDev J = csr_view(c, f64);
  DevBuf dsrc, dv, djv, dtx, des, dab, dout, dsp;
  const int64_t tot = n * R;
  dv.alloc(tot * sizeof(T));
  djv.alloc(tot * sizeof(T));
  if (spins) {
    dsp.alloc(tot);
    CK(cudaMemcpyAsync(dsp.p, spins, tot, cudaMemcpyHostToDevice, c->stream));
    dsrc.alloc(tot * 8);
    spins_to_device<<<grid_for(tot), 256, 0, c->stream>>>(dsp.as<int8_t>(), dsrc.as<double>(), n, R);
    // spins are exact in T; reuse the [n][R] buffer converted to T
    if (f64) CK(cudaMemcpyAsync(dv.p, dsrc.p, tot * 8, cudaMemcpyDeviceToDevice, c->stream));
    else {
      // convert double +-1 to float +-1 in place layout
      DevBuf tmp;
      tmp.alloc(tot * 8);
      from_device_layout<double><<<grid_for(tot), 256, 0, c->stream>>>(dsrc.as<double>(), tmp.as<double>(), n, R);
      to_device_layout<T><<<grid_for(tot), 256, 0, c->stream>>>(tmp.as<double>(), dv.as<T>(), n, R);
      CK(cudaStreamSynchronize(c->stream));
    }
    des.alloc(tot * 8);
  } else {
    dsrc.alloc(tot * 8);
    CK(cudaMemcpyAsync(dsrc.p, v, tot * 8, cudaMemcpyHostToDevice, c->stream));
    to_device_layout<T><<<grid_for(tot), 256, 0, c->stream>>>(dsrc.as<double>(), dv.as<T>(), n, R);
  }
  launch_csr_apply<T>(J, dv.as<T>(), R, djv.as<T>(), des.as<double>(), c->stream);
  CK(cudaGetLastError());
  if (jv_out) {
    DevBuf o;
    o.alloc(tot * 8);
    from_device_layout<T><<<grid_for(tot), 256, 0, c->stream>>>(djv.as<T>(), o.as<double>(), n, R);
    CK(cudaMemcpyAsync(jv_out, o.p, tot * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  if (tx_out || h_out || e_out) {
    dab.alloc(2 * R * 8 + 8);
    dout.alloc(R * 8);
    if (alpha) {
      CK(cudaMemcpyAsync(dab.p, alpha, R * 8, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(dab.as<double>() + R, beta, R * 8, cudaMemcpyHostToDevice, c->stream));
    }
    if (tx_out) dtx.alloc(tot * sizeof(T));
    const int mode = spins ? 1 : 0;
    const double es_scale = c->vk_int >= 0 ? c->scale : 1.0;
    rows_epilogue<T><<<R, 256, 0, c->stream>>>(mode, dv.as<T>(), djv.as<T>(), des.as<double>(), dab.as<double>(),
                                                dab.as<double>() + R, es_scale, n, R, dtx.as<T>(), dout.as<double>());
    CK(cudaGetLastError());
    if (tx_out) {
      DevBuf o;
      o.alloc(tot * 8);
      from_device_layout<T><<<grid_for(tot), 256, 0, c->stream>>>(dtx.as<T>(), o.as<double>(), n, R);
      CK(cudaMemcpyAsync(tx_out, o.p, tot * 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    double* dst = spins ? e_out : h_out;
    if (dst) CK(cudaMemcpyAsync(dst, dout.p, R * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
}

// ====================================================================== ABI
extern "C" {

int dcx_abi_version(void) { return DCX_ABI_VERSION; }

const char* dcx_last_error(const dcx_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int dcx_create(int device, dcx_ctx** out) {
  if (!out) return fail(nullptr, DCX_E_INVALID, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, DCX_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, DCX_E_INVALID, "device index out of range");
  dcx_ctx* c = new (std::nothrow) dcx_ctx();
  if (!c) return fail(nullptr, DCX_E_OOM, "host allocation failed");
  c->device = device;
  int rc = guarded(c, [&] {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreateWithFlags(&c->hist_go, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->hist_copied, cudaEventDisableTiming));
    if (const char* g = std::getenv("DCX_L2_FETCH")) {  // experiment: L2 fetch granularity of random gathers
      CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(std::atoi(g))));
      size_t v = 0;
      CK(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity));
      std::fprintf(stderr, "dcx: L2 fetch granularity %zu\n", v);
    }
  });
  if (rc != DCX_OK) {
    g_last_error = c->err;
    delete c;
    return rc;
  }
  *out = c;
  return DCX_OK;
}

void dcx_destroy(dcx_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

static int upload_csr(dcx_ctx* c, int64_t n, int64_t nnz, const int64_t* ro, const int64_t* ci, const double* v,
                      int64_t n_cols, int64_t row_base);

int dcx_set_csr(dcx_ctx* c, int64_t n, int64_t nnz, const int64_t* ro, const int64_t* ci, const double* v) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  c->dense = false;
  c->proc = false;
  c->csr_ready = false;
  c->chunks.release();
  c->dense_host.clear();
  c->dn.release();
  return upload_csr(c, n, nnz, ro, ci, v, n, 0);
}

int dcx_set_csr_block(dcx_ctx* c, int64_t n_rows, int64_t n_cols, int64_t row_base, int64_t nnz,
                      const int64_t* ro, const int64_t* ci, const double* v) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (n_rows < 1 || n_cols < n_rows || row_base < 0 || row_base + n_rows > n_cols)
    return fail(c, DCX_E_INVALID, "row block outside the spin index space");
  c->dense = false;
  c->proc = false;
  c->csr_ready = false;
  c->chunks.release();
  c->dense_host.clear();
  c->dn.release();
  return upload_csr(c, n_rows, nnz, ro, ci, v, n_cols, row_base);
}

// The periodic L x L lattice of BASELINE configs[2] (SURVEY.md Appendix A ``torus``):
// row i = (a, b) holds exactly up, left, right, down (ascending column order, L >= 3)
// with +-1 integer values, symmetric. Recognised here so the stencil pass (pass_torus,
// dcx_csr.cu) can read two int8 bond arrays instead of the CSR.
static void detect_torus(dcx_ctx* c, int64_t n, int64_t nnz, const int64_t* ro, const int32_t* col, const int8_t* q) {
  c->torus_L = 0;  // the bond buffers are kept for a re-upload of the same size (no cudaFree / cudaMalloc)
  const int64_t L = int64_t(std::llround(std::sqrt(double(n))));
  if (L < 3 || L * L != n || nnz != 4 * n) return;
  std::vector<int8_t> br(n), bd(n), bl(n), bu(n);
  std::atomic<bool> ok{true};
  // on all host threads (a single thread spent ~25 ms on T6's 10^6 rows every upload)
  par_for(n, [&](int64_t lo, int64_t hi, int) {
    int64_t a = lo / L, b = lo % L;
    for (int64_t i = lo; i < hi && ok.load(std::memory_order_relaxed); ++i) {
      if (ro[i] != 4 * i) { ok = false; return; }
      const int64_t up = (a == 0 ? L - 1 : a - 1) * L + b, left = a * L + (b == 0 ? L - 1 : b - 1),
                    right = a * L + (b == L - 1 ? 0 : b + 1), down = (a == L - 1 ? 0 : a + 1) * L + b;
      int64_t want[4] = {up, left, right, down};
      std::sort(want, want + 4);
      for (int k = 0; k < 4; ++k)
        if (col[4 * i + k] != want[k]) { ok = false; return; }
      for (int k = 0; k < 4; ++k) {
        const int8_t v = q[4 * i + k];
        if (v != 1 && v != -1) { ok = false; return; }
        const int64_t j = col[4 * i + k];
        if (j == right) br[i] = v;
        else if (j == down) bd[i] = v;
        else if (j == left) bl[i] = v;
        else bu[i] = v;
      }
      if (++b == L) { b = 0; ++a; }
    }
  });
  if (!ok) return;
  par_for(n, [&](int64_t lo, int64_t hi, int) {  // symmetric: q(i, left(i)) = q(left(i), i), q(i, up(i)) = q(up(i), i)
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t a = i / L, b = i % L;
      if (bl[i] != br[a * L + (b + L - 1) % L] || bu[i] != bd[((a + L - 1) % L) * L + b]) { ok = false; return; }
    }
  });
  if (!ok) return;
  PhaseClock pc("detect_torus");
  pc.mark("classify bonds");
  c->bond_r.alloc(n);
  c->bond_d.alloc(n);
  CK(cudaMemcpy(c->bond_r.p, br.data(), n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->bond_d.p, bd.data(), n, cudaMemcpyHostToDevice));
  pc.mark("bond upload");
  c->torus_L = L;
}

static int upload_csr(dcx_ctx* c, int64_t n, int64_t nnz, const int64_t* ro, const int64_t* ci, const double* v,
                      int64_t n_cols, int64_t row_base) {
  return guarded(c, [&] {
    PhaseClock pc("set_csr");
    c->chunks.release();
    if (n < 1) throw InvalidArg("n must be >= 1");
    if (n_cols >= (int64_t(1) << 31)) throw InvalidArg("n >= 2^31 is not supported");
    if (nnz < 0 || (nnz > 0 && (!ci || !v)) || !ro) throw InvalidArg("null CSR array");
    if (nnz >= (int64_t(1) << 32) - 1) throw InvalidArg("nnz >= 2^32 is not supported");
    if (n >= (int64_t(1) << 31)) throw InvalidArg("n >= 2^31 is not supported");
    if (ro[0] != 0 || ro[n] != nnz) throw InvalidArg("row_offsets must start at 0 and end at nnz");
    // row offsets and columns are converted straight into pinned staging (no host vectors
    // to zero-fill, DMA at full PCIe rate); the staging is kept for re-uploads
    const size_t qoff = (size_t(n + 1) * 4 + size_t(nnz) * 4 + 63) / 64 * 64;  // int8/int16 values
    const size_t stage = qoff + size_t(nnz) * 2;
    if (c->pin_bytes < stage) {
      if (c->pin) cudaFreeHost(c->pin);
      c->pin = nullptr;
      c->pin_bytes = 0;
      CK(cudaHostAlloc(reinterpret_cast<void**>(&c->pin), stage, cudaHostAllocDefault));
      c->pin_bytes = stage;
    }
    uint32_t* rp32 = reinterpret_cast<uint32_t*>(c->pin);
    int32_t* c32 = reinterpret_cast<int32_t*>(c->pin + size_t(n + 1) * 4);
    std::vector<unsigned char> bad(32, 0);
    std::vector<int64_t> maxlens(32, 0);
    par_for(n + 1, [&](int64_t lo, int64_t hi, int t) {
      int64_t ml = 0;
      bool b = false;
      stream_fill(rp32, lo, hi, [&](int64_t i) {
        if (i > 0) {
          b |= ro[i] < ro[i - 1];
          ml = std::max<int64_t>(ml, ro[i] - ro[i - 1]);
        }
        return uint32_t(ro[i]);
      });
      bad[t] = b;
      maxlens[t] = ml;
    });
    for (int t = 0; t < 32; ++t)
      if (bad[t]) throw InvalidArg("row_offsets must be nondecreasing");
    const int64_t row_maxlen = *std::max_element(maxlens.begin(), maxlens.end());
    c->have = false;  // the device arrays are overwritten from here on
    c->rp.alloc((n + 1) * 4);
    CK(cudaMemcpyAsync(c->rp.p, rp32, (n + 1) * 4, cudaMemcpyHostToDevice, c->stream));
    // 16 zero entries of padding: the R = 1 entry-parallel pass reads whole 16-byte vectors
    c->col.alloc((nnz + 16) * 4);
    CK(cudaMemsetAsync(static_cast<char*>(c->col.p) + nnz * 4, 0, 64, c->stream));
    pc.mark("offsets");
    // columns in pieces: the DMA of piece i overlaps the conversion of piece i + 1 and the
    // last pieces' DMA the value classification below
    const int64_t piece = std::max<int64_t>(int64_t(1) << 22, (nnz / 8 + 63) / 64 * 64);
    for (int64_t e0 = 0; e0 < nnz; e0 += piece) {
      const int64_t m = std::min(piece, nnz - e0);
      std::fill(bad.begin(), bad.end(), 0);
      par_for(m, [&](int64_t lo, int64_t hi, int t) { bad[t] = stage_columns(ci + e0, c32 + e0, lo, hi, n_cols); });
      if (std::any_of(bad.begin(), bad.end(), [](unsigned char b) { return b != 0; })) {
        CK(cudaStreamSynchronize(c->stream));
        throw InvalidArg("column index out of range");
      }
      CK(cudaMemcpyAsync(c->col.as<int32_t>() + e0, c32 + e0, size_t(m) * 4, cudaMemcpyHostToDevice, c->stream));
    }
    pc.mark("columns (+H2D issue)");
    int vk;
    double scale;
    classify_values(v, nnz, vk, scale);
    pc.mark("classify");
    if (vk == VK_I8 || vk == VK_UNIFORM) {
      // the UNIFORM / I8 kernels sum q * sign(x) per row in f32, exact while
      // every row's sum of |q| stays below 2^24; longer rows use the int32
      // (I16) path
      const int64_t maxlen = row_maxlen;
      if (maxlen * (vk == VK_I8 ? 127 : 1) >= (int64_t(1) << 24) && scale != 0.0) vk = VK_I16;
    }
    c->torus_L = 0;
    c->n = n;
    c->n_cols = n_cols;
    c->row_base = row_base;
    c->nnz = nnz;
    CK(cudaStreamSynchronize(c->stream));
    pc.mark("columns H2D wait");
    pc.mark("offsets+columns H2D");
    c->col16.release();
    if (n_cols <= 65536 && n == n_cols && nnz) {
      std::vector<uint16_t> c16(nnz);
      for (int64_t e = 0; e < nnz; ++e) c16[e] = uint16_t(c32[e]);
      c->col16.alloc(nnz * 2);
      CK(cudaMemcpy(c->col16.p, c16.data(), nnz * 2, cudaMemcpyHostToDevice));
    }
    c->vint.release();
    c->v64.release();
    c->v32.release();
    c->vk_int = (vk == VK_UNIFORM || vk == VK_I8 || vk == VK_I16) ? vk : -1;
    c->scale = scale;
    if (vk == VK_I8 || vk == VK_I16) {
      const int b = vk == VK_I8 ? 1 : 2;
      int8_t* q8 = reinterpret_cast<int8_t*>(c->pin + qoff);  // pinned staging, streamed
      int16_t* q16 = reinterpret_cast<int16_t*>(c->pin + qoff);
      par_for(nnz, [&](int64_t lo, int64_t hi, int) {
        if (b == 1) stream_fill(q8, lo, hi, [&](int64_t e) { return int8_t(rne(v[e] / scale)); });
        else stream_fill(q16, lo, hi, [&](int64_t e) { return int16_t(rne(v[e] / scale)); });
      });
      pc.mark("values q");
      c->vint.alloc((nnz + 16) * b);
      CK(cudaMemset(static_cast<char*>(c->vint.p) + nnz * b, 0, 16 * b));
      CK(cudaMemcpy(c->vint.p, c->pin + qoff, nnz * b, cudaMemcpyHostToDevice));
      pc.mark("values H2D");
      if (b == 1 && n == n_cols && row_base == 0) detect_torus(c, n, nnz, ro, c32, q8);
    pc.mark("values q + H2D");
    } else if (vk != VK_UNIFORM) {
      c->v64.alloc(nnz * 8);
      CK(cudaMemcpy(c->v64.p, v, nnz * 8, cudaMemcpyHostToDevice));
      std::vector<float> f(nnz);
      for (int64_t e = 0; e < nnz; ++e) f[e] = float(v[e]);
      c->v32.alloc(nnz * 4);
      CK(cudaMemcpy(c->v32.p, f.data(), nnz * 4, cudaMemcpyHostToDevice));
    }
    c->V32 = lanes_for_degree(double(nnz) / double(n));
    c->ell_entries = 0;
    {
      const int64_t maxlen = row_maxlen;
      double qmax = vk == VK_UNIFORM ? 1.0 : 0.0;
      if (vk == VK_I8 || vk == VK_I16) {
        std::vector<double> qm(32, 0.0);
        par_for(nnz, [&](int64_t lo, int64_t hi, int t) {
          double m = 0.0;
          for (int64_t e = lo; e < hi; ++e) m = std::max(m, std::fabs(rne(v[e] / scale)));
          qm[t] = m;
        });
        qmax = std::max(qmax, *std::max_element(qm.begin(), qm.end()));
      }
      c->es_row_bound = double(maxlen) * qmax;
    }
    pc.mark("qmax");
    if (n_cols <= 65536 && n == n_cols)
      for (int64_t s0 = 0; s0 < n; s0 += 32) {
        int64_t mx = 0;
        for (int64_t i = s0; i < std::min<int64_t>(n, s0 + 32); ++i) mx = std::max<int64_t>(mx, ro[i + 1] - ro[i]);
        c->ell_entries += 32 * mx;
      }
    c->have = true;
  });
}

// CSR of the nonzero off-diagonal entries of the dense coupling, built on first
// use by a CSR path (the tensor-core path never needs it).
static int ensure_csr(dcx_ctx* c) {
  if (!c->dense || c->csr_ready) return DCX_OK;
  const int64_t n = c->n;
  if (c->dense_host.size() != size_t(n * n)) {
    // the f64 coupling as uploaded (dense_upload keeps it in dn.scratch)
    try {
      c->dense_host.resize(size_t(n * n));
    } catch (const std::bad_alloc&) {
      return fail(c, DCX_E_OOM, "host allocation failed");
    }
    if (!c->dn.scratch || c->dn.scratch_bytes < size_t(n * n) * 8) return fail(c, DCX_E_STATE, "dense coupling not on the device");
    const cudaError_t e = cudaMemcpy(c->dense_host.data(), c->dn.scratch, size_t(n * n) * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(c, DCX_E_CUDA, cudaGetErrorString(e));
  }
  const double* A = c->dense_host.data();
  std::vector<int64_t> ro(n + 1, 0), ci;
  std::vector<double> vv;
  try {
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t j = 0; j < n; ++j) {
        const double a = A[i * n + j];
        if (i != j && a != 0.0) {
          ci.push_back(j);
          vv.push_back(a);
        }
      }
      ro[i + 1] = (int64_t)ci.size();
    }
  } catch (const std::bad_alloc&) {
    return fail(c, DCX_E_OOM, "host allocation failed");
  }
  const int rc = upload_csr(c, n, (int64_t)ci.size(), ro.data(), ci.data(), vv.data(), n, 0);
  if (rc == DCX_OK) c->csr_ready = true;
  return rc;
}

int dcx_set_dense(dcx_ctx* c, int64_t n, const double* A) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (!A || n < 1) return fail(c, DCX_E_INVALID, "bad dense coupling");
  for (int64_t i = 0; i < n; ++i)
    if (A[i * n + i] != 0.0) return fail(c, DCX_E_INVALID, "diagonal must be zero");
  return guarded(c, [&] {
    c->have = false;
    c->proc = false;
    c->csr_ready = false;
    c->chunks.release();
    c->dense_host.clear();  // no 8 n^2-byte host copy per upload: ensure_csr reads the device copy
    c->n = n;
    c->n_cols = n;
    c->row_base = 0;
    c->nnz = n * (n - 1);  // upper bound until the CSR form is built
    // J = scale * q with int8 q (the K2000 instance: 1/2 x {0, -1}), classified on every host
    // thread into the pinned staging: 1 byte per entry crosses PCIe instead of 8
    PhaseClock pc("set_dense");
    const int64_t tot = n * n;
    bool done = false;
    if (tot >= 4096) {
      if (c->pin_bytes < size_t(tot)) {
        if (c->pin) cudaFreeHost(c->pin);
        c->pin = nullptr;
        c->pin_bytes = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->pin), size_t(tot), cudaHostAllocDefault));
        c->pin_bytes = size_t(tot);
      }
      int8_t* q = reinterpret_cast<int8_t*>(c->pin);
      // one pass per candidate scale: the first nonzero |J| (the K2000 instance: 1/2), then
      // 1 and 1/2; each pass checks J = scale * q with |q| <= 127 and writes q
      double first = 0.0;
      for (int64_t k = 0; k < tot && first == 0.0; ++k) first = std::fabs(A[k]);
      const int T = int(std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency())));
      for (double cand : {first, 1.0, 0.5}) {
        if (!(cand > 0.0) || !std::isfinite(cand)) continue;
        std::vector<unsigned char> ok(64, 1);
        // J = cand * r exactly with |r| <= 127 (r found with the reciprocal, checked by the
        // product: the device operand cand * q reproduces every entry bit for bit)
        const double inv = 1.0 / cand;
        par_for(tot, [&](int64_t lo, int64_t hi, int t) {
          bool g = true;
          stream_fill(q, lo, hi, [&](int64_t k) {
            const double r = rne(A[k] * inv);
            g &= std::fabs(r) <= 127.0 && r * cand == A[k];
            return int8_t(r);
          });
          ok[t] = g;
        }, T);
        if (std::all_of(ok.begin(), ok.end(), [](unsigned char b) { return b != 0; })) {
          pc.mark("classify");
          // candidates coarser than the true grid are rejected above; a finer-than-needed one
          // (first > min |J|) cannot pass, so cand is the operand scale
          dense_upload_int8(c->dn, n, q, cand, c->stream);
          pc.mark("upload+operands");
          done = true;
          break;
        }
      }
    }
    if (!done) dense_upload(c->dn, n, A, c->stream);
    c->dense = true;
    c->have = true;
  });
}

int dcx_set_procedural(dcx_ctx* c, int64_t n, int64_t seed, int32_t formula) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (n < 2) return fail(c, DCX_E_INVALID, "procedural matrices need n >= 2");
  if (n >= (int64_t(1) << 31)) return fail(c, DCX_E_INVALID, "n >= 2^31 is not supported");
  if (formula != DCX_FORMULA_SIN_PRODUCT) return fail(c, DCX_E_INVALID, "unknown procedural formula");
  const double top = double(n - 1) * double(n - 1) + std::fabs(double(seed));
  if (top >= 9.2e18) return fail(c, DCX_E_INVALID, "i*j + seed must fit in int64");
  return guarded(c, [&] {
    c->have = false;
    c->dense = false;
    c->csr_ready = false;
    c->chunks.release();
    c->dense_host.clear();
    c->dn.release();
    c->rp.release();
    c->col.release();
    c->col16.release();
    c->vint.release();
    c->v64.release();
    c->v32.release();
    c->n = n;
    c->n_cols = n;
    c->row_base = 0;
    c->nnz = n * (n - 1);
    c->vk_int = -1;
    c->scale = 1.0;
    c->V32 = 1;
    c->ell_entries = 0;
    c->es_row_bound = 0;
    c->proc = true;
    c->proc_seed = seed;
    c->have = true;
  });
}

int dcx_proc_row_stats(dcx_ctx* c, double* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    require_coupling(c);
    if (!c->proc) throw InvalidArg("the coupling is not procedural");
    const int64_t n = c->n;
    DevBuf& tmp = c->scratch;
    if (tmp.bytes < size_t(n) * 24) tmp.alloc(size_t(n) * 24);
    launch_proc_row_stats(n, c->proc_seed, tmp.as<double>(), c->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp.p, size_t(n) * 24, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

// Row statistics of a stored coupling over j != i: (sum J_ij, sum J_ij^2, sum |J_ij|) per row,
// the inputs of offdiag_moments and abs_row_sums (dc/coupling.py:104-109 dense,
// :197-206 CSR) for derive_params' Wigner estimate and beta (dc/spectral.py:175-189, 246-247).
// Each row is summed sequentially in column order (numpy's bincount order for CSR).
namespace {
__global__ void csr_row_stats(const uint32_t* rp, const int32_t* col, const void* val, int vk, double scale,
                              int64_t n, int64_t row_base, double* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s1 = 0.0, s2 = 0.0, sa = 0.0;
    for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
      double v;
      if (vk == VK_UNIFORM) v = scale;
      else if (vk == VK_I8) v = scale * double(reinterpret_cast<const int8_t*>(val)[e]);
      else if (vk == VK_I16) v = scale * double(reinterpret_cast<const int16_t*>(val)[e]);
      else v = reinterpret_cast<const double*>(val)[e];
      if (int64_t(col[e]) == row_base + i) continue;  // the diagonal is excluded (zero for valid couplings)
      s1 += v;
      s2 += v * v;
      sa += fabs(v);
    }
    out[3 * i] = s1;
    out[3 * i + 1] = s2;
    out[3 * i + 2] = sa;
  }
}
__global__ void dense_row_stats(const double* A, int64_t n, double* out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; i < n;
       i += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    double s1 = 0.0, s2 = 0.0, sa = 0.0;
    for (int64_t j = lane; j < n; j += 32) {  // lane-strided, then a fixed-order warp tree
      const double v = j == i ? 0.0 : A[i * n + j];
      s1 += v;
      s2 += v * v;
      sa += fabs(v);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    sa = warp_sum(sa);
    if (lane == 0) {
      out[3 * i] = s1;
      out[3 * i + 1] = s2;
      out[3 * i + 2] = sa;
    }
  }
}
}  // namespace

int dcx_row_stats(dcx_ctx* c, double* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    require_coupling(c);
    const int64_t n = c->n;
    DevBuf& tmp = c->scratch;
    if (c->proc) {
      if (tmp.bytes < size_t(n) * 24) tmp.alloc(size_t(n) * 24);
      launch_proc_row_stats(n, c->proc_seed, tmp.as<double>(), c->stream);
    } else if (c->dense) {
      // the f64 coupling as uploaded stays in dn.scratch; row stats go to a separate buffer
      if (!c->dn.scratch || c->dn.scratch_bytes < size_t(n * n) * 8) throw InvalidArg("dense coupling not on the device");
      if (tmp.bytes < size_t(n) * 24) tmp.alloc(size_t(n) * 24);
      dense_row_stats<<<int(std::min<int64_t>((n + 7) / 8, 148 * 16)), 256, 0, c->stream>>>(
          static_cast<const double*>(c->dn.scratch), n, tmp.as<double>());
    } else {
      if (tmp.bytes < size_t(n) * 24) tmp.alloc(size_t(n) * 24);
      const void* val = c->vk_int >= 0 ? c->vint.p : c->v64.p;
      const int vk = c->vk_int >= 0 ? c->vk_int : VK_F64;
      csr_row_stats<<<grid_for(n), 256, 0, c->stream>>>(c->rp.as<uint32_t>(), c->col.as<int32_t>(), val, vk,
                                                       c->scale, n, c->row_base, tmp.as<double>());
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp.p, size_t(n) * 24, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dcx_coupling(const dcx_ctx* c, dcx_coupling_info* out) {
  if (!c || !out) return fail(nullptr, DCX_E_INVALID, "null argument");
  if (!c->have) return fail(const_cast<dcx_ctx*>(c), DCX_E_STATE, "no coupling set");
  out->n = c->n;
  out->nnz = c->nnz;
  out->value_kind = c->proc ? VK_PROC : (c->vk_int >= 0 ? c->vk_int : VK_F64);
  out->lanes = c->V32;
  out->scale = c->scale;
  out->dense = c->dense ? 1 : 0;
  out->lattice_L = int32_t(c->torus_L);
  return DCX_OK;
}

int dcx_matvec(dcx_ctx* c, int32_t R, const double* v, double* out, int32_t precision) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    require_coupling(c);
    if (ensure_csr(c) != DCX_OK) throw CudaError(c->err);
    if (R < 1 || !v || !out) throw InvalidArg("bad matvec arguments");
    if (precision == DCX_PREC_F32) apply_impl<float>(c, R, nullptr, nullptr, v, out, nullptr, nullptr, nullptr, nullptr);
    else apply_impl<double>(c, R, nullptr, nullptr, v, out, nullptr, nullptr, nullptr, nullptr);
  });
}

int dcx_apply(dcx_ctx* c, int32_t R, const double* alpha, const double* beta, const double* v, double* tx,
              double* h, int32_t precision) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    require_coupling(c);
    if (ensure_csr(c) != DCX_OK) throw CudaError(c->err);
    if (R < 1 || !v || !alpha || !beta) throw InvalidArg("bad apply arguments");
    for (int r = 0; r < R; ++r)
      if (!(alpha[r] > 0) || !(beta[r] > 0)) throw InvalidArg("alpha and beta must be positive");
    if (precision == DCX_PREC_F32) apply_impl<float>(c, R, alpha, beta, v, nullptr, tx, h, nullptr, nullptr);
    else apply_impl<double>(c, R, alpha, beta, v, nullptr, tx, h, nullptr, nullptr);
  });
}

int dcx_energy(dcx_ctx* c, int32_t R, const int8_t* spins, double* energies) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    require_coupling(c);
    if (ensure_csr(c) != DCX_OK) throw CudaError(c->err);
    if (R < 1 || !spins || !energies) throw InvalidArg("bad energy arguments");
    apply_impl<double>(c, R, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, spins, energies);
  });
}

// ------------------------------------------------------------------ solve
static void build_graph(dcx_ctx* c) {
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  cudaGraph_t gr;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  for (int it = 0; it < c->chunk; ++it) enqueue_iteration(c->mp, c->stream);
  CK(cudaStreamEndCapture(c->stream, &gr));
  CK(cudaGraphInstantiate(&c->graph, gr, 0));
  cudaGraphDestroy(gr);
}

static void drain(dcx_ctx* c);

// Shared by dcx_solve_begin and dcx_dist_begin (xe0 / xe1: the caller's iterate
// buffers of a row-partitioned run, else NULL).
static void begin_impl(dcx_ctx* c, const dcx_params* P, int32_t R, const double* alpha, const double* beta,
                       const double* x0, void* xe0, void* xe1) {
    const bool dist = xe0 != nullptr;
    require_coupling(c);
    if (!dist && (c->row_base != 0 || c->n_cols != c->n))
      throw InvalidArg("the coupling is a row block: use dcx_dist_begin");
    if (dist) {
      if (c->dense) throw InvalidArg("row-partitioned runs need a CSR row block");
      if (P->precision == DCX_PREC_F16TC) throw InvalidArg("row-partitioned runs use precision f64 or f32");
      if (P->path == DCX_PATH_PERSISTENT || P->path == DCX_PATH_DENSE_TC)
        throw InvalidArg("row-partitioned runs use the multipass path");
      if (P->solver == DCX_SOLVER_ADOCH && P->window_mode == DCX_WINDOW_EXACT)
        throw InvalidArg("row-partitioned ADOCH supports window_mode 'economy'");
    }
    if (!P || !alpha || !beta || !x0) throw InvalidArg("null argument");
    if (R < 1) throw InvalidArg("R must be >= 1");
    if (P->solver != DCX_SOLVER_DOCH && P->solver != DCX_SOLVER_ADOCH) throw InvalidArg("unknown solver");
    if (P->window_mode != DCX_WINDOW_ECONOMY && P->window_mode != DCX_WINDOW_EXACT)
      throw InvalidArg("window_mode must be 'economy' or 'exact'");
    if (P->lookback_q < 1) throw InvalidArg("lookback_q must be >= 1");
    if (P->max_iters < 0 || P->max_iters > (int64_t(1) << 30)) throw InvalidArg("max_iters out of range");
    if (P->trace_stride < 1) throw InvalidArg("trace_stride must be >= 1");
    for (int r = 0; r < R; ++r)
      if (!(alpha[r] > 0) || !(beta[r] > 0)) throw InvalidArg("alpha and beta must be positive");
    PhaseClock pc("begin");
    if (c->hist_inflight) {  // the last run's history copy still reads `hist`
      CK(cudaEventSynchronize(c->hist_copied));
      c->hist_inflight = false;
    }
    c->prm = *P;
    c->R = R;
    c->begun = false;
    c->finished = false;
    const int64_t n = c->n;
    const bool use_tc = P->precision == DCX_PREC_F16TC;
    if (!use_tc && ensure_csr(c) != DCX_OK) throw CudaError(c->err);
    if (use_tc && !c->dense) throw InvalidArg("the tensor-core path needs a dense coupling");
    if (c->proc && P->path == DCX_PATH_PERSISTENT) throw InvalidArg("procedural couplings run on the multipass path");
    c->f64 = P->precision == DCX_PREC_F64;
    const size_t tb = c->f64 ? 8 : 4;
    c->J = csr_view(c, c->f64);
    c->sp = plan_small(c->J, P->solver, P->window_mode, c->f64);
    pc.mark("views");
    c->dist = dist;
    if (dist) c->path = DCX_PATH_MULTIPASS;
    else if (use_tc) c->path = DCX_PATH_DENSE_TC;
    else if (P->path == DCX_PATH_PERSISTENT) {
      if (!c->sp.fits) throw InvalidArg("instance too large for the persistent path");
      c->path = DCX_PATH_PERSISTENT;
    } else if (P->path == DCX_PATH_MULTIPASS) c->path = DCX_PATH_MULTIPASS;
    else if (P->path == DCX_PATH_DENSE_TC) throw InvalidArg("tensor-core path needs precision F16TC");
    else c->path = c->sp.fits ? DCX_PATH_PERSISTENT : DCX_PATH_MULTIPASS;
    // history ring
    const int64_t total_hist = int64_t(1) << 21;
    int64_t cap = std::min<int64_t>(P->max_iters + 1, std::max<int64_t>(1024, total_hist / R));
    c->cap = (int)cap;
    c->wcap = (int)std::min<int64_t>(int64_t(P->lookback_q) + 1, P->max_iters + 1);
    if (c->path == DCX_PATH_MULTIPASS) c->chunk = P->chunk > 0 ? P->chunk : 32;
    else c->chunk = P->chunk > 0 ? P->chunk : (int)cap;
    c->chunk = (int)std::min<int64_t>(c->chunk, cap);
    if (c->chunk < 1) c->chunk = 1;
    // buffers
    const int64_t tot = n * R;
    // three iterate buffers for DOCH on the CSR passes (pass_r1 / pass_r1w / pass_rv): x_{p-2}
    // survives pass p, so the best-spin copy of x_q is made only when x_{q+1} does not improve on
    // it -- at the end of an improvement streak, not after every improvement.
    // Not on the row-partitioned (caller's two buffers), procedural, column-chunked or stencil
    // passes; DCX_XBUF3=0 keeps two.
    auto env_is = [](const char* k, const char* v) { const char* e = std::getenv(k); return e && std::strcmp(e, v) == 0; };
    int nbuf = (c->path == DCX_PATH_MULTIPASS && !dist && P->solver == DCX_SOLVER_DOCH && !c->proc &&
                !std::getenv("DCX_CHUNKS") && !env_is("DCX_TORUS", "1") && !env_is("DCX_XBUF3", "0"))
                   ? 3 : 2;
    if (const char* e = std::getenv("DCX_XBUF"); e && nbuf > 2) nbuf = std::max(2, std::min(4, std::atoi(e)));
    if (dist) {
      c->xb0.release();
      c->xb1.release();
      c->xb2.release();
      c->xb3.release();
    } else {
      c->xb0.alloc(tot * tb);
      c->xb1.alloc(tot * tb);
      if (nbuf >= 3) c->xb2.alloc(tot * tb); else c->xb2.release();
      if (nbuf >= 4) c->xb3.alloc(tot * tb); else c->xb3.release();
    }
    const bool ad = P->solver == DCX_SOLVER_ADOCH;
    if (ad) { c->ax0.alloc(tot * tb); c->ax1.alloc(tot * tb); } else { c->ax0.release(); c->ax1.release(); }
    if (ad && P->window_mode == DCX_WINDOW_EXACT) c->ay.alloc(tot * tb); else c->ay.release();
    c->best.alloc(tot);
    c->ctl.alloc(sizeof(RepCtl) * R);
    c->g.alloc(sizeof(GState));
    c->hist.alloc(sizeof(HistRec) * R * cap);
    c->window.alloc(sizeof(double) * R * std::max(1, c->wcap));
    c->states.release();
    if (P->record_states) {
      const double bytes = double(P->max_iters + 1) * double(tot) * double(tb);
      if (bytes > 4e9) throw InvalidArg("record_states would need more than 4 GB; lower max_iters");
      c->states.alloc(size_t(bytes));
    }
    // partial slots
    c->mp = MultiPass{};
    c->mp.f64 = c->f64;
    c->mp.solver = P->solver;
    c->mp.vk = c->J.vk;
    c->mp.V = c->J.V;
    int slots;
    if (c->proc) {
      c->mp.grid = proc_pass_grid(n);  // pass_proc: grid.x row blocks, grid.y replica chunks
      slots = c->mp.grid;
    } else if (R == 1) {
      c->mp.grid = c->J.grid;
      slots = c->mp.grid;  // one partial slot per block (pass_r1)
    } else {
      // pass_rv: grid.y = replica chunks, grid.x = row blocks, one partial slot per row block;
      // two resident 256-thread blocks per SM (the kernel needs up to 128 registers)
      const int vw = replica_vector_width(R, c->f64);
      const int chunks = (R + 32 * vw - 1) / (32 * vw);
      const int per_sm = (vw * (c->f64 ? 8 : 4) >= 16) ? 2 : 3;  // resident blocks (pass_rv launch bounds)
      c->mp.grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, std::max(1, 148 * per_sm / chunks)));
      slots = c->mp.grid;
    }
    // a row-partitioned run may split its pass into two row ranges (dcx_dist_pass_rows):
    // each writes its own half of the slots, zero until written
    if (dist) slots *= 2;
    c->part.alloc(sizeof(double) * R * NQ * slots);
    if (dist) CK(cudaMemsetAsync(c->part.p, 0, c->part.bytes, c->stream));
    {
      int64_t fthreads = std::min<int64_t>(std::max<int64_t>(tot, R), int64_t(148) * 8 * 256);
      int fg = (int)((fthreads + 255) / 256);
      if ((int64_t)fg * 256 < R) fg = (R + 255) / 256;
      c->mp.fgrid = fg;
      c->mp.sslots = R == 1 ? fg * 8 : (fg * 256) / R;
      c->spart.alloc(sizeof(double) * std::max(1, c->mp.sslots) * R);
      CK(cudaMemsetAsync(c->spart.p, 0, c->spart.bytes, c->stream));
    }
    PassArgs& a = c->mp.args;
    a.rp = c->J.rp;
    a.col = c->J.col;
    a.val = c->J.val;
    a.scale = c->J.scale;
    a.ctl = c->ctl.as<RepCtl>();
    a.g = c->g.as<GState>();
    a.nbuf = nbuf;
    a.x[2] = a.gx[2] = a.x[3] = a.gx[3] = nullptr;
    if (dist) {  // own rows start at row_base of the caller's [n_cols][R] buffers
      a.gx[0] = xe0;
      a.gx[1] = xe1;
      a.x[0] = static_cast<char*>(xe0) + size_t(c->row_base) * R * tb;
      a.x[1] = static_cast<char*>(xe1) + size_t(c->row_base) * R * tb;
    } else {
      a.x[0] = a.gx[0] = c->xb0.p;
      a.x[1] = a.gx[1] = c->xb1.p;
      if (nbuf >= 3) a.x[2] = a.gx[2] = c->xb2.p;
      if (nbuf >= 4) a.x[3] = a.gx[3] = c->xb3.p;
    }
    a.ax[0] = c->ax0.p;
    a.ax[1] = c->ax1.p;
    a.ay = c->ay.p;
    a.best = c->best.as<int8_t>();
    a.states = c->states.p;
    a.part = c->part.as<double>();
    a.slots = slots;
    a.xmap[0] = a.xmap[1] = a.xmap[2] = nullptr;
    a.proc_seed = c->J.proc_seed;
    a.torus_L = (!dist && c->torus_L > 0 && !c->proc) ? int32_t(c->torus_L) : 0;
    a.bond_r = c->bond_r.as<int8_t>();
    a.bond_d = c->bond_d.as<int8_t>();
    a.sgnw[0] = a.sgnw[1] = nullptr;
    a.chunks = ChunkArgs{};
    if (!dist && R == 1 && !c->f64 && !c->proc && (c->vk_int == VK_UNIFORM || c->vk_int == VK_I8)) {
      const int C = chunk_count(n);
      if (C != c->chunks.C)
        build_chunk_plan(c->chunks, c->J.rp, c->J.col, c->vk_int == VK_I8 ? static_cast<const int8_t*>(c->J.val) : nullptr,
                         n, c->nnz, C, c->stream);
      if (c->chunks.C > 0) {
        CK(cudaMemsetAsync(c->chunks.acc, 0, size_t(n) * sizeof(float2), c->stream));
        a.chunks = c->chunks;
      }
    }
    if (a.torus_L > 0 && R > 1 && !c->f64) {
      const size_t words = size_t(n) * 4 * size_t((R + 127) / 128);
      c->sgn0.alloc(words * 4);
      c->sgn1.alloc(words * 4);
      a.sgnw[0] = c->sgn0.as<uint32_t>();
      a.sgnw[1] = c->sgn1.as<uint32_t>();
    } else {
      c->sgn0.release();
      c->sgn1.release();
    }
    if (R > 1 && !c->proc && replica_vector_width(R, c->f64) > 1) {
      const char* e = std::getenv("DCX_RV_TMA");
      if (!(e && std::atoi(e) == 0)) {
        alignas(64) unsigned char maps[4][128] = {};
        const int vw = replica_vector_width(R, c->f64);
        for (int k = 0; k < nbuf; ++k)
          encode_row_gather_map(maps[k], a.gx[k], uint64_t(R), uint64_t(c->n_cols), c->f64, uint32_t(32 * vw));
        c->xmaps.alloc(sizeof(maps));
        CK(cudaMemcpy(c->xmaps.p, maps, sizeof(maps), cudaMemcpyHostToDevice));
        for (int k = 0; k < 4; ++k) a.xmap[k] = k < nbuf ? static_cast<char*>(c->xmaps.p) + 128 * k : nullptr;
      }
    }
    // pass_rv lanes sum the spin energy of ceil(n / (8 grid)) rows; integer couplings keep that exact in f32
    a.es_f32 = (R > 1 && c->vk_int >= 0 &&
                double((n + 8 * int64_t(c->mp.grid) - 1) / (8 * int64_t(c->mp.grid))) * c->es_row_bound < 16777216.0)
                   ? 1 : 0;
    RunCfg& cfg = a.cfg;
    cfg.n = n;
    cfg.R = R;
    cfg.solver = P->solver;
    cfg.window_mode = P->window_mode;
    cfg.lookback_q = P->lookback_q;
    cfg.max_iters = P->max_iters;
    cfg.stride = P->trace_stride;
    cfg.budget = P->time_budget_s;
    cfg.conv_tol = P->conv_tol;
    cfg.descent_tol = P->descent_tol;
    cfg.momentum_floor = 0.0;
    if (P->solver == DCX_SOLVER_ADOCH && P->precision != DCX_PREC_F64) {
      // relative step (to sqrt(alpha / beta)) below which f32 / tensor-core ADOCH takes plain
      // steps; DCX_ADOCH_FLOOR overrides, 0 keeps the momentum to the end
      const char* e = std::getenv("DCX_ADOCH_FLOOR");
      cfg.momentum_floor = e ? std::atof(e) : 2e-3;
    }
    cfg.hist_cap = (int)cap;
    cfg.wcap = std::max(1, c->wcap);
    cfg.es_scale = use_tc ? c->dn.jscale_d : (c->vk_int >= 0 ? c->scale : 1.0);
    cfg.hist = c->hist.as<HistRec>();
    cfg.window = c->window.as<double>();
    c->mp.spart = c->spart.as<double>();
    // initial state
    {
      DevBuf& src = c->scratch;
      if (src.bytes < size_t(tot) * 8) src.alloc(size_t(tot) * 8);
      if (c->f64) {
        CK(cudaMemcpyAsync(src.p, x0, tot * 8, cudaMemcpyHostToDevice, c->stream));
        to_device_layout<double><<<grid_for(tot), 256, 0, c->stream>>>(src.as<double>(), static_cast<double*>(a.x[0]), n, R);
      } else {
        // f32 runs start from x0 rounded to f32 (round to nearest either side): round on all
        // host threads into the pinned staging and move half the bytes at the DMA rate
        const size_t bytes = size_t(tot) * 4;
        if (c->pin_bytes < bytes) {
          if (c->pin) cudaFreeHost(c->pin);
          c->pin = nullptr;
          c->pin_bytes = 0;
          CK(cudaHostAlloc(reinterpret_cast<void**>(&c->pin), bytes, cudaHostAllocDefault));
          c->pin_bytes = bytes;
        }
        float* x32 = reinterpret_cast<float*>(c->pin);
        // in pieces: the DMA of piece i overlaps the rounding of piece i + 1
        const int64_t piece = std::max<int64_t>(int64_t(1) << 18, (tot / 8 + 63) / 64 * 64);
        for (int64_t k0 = 0; k0 < tot; k0 += piece) {
          const int64_t m = std::min(piece, tot - k0);
          par_for(m, [&](int64_t lo, int64_t hi, int) {
            stream_fill(x32 + k0, lo, hi, [&](int64_t k) { return float(x0[k0 + k]); });
          }, 16);
          CK(cudaMemcpyAsync(src.as<float>() + k0, x32 + k0, size_t(m) * 4, cudaMemcpyHostToDevice, c->stream));
        }
        pc.mark("x0 to f32 + H2D issue");
        if (timing_on()) {
          CK(cudaStreamSynchronize(c->stream));
          pc.mark("x0 H2D");
        }
        to_device_layout_s<float, float><<<grid_for(tot), 256, 0, c->stream>>>(src.as<float>(), static_cast<float*>(a.x[0]), n, R);
        if (timing_on()) {
          CK(cudaStreamSynchronize(c->stream));
          pc.mark("x0 layout");
        }
      }
      CK(cudaMemsetAsync(a.x[1], 0, tot * tb, c->stream));
      for (int k = 2; k < 4; ++k)
        if (a.x[k]) CK(cudaMemsetAsync(a.x[k], 0, tot * tb, c->stream));
      if (ad) {
        CK(cudaMemsetAsync(c->ax0.p, 0, tot * tb, c->stream));
        CK(cudaMemsetAsync(c->ax1.p, 0, tot * tb, c->stream));
      }
      CK(cudaMemsetAsync(c->best.p, 1, tot, c->stream));
      if (c->states.p) CK(cudaMemcpyAsync(c->states.p, a.x[0], tot * tb, cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      pc.mark("x0 upload");
    }
    std::vector<RepCtl> h(R);
    for (int r = 0; r < R; ++r) {
      RepCtl& q = h[r];
      std::memset(&q, 0, sizeof(q));
      q.alpha = alpha[r];
      q.beta = beta[r];
      q.best = std::numeric_limits<double>::infinity();
      q.t = 1.0;
      q.k = -1;
      q.status = DCX_STOP_RUNNING;
      q.best_iter = -1;
      q.pend = -1;
      q.accept = 1;
      q.warned = -1;
    }
    CK(cudaMemcpyAsync(c->ctl.p, h.data(), sizeof(RepCtl) * R, cudaMemcpyHostToDevice, c->stream));
    c->hg = GState{};
    c->hg.p = 0;
    c->hg.live = 1;
    c->hg.running = R;
    CK(cudaMemcpyAsync(c->g.p, &c->hg, sizeof(GState), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->ring_direct = cap >= P->max_iters + 1;
    c->hcnt.assign(R, 0);
    c->hh.resize(c->ring_direct ? 0 : R);  // keep each replica's capacity across runs
    for (auto& v : c->hh) {
      v.clear();
      v.reserve(std::min<int64_t>(P->max_iters + 1, 4096));
    }
    c->hctl = h;
    // a ring a detached result still reads is left to it: take a free one (or allocate)
    const size_t need = size_t(R) * cap;
    if (!c->ringp || c->ringp.use_count() > 1 || c->ringp->n < need) {
      if (c->ringp && c->ringp.use_count() > 1) c->spare.push_back(c->ringp);
      c->ringp.reset();
      for (auto& sp : c->spare)
        if (sp && sp.use_count() == 1 && sp->n >= need) {
          c->ringp = sp;
          sp.reset();
          break;
        }
      c->spare.erase(std::remove_if(c->spare.begin(), c->spare.end(),
                                    [](const std::shared_ptr<PinnedRing>& q) { return !q || q.use_count() == 1; }),
                     c->spare.end());  // free rings that no result holds (a fitting one was taken)
      if (!c->ringp) {
        auto r = std::make_shared<PinnedRing>();
        CK(cudaHostAlloc(reinterpret_cast<void**>(&r->p), sizeof(HistRec) * need, cudaHostAllocDefault));
        r->n = need;
        c->ringp = r;
      }
    }
    c->ring = c->ringp->p;
    c->ring_n = c->ringp->n;
    c->p_host = 0;
    pc.mark("state+ring");
    if (c->path == DCX_PATH_MULTIPASS && !dist) build_graph(c);
    if (c->path == DCX_PATH_DENSE_TC) dense_begin(c->dn, c->mp, c->stream);
    pc.mark("graph/dense_begin");
    CK(cudaEventRecord(c->ev0, c->stream));
    enqueue_start_clock(c->g.as<GState>(), c->stream);
    CK(cudaGetLastError());
    c->begun = true;
}

int dcx_solve_begin(dcx_ctx* c, const dcx_params* P, int32_t R, const double* alpha, const double* beta,
                    const double* x0) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] { begin_impl(c, P, R, alpha, beta, x0, nullptr, nullptr); });
}

int dcx_stream(dcx_ctx* c, void** stream) {
  if (!c || !stream) return fail(c, DCX_E_INVALID, "null argument");
  *stream = static_cast<void*>(c->stream);
  return DCX_OK;
}

int dcx_dist_begin(dcx_ctx* c, const dcx_params* P, int32_t R, const double* alpha, const double* beta,
                   const double* x0_rows, void* x_buf0, void* x_buf1, double* q_sum, double* q_max) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (!x_buf0 || !x_buf1 || !q_sum || !q_max) return fail(c, DCX_E_INVALID, "null buffer");
  return guarded(c, [&] {
    begin_impl(c, P, R, alpha, beta, x0_rows, x_buf0, x_buf1);
    c->qs = q_sum;
    c->qm = q_max;
  });
}

int dcx_dist_pass(dcx_ctx* c) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun || !c->dist || c->finished) throw InvalidArg("no row-partitioned run in progress");
    enqueue_dist_pass(c->mp, c->qs, c->qm, c->stream);
    CK(cudaGetLastError());
  });
}

int dcx_dist_pass_rows(dcx_ctx* c, int64_t row_lo, int64_t row_hi, int32_t half) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun || !c->dist || c->finished) throw InvalidArg("no row-partitioned run in progress");
    if (row_lo < 0 || row_hi < row_lo || row_hi > c->n || (half != 0 && half != 1))
      throw InvalidArg("row range outside the block");
    if (row_hi > row_lo) enqueue_dist_pass_rows(c->mp, row_lo, row_hi, half, c->stream);
    CK(cudaGetLastError());
  });
}

int dcx_dist_reduce(dcx_ctx* c) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun || !c->dist || c->finished) throw InvalidArg("no row-partitioned run in progress");
    enqueue_dist_reduce(c->mp, c->qs, c->qm, c->stream);
    CK(cudaGetLastError());
  });
}

int dcx_dist_control(dcx_ctx* c) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun || !c->dist || c->finished) throw InvalidArg("no row-partitioned run in progress");
    enqueue_dist_control(c->mp, c->qs, c->qm, c->stream);
    CK(cudaGetLastError());
  });
}

int dcx_dist_poll(dcx_ctx* c, int32_t* live, int64_t* passes) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun || !c->dist) throw InvalidArg("no row-partitioned run");
    if (!c->finished) drain(c);
    if (live) *live = (!c->finished && c->hg.live != 0 && c->hg.running > 0) ? 1 : 0;
    if (passes) *passes = c->hg.p;
  });
}

int dcx_dist_finish(dcx_ctx* c) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun || !c->dist) throw InvalidArg("no row-partitioned run");
    if (c->finished) return;
    CK(cudaEventRecord(c->ev1, c->stream));
    enqueue_flush(c->mp, c->stream);
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->dev_seconds = ms * 1e-3;
    drain(c);
    c->finished = true;
  });
}

static void pull_ctl(dcx_ctx* c) {
  CK(cudaMemcpyAsync(c->hctl.data(), c->ctl.p, sizeof(RepCtl) * c->R, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&c->hg, c->g.p, sizeof(GState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// new history records -> the pinned ring. defer: the last drain of a run whose records
// sit in place in the ring (ring_direct) leaves the copy in flight (PinnedRing::wait)
static void copy_hist(dcx_ctx* c, bool defer) {
  const int R = c->R;
  // new history entries: k in [lo, hi] over all replicas (replicas advance in lockstep)
  int64_t lo = std::numeric_limits<int64_t>::max(), hi = -1;
  for (int r = 0; r < R; ++r) {
    const int64_t kr = c->hctl[r].k;
    const int64_t done = c->nhist(r);
    if (kr >= done) {
      lo = std::min(lo, done);
      hi = std::max(hi, kr);
    }
  }
  if (hi < 0) return;
  const size_t rec = sizeof(HistRec);
  const size_t pitch = rec * c->cap;
  const bool async = defer && c->ring_direct;
  cudaStream_t cs = async ? c->hstream : c->stream;
  auto copy_cols = [&](int64_t k0, int64_t k1) {  // ring columns [k0, k1] without wrap
    CK(cudaMemcpy2DAsync(c->ring + k0, pitch, c->hist.as<HistRec>() + k0, pitch, rec * (k1 - k0 + 1), R,
                         cudaMemcpyDeviceToHost, cs));
  };
  c->ringp->wait();  // an earlier deferred copy into this ring
  if (async) {
    CK(cudaEventRecord(c->hist_go, c->stream));
    CK(cudaStreamWaitEvent(c->hstream, c->hist_go, 0));
  }
  if (hi - lo + 1 >= c->cap) copy_cols(0, c->cap - 1);
  else {
    const int64_t a = lo % c->cap, b = hi % c->cap;
    if (a <= b) copy_cols(a, b);
    else { copy_cols(a, c->cap - 1); copy_cols(0, b); }
  }
  if (async) {
    c->ringp->mark_pending(c->hstream);
    CK(cudaEventRecord(c->hist_copied, c->hstream));
    c->hist_inflight = true;
  } else {
    CK(cudaStreamSynchronize(c->stream));
  }
  for (int r = 0; r < R; ++r) {
    const int64_t kr = c->hctl[r].k;
    if (c->ring_direct) {
      c->hcnt[r] = std::max<int64_t>(c->hcnt[r], kr + 1);
      continue;
    }
    auto& v = c->hh[r];
    for (int64_t k = (int64_t)v.size(); k <= kr; ++k) v.push_back(c->ring[(size_t)r * c->cap + (k % c->cap)]);
  }
}

static void drain(dcx_ctx* c) {
  pull_ctl(c);
  copy_hist(c, false);
}

int dcx_solve_step(dcx_ctx* c, int32_t* live) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->begun) throw InvalidArg("dcx_solve_begin has not been called");
    if (c->finished) {
      if (live) *live = 0;
      return;
    }
    if (c->path == DCX_PATH_MULTIPASS) {
      CK(cudaGraphLaunch(c->graph, c->stream));
    } else if (c->path == DCX_PATH_PERSISTENT) {
      const int p_end = (int)std::min<int64_t>(c->p_host + c->chunk, c->prm.max_iters + 1);
      launch_small(c->mp, c->J, c->sp, p_end, c->stream);
      CK(cudaGetLastError());
      c->p_host = p_end;
      GState tmp{};
      // advance the shared pass counter for the next chunk (running is kept)
      CK(cudaMemcpyAsync(&c->hg, c->g.p, sizeof(GState), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      tmp = c->hg;
      tmp.p = p_end;
      tmp.live = tmp.running > 0 ? 1 : 0;
      CK(cudaMemcpyAsync(c->g.p, &tmp, sizeof(GState), cudaMemcpyHostToDevice, c->stream));
    } else {
      dense_step(c->dn, c->mp, c->chunk, c->stream);
    }
    CK(cudaGetLastError());
    // device time of the solve ends with the last compute launch; history / result
    // downloads that follow belong to the end-to-end time only
    CK(cudaEventRecord(c->ev1, c->stream));
    pull_ctl(c);
    bool alive = c->hg.live != 0 && c->hg.running > 0;
    if (c->path == DCX_PATH_PERSISTENT && c->p_host >= c->prm.max_iters + 1) alive = false;
    if (!alive) {
      if (c->path == DCX_PATH_MULTIPASS) enqueue_flush(c->mp, c->stream);
      if (c->path == DCX_PATH_DENSE_TC) dense_finish(c->dn, c->mp, c->stream);
      CK(cudaStreamSynchronize(c->stream));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      c->dev_seconds = ms * 1e-3;
      pull_ctl(c);
      c->finished = true;
    }
    copy_hist(c, !alive);
    if (live) *live = alive ? 1 : 0;
  });
}

int dcx_solve_run(dcx_ctx* c) {
  PhaseClock pc("run");
  int32_t live = 1;
  while (live) {
    int rc = dcx_solve_step(c, &live);
    if (rc != DCX_OK) return rc;
  }
  pc.mark("steps");
  return DCX_OK;
}

int dcx_result_summary(dcx_ctx* c, int32_t r, dcx_summary* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  if (!c->begun) return fail(c, DCX_E_STATE, "no run");
  if (r < 0 || r >= c->R) return fail(c, DCX_E_INVALID, "replica index out of range");
  const RepCtl& q = c->hctl[r];
  out->iterations = std::max(0, q.k);
  out->stop_reason = q.status;
  out->best_iter = q.best_iter;
  out->best_energy = q.best;
  out->n_hist = c->nhist(r);
  out->descent_warn = q.warned;
  out->path_used = c->path;
  return DCX_OK;
}

int dcx_result_history(dcx_ctx* c, int32_t r, int64_t from, int64_t count, double* h, double* e, double* t,
                       int32_t* ev) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (!c->begun || r < 0 || r >= c->R) return fail(c, DCX_E_INVALID, "bad replica");
  if (c->ringp) c->ringp->wait();
  if (from < 0 || count < 0 || from + count > c->nhist(r)) return fail(c, DCX_E_INVALID, "history range");
  for (int64_t k = 0; k < count; ++k) {
    const HistRec& q = c->rec(r, from + k);
    if (h) h[k] = q.h;
    if (e) e[k] = q.e;
    if (t) t[k] = q.t;
    if (ev) ev[k] = q.ev;
  }
  return DCX_OK;
}

int dcx_result_summaries(dcx_ctx* c, int64_t* iterations, int32_t* stop_reason, double* best_energy,
                         int64_t* n_hist, int32_t* descent_warn) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (!c->begun) return fail(c, DCX_E_STATE, "no run");
  for (int r = 0; r < c->R; ++r) {
    const RepCtl& q = c->hctl[r];
    if (iterations) iterations[r] = std::max(0, q.k);
    if (stop_reason) stop_reason[r] = q.status;
    if (best_energy) best_energy[r] = q.best;
    if (n_hist) n_hist[r] = c->nhist(r);
    if (descent_warn) descent_warn[r] = q.warned;
  }
  return DCX_OK;
}

int dcx_result_history_all(dcx_ctx* c, int64_t K, double* h, double* e, double* t, int32_t* ev) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (!c->begun) return fail(c, DCX_E_STATE, "no run");
  if (c->ringp) c->ringp->wait();
  auto rows = [&](int r0, int r1) {
    for (int r = r0; r < r1; ++r) {
      const int64_t cnt = std::min<int64_t>(K, c->nhist(r));
      const int64_t base = (int64_t)r * K;
      if (c->ring_direct && h && e && t && ev) {  // records in place in the pinned ring: one tight de-interleave
        const HistRec* q = c->ring + size_t(r) * c->cap;
        double *hp = h + base, *ep = e + base, *tp = t + base;
        int32_t* vp = ev + base;
        for (int64_t k = 0; k < cnt; ++k) {
          hp[k] = q[k].h;
          ep[k] = q[k].e;
          tp[k] = q[k].t;
          vp[k] = q[k].ev;
        }
        continue;
      }
      for (int64_t k = 0; k < cnt; ++k) {
        const HistRec& q = c->rec(r, k);
        if (h) h[base + k] = q.h;
        if (e) e[base + k] = q.e;
        if (t) t[base + k] = q.t;
        if (ev) ev[base + k] = q.ev;
      }
    }
  };
  // a bulk download of many replicas (K2000 x 1024: 1e6 records) is split over host threads
  const int R = c->R;
  const int64_t work = int64_t(R) * K;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = int(std::min<int64_t>({int64_t(hw), 8, work / 65536 + 1, int64_t(R)}));
  if (nt <= 1) {
    rows(0, R);
    return DCX_OK;
  }
  std::vector<std::thread> pool;
  for (int i = 1; i < nt; ++i) pool.emplace_back(rows, int(int64_t(R) * i / nt), int(int64_t(R) * (i + 1) / nt));
  rows(0, int(int64_t(R) / nt));
  for (auto& th : pool) th.join();
  return DCX_OK;
}

int dcx_result_best_spins(dcx_ctx* c, int8_t* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    if (!c->begun) throw InvalidArg("no run");
    const int64_t n = c->n, R = c->R;
    DevBuf& tmp = c->scratch;
    if (tmp.bytes < size_t(n * R)) tmp.alloc(size_t(n * R));
    gather_best<<<grid_for(n * R), 256, 0, c->stream>>>(c->best.as<int8_t>(), n, (int)R, tmp.as<int8_t>());
    CK(cudaMemcpyAsync(out, tmp.p, n * R, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dcx_result_state(dcx_ctx* c, double* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    if (!c->begun) throw InvalidArg("no run");
    const int64_t n = c->n, R = c->R, tot = n * R;
    DevBuf& tmp = c->scratch;
    if (tmp.bytes < size_t(tot) * 8) tmp.alloc(size_t(tot) * 8);
    if (c->f64)
      gather_final_state<double><<<grid_for(tot), 256, 0, c->stream>>>(
          static_cast<const double*>(c->mp.args.x[0]), static_cast<const double*>(c->mp.args.x[1]),
          static_cast<const double*>(c->mp.args.x[2]), static_cast<const double*>(c->mp.args.x[3]), c->mp.args.nbuf,
          c->ctl.as<RepCtl>(),
          n, (int)R, tmp.as<double>());
    else
      gather_final_state<float><<<grid_for(tot), 256, 0, c->stream>>>(
          static_cast<const float*>(c->mp.args.x[0]), static_cast<const float*>(c->mp.args.x[1]),
          static_cast<const float*>(c->mp.args.x[2]), static_cast<const float*>(c->mp.args.x[3]), c->mp.args.nbuf,
          c->ctl.as<RepCtl>(),
          n, (int)R, tmp.as<double>());
    CK(cudaMemcpyAsync(out, tmp.p, tot * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int dcx_result_states(dcx_ctx* c, int32_t r, double* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    if (!c->begun || !c->states.p) throw InvalidArg("states were not recorded");
    if (r < 0 || r >= c->R) throw InvalidArg("replica index out of range");
    const int64_t n = c->n, R = c->R, tot = n * R;
    const size_t tb = c->f64 ? 8 : 4;
    const int64_t K = std::max(0, c->hctl[r].k) + 1;
    std::vector<unsigned char> tmp(K * tot * tb);
    CK(cudaMemcpyAsync(tmp.data(), c->states.p, K * tot * tb, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t k = 0; k < K; ++k)
      for (int64_t i = 0; i < n; ++i) {
        const int64_t idx = k * tot + i * R + r;
        out[k * n + i] = c->f64 ? reinterpret_cast<const double*>(tmp.data())[idx]
                                : double(reinterpret_cast<const float*>(tmp.data())[idx]);
      }
  });
}

int dcx_profile_kernel(dcx_ctx* c, int32_t launches, double* ms_per_launch, int32_t* kernel_id) {
  if (!c || !ms_per_launch) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    if (!c->begun || c->finished) throw InvalidArg("profile needs a freshly begun run");
    if (launches < 1) throw InvalidArg("launches must be >= 1");
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    int kid = 0;
    // one warm launch, then the timed ones (same input every launch: the pass
    // counter does not advance without the control kernel)
    if (c->path == DCX_PATH_MULTIPASS) {
      enqueue_pass_only(c->mp, c->stream);
      CK(cudaEventRecord(a, c->stream));
      for (int i = 0; i < launches; ++i) enqueue_pass_only(c->mp, c->stream);
      CK(cudaEventRecord(b, c->stream));
      kid = 1;
    } else if (c->path == DCX_PATH_DENSE_TC) {
      // every timed launch runs the same window, iterations [0, it) from the initial
      // states (no replica has converged yet, so every replica-iteration is live work):
      // the run state is reset from the begin-time copies between launches, outside the events
      const std::vector<RepCtl> ctl0 = c->hctl;
      const GState g0 = c->hg;
      float total = 0.f;
      for (int l = 0; l <= launches; ++l) {  // launch 0 warms up
        CK(cudaMemcpyAsync(c->ctl.p, ctl0.data(), sizeof(RepCtl) * c->R, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->g.p, &g0, sizeof(GState), cudaMemcpyHostToDevice, c->stream));
        dense_begin(c->dn, c->mp, c->stream);
        enqueue_start_clock(c->g.as<GState>(), c->stream);
        dense_profile(c->dn, c->mp, a, b, c->stream);
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (l > 0) total += ms;
      }
      CK(cudaEventRecord(a, c->stream));
      CK(cudaEventRecord(b, c->stream));
      kid = 3;
      c->prof_ms = total;
    } else {
      throw InvalidArg("profiling covers the multipass and dense paths");
    }
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (kid == 3) ms = c->prof_ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_per_launch = double(ms) / launches;
    if (kernel_id) *kernel_id = kid;
    c->finished = true;
    c->begun = false;
  });
}

int dcx_power(dcx_ctx* c, int32_t use_shift, double shift, double tol, int64_t max_iters, const double* restart,
              double* mag, double* rayleigh, int64_t* iterations, int32_t* converged) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    require_coupling(c);
    if (c->row_base != 0 || c->n_cols != c->n) throw InvalidArg("power iteration needs the whole coupling");
    if (c->proc) throw InvalidArg("device power iteration needs a stored coupling (procedural: dcx_matvec)");
    if (!restart || max_iters < 0) throw InvalidArg("bad power-iteration arguments");
    if (ensure_csr(c) != DCX_OK) throw CudaError(c->err);
    const CsrDev J = csr_view(c, true);
    const int64_t n = c->n;
    int dev = 0, blocks_per_sm = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    blocks_per_sm = 1;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(sms) * blocks_per_sm, (n + 7) / 8));
    DevBuf v, w, rs, part, part2, bar, out;
    v.alloc(n * 8);
    w.alloc(n * 8);
    rs.alloc(n * 8);
    part.alloc(size_t(grid) * 16);
    part2.alloc(size_t(grid) * 8);
    bar.alloc(8);
    out.alloc(32);
    CK(cudaMemcpyAsync(rs.p, restart, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(bar.p, 0, 8, c->stream));
    launch_power(J, use_shift, shift, tol, max_iters, v.as<double>(), w.as<double>(), rs.as<double>(),
                 part.as<double>(), part2.as<double>(), bar.as<unsigned>(), out.as<double>(), grid, c->stream);
    CK(cudaGetLastError());
    double h[4];
    CK(cudaMemcpyAsync(h, out.p, 32, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (mag) *mag = h[0];
    if (rayleigh) *rayleigh = h[1];
    if (iterations) *iterations = int64_t(h[2]);
    if (converged) *converged = int32_t(h[3]);
  });
}

int dcx_result_device_seconds(dcx_ctx* c, double* out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  *out = c->dev_seconds;
  return DCX_OK;
}

// ------------------------------------------------------------ generation / ingest (dcx_gen.cu)
}  // extern "C"

// ---------------------------------------------------------------- detached results
struct dcx_result {
  int device = 0;
  int64_t n = 0;
  int R = 0, cap = 0;
  bool ring_direct = false;
  std::shared_ptr<PinnedRing> ring;
  std::vector<std::vector<HistRec>> hh;
  std::vector<int64_t> hcnt;
  std::vector<double> warn_delta;
  std::shared_ptr<SharedDev> x, best;  // gathered [R][n]: final states (f64), best spins (int8)
  std::string err;
  int64_t nhist(int r) const { return ring_direct ? hcnt[r] : (int64_t)hh[r].size(); }
  const HistRec& rec(int r, int64_t k) const { return ring_direct ? ring->p[size_t(r) * cap + k] : hh[r][k]; }
};

namespace {
// a result-owned device buffer of at least `bytes`, reusing one no live result holds
std::shared_ptr<SharedDev> take_dev(dcx_ctx* c, size_t bytes) {
  for (auto& d : c->dspare)
    if (d && d.use_count() == 1 && d->bytes >= bytes) return d;
  c->dspare.erase(std::remove_if(c->dspare.begin(), c->dspare.end(),
                                 [](const std::shared_ptr<SharedDev>& d) { return !d || d.use_count() == 1; }),
                  c->dspare.end());
  auto d = std::make_shared<SharedDev>();
  cudaError_t e = cudaMalloc(&d->p, std::max<size_t>(bytes, 1));
  if (e != cudaSuccess) {
    d->p = nullptr;
    cudaGetLastError();
    throw std::runtime_error(std::string("OOM: result buffer: ") + cudaGetErrorString(e));
  }
  d->bytes = bytes;
  c->dspare.push_back(d);
  return d;
}

template <class Src>
void history_rows(const Src& src, int R, int64_t K, double* h, double* e, double* t, int32_t* ev) {
  auto rows = [&](int r0, int r1) {
    for (int r = r0; r < r1; ++r) {
      const int64_t cnt = std::min<int64_t>(K, src.nhist(r));
      const int64_t base = (int64_t)r * K;
      for (int64_t k = 0; k < cnt; ++k) {
        const HistRec& q = src.rec(r, k);
        if (h) h[base + k] = q.h;
        if (e) e[base + k] = q.e;
        if (t) t[base + k] = q.t;
        if (ev) ev[base + k] = q.ev;
      }
    }
  };
  const int64_t work = int64_t(R) * K;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = int(std::min<int64_t>({int64_t(hw), 8, work / 65536 + 1, int64_t(R)}));
  if (nt <= 1) {
    rows(0, R);
    return;
  }
  std::vector<std::thread> pool;
  for (int i = 1; i < nt; ++i) pool.emplace_back(rows, int(int64_t(R) * i / nt), int(int64_t(R) * (i + 1) / nt));
  rows(0, int(int64_t(R) / nt));
  for (auto& th : pool) th.join();
}
}  // namespace

extern "C" {

int dcx_result_detach(dcx_ctx* c, dcx_result** out) {
  if (!c || !out) return fail(c, DCX_E_INVALID, "null argument");
  *out = nullptr;
  if (!c->begun) return fail(c, DCX_E_STATE, "no run");
  auto res = std::unique_ptr<dcx_result>(new (std::nothrow) dcx_result());
  if (!res) return fail(c, DCX_E_OOM, "host allocation failed");
  int rc = guarded(c, [&] {
    const int64_t n = c->n, R = c->R, tot = n * R;
    res->device = c->device;
    res->n = n;
    res->R = int(R);
    res->x = take_dev(c, size_t(tot) * 8);
    res->best = take_dev(c, size_t(tot));
    if (c->f64)
      gather_final_state<double><<<grid_for(tot), 256, 0, c->stream>>>(
          static_cast<const double*>(c->mp.args.x[0]), static_cast<const double*>(c->mp.args.x[1]),
          static_cast<const double*>(c->mp.args.x[2]), static_cast<const double*>(c->mp.args.x[3]), c->mp.args.nbuf,
          c->ctl.as<RepCtl>(),
          n, (int)R, static_cast<double*>(res->x->p));
    else
      gather_final_state<float><<<grid_for(tot), 256, 0, c->stream>>>(
          static_cast<const float*>(c->mp.args.x[0]), static_cast<const float*>(c->mp.args.x[1]),
          static_cast<const float*>(c->mp.args.x[2]), static_cast<const float*>(c->mp.args.x[3]), c->mp.args.nbuf,
          c->ctl.as<RepCtl>(),
          n, (int)R, static_cast<double*>(res->x->p));
    gather_best<<<grid_for(tot), 256, 0, c->stream>>>(c->best.as<int8_t>(), n, (int)R, static_cast<int8_t*>(res->best->p));
    CK(cudaGetLastError());
    res->ring_direct = c->ring_direct;
    res->cap = c->cap;
    if (c->ring_direct) {
      res->ring = c->ringp;  // the context takes another ring for its next run
      res->hcnt = c->hcnt;
    } else {
      res->hh = c->hh;  // (runs longer than the ring: the drained copies)
    }
    res->warn_delta.assign(R, std::numeric_limits<double>::quiet_NaN());
    if (c->ring_direct) {  // from the device records: the history copy may still be in flight
      if (c->wdelta_n < size_t(R)) {
        if (c->wdelta) cudaFreeHost(c->wdelta);
        c->wdelta = nullptr;
        c->wdelta_n = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->wdelta), size_t(R) * 8, cudaHostAllocMapped));
        c->wdelta_n = size_t(R);
      }
      double* wd = nullptr;
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&wd), c->wdelta, 0));
      gather_warn_delta<<<int((R + 255) / 256), 256, 0, c->stream>>>(c->hist.as<HistRec>(), c->ctl.as<RepCtl>(),
                                                                    c->cap, int(R), wd);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(c->stream));
      std::copy(c->wdelta, c->wdelta + R, res->warn_delta.begin());
    } else {
      for (int r = 0; r < R; ++r) {
        const int k = c->hctl[r].warned;
        if (k >= 1 && k < res->nhist(r)) res->warn_delta[r] = res->rec(r, k).h - res->rec(r, k - 1).h;
      }
    }
    CK(cudaStreamSynchronize(c->stream));
  });
  if (rc == DCX_OK) *out = res.release();
  return rc;
}

}  // extern "C"

namespace {
template <typename F>
int res_guarded(dcx_result* res, F&& f) {
  if (!res) return fail(nullptr, DCX_E_INVALID, "result is NULL");
  try {
    CK(cudaSetDevice(res->device));
    f();
    return DCX_OK;
  } catch (const std::exception& e) {
    res->err = e.what();
    return fail(nullptr, DCX_E_CUDA, e.what());
  }
}
}  // namespace

extern "C" {

int dcx_res_state(dcx_result* res, double* out) {
  return res_guarded(res, [&] {
    if (!out) throw std::runtime_error("null output");
    CK(cudaMemcpy(out, res->x->p, size_t(res->n) * res->R * 8, cudaMemcpyDeviceToHost));
  });
}

int dcx_res_best_spins(dcx_result* res, int8_t* out) {
  return res_guarded(res, [&] {
    if (!out) throw std::runtime_error("null output");
    CK(cudaMemcpy(out, res->best->p, size_t(res->n) * res->R, cudaMemcpyDeviceToHost));
  });
}

int dcx_res_history_all(dcx_result* res, int64_t K, double* h, double* e, double* t, int32_t* ev) {
  if (!res) return fail(nullptr, DCX_E_INVALID, "result is NULL");
  if (res->ring) res->ring->wait();
  history_rows(*res, res->R, K, h, e, t, ev);
  return DCX_OK;
}

int dcx_res_warn_delta(dcx_result* res, double* out) {
  if (!res || !out) return fail(nullptr, DCX_E_INVALID, "null argument");
  std::copy(res->warn_delta.begin(), res->warn_delta.end(), out);
  return DCX_OK;
}

void dcx_result_free(dcx_result* res) {
  if (!res) return;
  cudaSetDevice(res->device);
  delete res;
}

int dcx_gen_sparse_9bit(dcx_ctx* c, int64_t n, int64_t n_p, uint64_t seed, int64_t* nnz) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    gen_sparse_9bit(n, n_p, seed, c->gen, c->stream);
    if (nnz) *nnz = c->gen.nnz;
  });
}

int dcx_gen_result(dcx_ctx* c, int64_t* ro, int64_t* col, double* val) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  return guarded(c, [&] {
    if (!c->gen.ro) throw InvalidArg("no generated coupling (dcx_gen_sparse_9bit)");
    if (!ro || (c->gen.nnz && (!col || !val))) throw InvalidArg("null output array");
    CK(cudaMemcpyAsync(ro, c->gen.ro, sizeof(int64_t) * (c->gen.n + 1), cudaMemcpyDeviceToHost, c->stream));
    if (c->gen.nnz) {
      CK(cudaMemcpyAsync(col, c->gen.col, sizeof(int64_t) * c->gen.nnz, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(val, c->gen.val, sizeof(double) * c->gen.nnz, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    c->gen.release();
  });
}

int dcx_validate_csr(dcx_ctx* c, int64_t n, int64_t nnz, const int64_t* ro, const int64_t* col, const double* val,
                     int32_t* check, int64_t* row, int32_t* all_int) {
  if (!c) return fail(nullptr, DCX_E_INVALID, "ctx is NULL");
  if (!ro || !check || !row || !all_int || (nnz > 0 && (!col || !val))) return fail(c, DCX_E_INVALID, "null argument");
  return guarded(c, [&] {
    if (n < 1 || nnz < 0) throw InvalidArg("n must be >= 1 and nnz >= 0");
    int ai = 0;
    *check = validate_csr_device(n, nnz, ro, col, val, row, &ai, c->stream);
    *all_int = ai;
  });
}

}  // extern "C"
