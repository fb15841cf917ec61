// Host->device copy rate of pinned staging right after the host wrote it: one thread, 16 threads with
// plain stores, 16 / 4 threads with streaming stores (DESIGN.md §5 "Host staging"). Build and run on the
// GPU box: nvcc -O2 -o h2d tools/h2d_after_host_writes.cu && ./h2d
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <emmintrin.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  const size_t n = 8 << 20;
  void* d; cudaMalloc(&d, 64 << 20);
  for (int flags : {0, 4 /*WC*/}) {
    char* h; cudaHostAlloc((void**)&h, 64 << 20, flags);
    memset(h, 0, 64 << 20);
    for (int mode = 0; mode < 6; ++mode) {
      double tw = 0, tc = 0;
      for (int it = 0; it < 20; ++it) {
        double t0 = now();
        if (mode == 1) memset(h, it, n);
        if (mode == 2) {
          std::vector<std::thread> th;
          for (int t = 0; t < 16; ++t) th.emplace_back([&, t] { memset(h + t * (n / 16), it, n / 16); });
          for (auto& x : th) x.join();
        }
        if (mode == 3) {  // write 16 MB elsewhere first (evict), then rewrite
          memset(h + (32 << 20), it, 32 << 20);
          memset(h, it, n);
        }
        if (mode == 4 || mode == 5) {  // 16 threads, streaming stores (mode 5: 4 threads)
          const int T = mode == 4 ? 16 : 4;
          std::vector<std::thread> th;
          for (int t = 0; t < T; ++t) th.emplace_back([&, t, T] {
            __m128i v = _mm_set1_epi8(char(it));
            __m128i* p = reinterpret_cast<__m128i*>(h + t * (n / T));
            for (size_t k = 0; k < n / T / 16; ++k) _mm_stream_si128(p + k, v);
            _mm_sfence();
          });
          for (auto& x : th) x.join();
        }
        double t1 = now();
        cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        double t2 = now();
        if (it >= 2) { tw += t1 - t0; tc += t2 - t1; }
      }
      printf("flags %d mode %d: write %.3f ms  copy %.3f ms (%.1f GB/s)\n", flags, mode, tw / 18 * 1e3, tc / 18 * 1e3, n / (tc / 18) / 1e9);
    }
    cudaFreeHost(h);
  }
  return 0;
}
