// Microbenchmark: back-to-back tcgen05.mma issue rate from resident shared memory
// (no TMA), cta_group::2, M = 256, N = 128 / 256, kind::f16 (K16) and kind::f8f6f4 (K32).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
template <int KIND>
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (KIND == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  // A: 4 atoms of 128 rows x 128 B (64 KB); B: 4 atoms of N/2 rows x 128 B
  const int bytes = 4 * 16384 + 4 * (N / 2) * 128;
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = KIND == 0 ? 0x3C003C00u : 0x38383838u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_f16(256, N);
  const uint32_t sa = smem_u32(base), sb = sa + 4 * 16384;
  if (rank == 0 && threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma2<KIND>(tmem, sw128_desc(sa + q * 16384 + k * 32), sw128_desc(sb + q * (N / 2) * 128 + k * 32), idesc,
                     (it | q | k) ? 1u : 0u);
    const long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)), "h"(uint16_t(3)) : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar)), "r"(0) : "memory");
    const long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  } else if (rank == 1 && threadIdx.x == 0) {
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar)), "r"(0) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int KIND, int N>
void run(const char* name, int grid) {
  long long* d;
  cudaMalloc(&d, 16);
  const int smem = 4 * 16384 + 4 * (N / 2) * 128 + 1024;
  cudaFuncSetAttribute(bench<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 256;
  for (int rep = 0; rep < 3; ++rep) {
    bench<KIND, N><<<grid, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  }
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double mmas = iters * 16.0;
  printf("%-28s grid %3d: issue %.1f cyc/MMA, complete %.1f cyc/MMA (ideal %d)\n", name, grid, h[0] / mmas, h[1] / mmas,
         256 * N / 512);
  cudaFree(d);
}

int main() {
  for (int grid : {2, 128, 148}) {
    run<0, 128>("f16 M256 N128 K16", grid);
    run<1, 128>("e4m3 M256 N128 K32", grid);
    run<0, 256>("f16 M256 N256 K16", grid);
    run<1, 256>("e4m3 M256 N256 K32", grid);
  }
  return 0;
}
