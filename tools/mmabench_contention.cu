// tcgen05.mma issue rate (M256 N128, cta_group::2, e4m3 K32) from resident smem, alone and with
// concurrent bulk-async global->smem copies into another smem region (the kernel's TMA ingress).
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
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(a), "r"(ph) : "memory");
}

template <int CE, int LAYOUT = 0, bool RANDOM = false, int SPIN = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) bench(int iters, int copy_kb, const char* gsrc, long long* out, int tmem_ld) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar, cbar, sbar[8];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int opbytes = 4 * 16384 + 4 * 8192;  // A 64 KB + B 32 KB (resident operands)
  for (int i = threadIdx.x; i < opbytes / 4; i += blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    // RANDOM: e4m3 bytes of random sign and magnitude in [2^-6, 2^3) (no NaN), like the deltas
    reinterpret_cast<uint32_t*>(base)[i] = RANDOM ? ((h & 0x3f3f3f3fu) | 0x08080808u) ^ (h & 0x80808080u) : 0x38383838u;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar)), "r"(1) : "memory");
    for (int k = 0; k < 8; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sbar[k])), "r"(1) : "memory");
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
  const uint32_t idesc = idesc_f16(256, 128);
  const uint32_t sa = smem_u32(base), sb = sa + 4 * 16384;
  const uint32_t cdst = sa + opbytes;  // copy target region: 96 KB after the operands
  if (threadIdx.x == 32 && copy_kb > 0) {
    // bulk copies of 16 KB chunks, 6 in flight, for the duration of the MMAs
    uint32_t ph = 0;
    const int nchunks = iters * copy_kb / 16;
    for (int c = 0; c < nchunks; c += 6) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&cbar)), "r"(6 * 16384) : "memory");
      for (int k = 0; k < 6; ++k)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(cdst + k * 16384),
                     "l"(gsrc + (size_t(blockIdx.x) * 6 + k) * 16384), "r"(16384), "r"(smem_u32(&cbar)) : "memory");
      mbar_wait(smem_u32(&cbar), ph);
      ph ^= 1;
    }
  }
  __shared__ __align__(8) uint64_t spinbar;
  __shared__ volatile int done;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&spinbar)), "r"(1) : "memory");
    done = 0;
  }
  __syncthreads();
  if (SPIN && threadIdx.x >= 128 && (threadIdx.x & 31) == 0 && ((threadIdx.x >> 5) - 4) < SPIN) {
    // one lane per spinning warp polls an mbarrier phase that does not complete (as the kernel's
    // producer / MMA issuer / epilogue do while they wait)
    while (!done) {
      uint32_t ok;
      asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                   : "=r"(ok) : "r"(smem_u32(&spinbar)), "r"(0) : "memory");
    }
  }
  if (tmem_ld && threadIdx.x >= 128) {
    // 4 warps (one per TMEM lane quadrant) read 3 x 16 columns and write 2 x 16 back, in a loop,
    // from columns 256.. (not the accumulator): the update's TMEM traffic
    const int w = (threadIdx.x >> 5) & 3;
    const uint32_t ta = tmem + (uint32_t(w * 32) << 16) + 256;
    uint32_t acc = 0;
    for (int it = 0; it < iters * tmem_ld; ++it) {
      uint32_t v[16];
      for (int c = 0; c < 3; ++c) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                     "tcgen05.wait::ld.sync.aligned;"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(ta + 16 * ((it + c) & 7)) : "memory");
        for (int j = 0; j < 16; ++j) acc += v[j];
      }
      for (int c = 0; c < 2; ++c)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + 128 + 16 * c),
                     "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc),
                     "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    if (acc == 0x12345) out[1] = acc;
  }
  if (rank == 0 && threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t acc = (it | q | k) ? 1u : 0u;
          const uint32_t aa = LAYOUT == 0 ? sa + q * 16384 : sa + (q >> 1) * 49152 + (q & 1) * 16384;
          const uint32_t bb = LAYOUT == 0 ? sb + q * 8192 : sa + (q >> 1) * 49152 + 32768 + (q & 1) * 8192;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                       "l"(sw128_desc(aa + k * 32)), "l"(sw128_desc(bb + k * 32)), "r"(idesc), "r"(acc) : "memory");
        }
        // a completion signal every CE MMAs (CE = 4: per atom, 8: per 2-atom stage as the kernel, 16: per 4 atoms)
        if (CE == 4 || (CE == 8 && (q & 1)) || (CE == 16 && q == 3))
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                           smem_u32(&sbar[q])), "h"(uint16_t(3)) : "memory");
      }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)), "h"(uint16_t(3)) : "memory");
    mbar_wait(smem_u32(&bar), 0);
    out[0] = clock64() - t0;
    done = 1;
  } else if (rank == 1 && threadIdx.x == 0) {
    mbar_wait(smem_u32(&bar), 0);
    done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// 8 MMAs per stage, commit per stage to sbar[k % 4], wait for stage k - DEPTH + 1 before issuing
// stage k + 1: the ring turnaround without TMA (MMA completion -> mbarrier -> waiting thread)
__device__ __forceinline__ void mbar_wait_test(uint32_t a, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nWT_%=:\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WT_%=;\n}\n" ::"r"(a), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_wait_hint(uint32_t a, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nWH_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 1000000;\n@!P1 bra WH_%=;\n}\n" ::"r"(a), "r"(ph) : "memory");
}
template <int DEPTH, int WAITMODE = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) ringbench(int stages, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[8];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * 8192) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x38383838u;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[k])), "r"(1) : "memory");
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
  const uint32_t tmem = tmem_base, idesc = idesc_f16(256, 128);
  const uint32_t sa = smem_u32(base), sb = sa + 4 * 16384;
  if (rank == 0 && threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int k = 0; k < stages; ++k) {
      if (k >= DEPTH) {
        if (WAITMODE == 0) mbar_wait(smem_u32(&bar[(k - DEPTH) & 7]), ((k - DEPTH) >> 3) & 1);
        else if (WAITMODE == 1) mbar_wait_hint(smem_u32(&bar[(k - DEPTH) & 7]), ((k - DEPTH) >> 3) & 1);
        else if (WAITMODE == 2) mbar_wait_test(smem_u32(&bar[(k - DEPTH) & 7]), ((k - DEPTH) >> 3) & 1);
        else if ((k & 3) == 0) mbar_wait(smem_u32(&bar[(k - DEPTH) & 7]), ((k - DEPTH) >> 3) & 1);  // every 4th stage
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const uint32_t acc = (k | m) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(sw128_desc(sa + (m >> 2) * 16384 + (m & 3) * 32)), "l"(sw128_desc(sb + (m >> 2) * 8192 + (m & 3) * 32)), "r"(idesc),
                     "r"(acc) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                       smem_u32(&bar[k & 7])), "h"(uint16_t(3)) : "memory");
    }
    for (int k = (stages > DEPTH ? stages - DEPTH : 0); k < stages; ++k) mbar_wait(smem_u32(&bar[k & 7]), (k >> 3) & 1);
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  {
    long long* dd;
    cudaMalloc(&dd, 16);
    const int sm = 4 * 16384 + 4 * 8192 + 1024;
    cudaFuncSetAttribute(ringbench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(ringbench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(ringbench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(ringbench<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(ringbench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int rep = 0; rep < 2; ++rep) { ringbench<4, 1><<<128, 128, sm>>>(512, dd); cudaDeviceSynchronize(); }
    {
      long long h;
      cudaMemcpy(&h, dd, 8, cudaMemcpyDeviceToHost);
      printf("commit/wait ring depth 4, try_wait with suspend-time hint: %.1f cycles per stage\n", h / 512.0);
    }
    cudaFuncSetAttribute(ringbench<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(ringbench<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int wm : {2, 3}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (wm == 2) ringbench<4, 2><<<128, 128, sm>>>(512, dd);
        else ringbench<4, 3><<<128, 128, sm>>>(512, dd);
        cudaDeviceSynchronize();
      }
      long long h;
      cudaMemcpy(&h, dd, 8, cudaMemcpyDeviceToHost);
      printf("commit/wait ring depth 4, %s: %.1f cycles per stage\n", wm == 2 ? "test_wait loop" : "wait every 4th stage", h / 512.0);
    }
    for (int rep = 0; rep < 2; ++rep) { ringbench<8><<<128, 128, sm>>>(512, dd); cudaDeviceSynchronize(); }
    {
      long long h;
      cudaMemcpy(&h, dd, 8, cudaMemcpyDeviceToHost);
      printf("commit/wait ring depth 8: %.1f cycles per stage\n", h / 512.0);
    }
    for (int depth : {1, 2, 4}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (depth == 1) ringbench<1><<<128, 128, sm>>>(512, dd);
        else if (depth == 2) ringbench<2><<<128, 128, sm>>>(512, dd);
        else ringbench<4><<<128, 128, sm>>>(512, dd);
        cudaDeviceSynchronize();
      }
      long long h;
      cudaMemcpy(&h, dd, 8, cudaMemcpyDeviceToHost);
      printf("commit/wait ring depth %d (8 MMAs per stage): %.1f cycles per stage\n", depth, h / 512.0);
    }
  }
  long long* d;
  cudaMalloc(&d, 16);
  char* g;
  cudaMalloc(&g, size_t(148) * 6 * 16384);
  cudaMemset(g, 0x38, size_t(148) * 6 * 16384);
  const int smem = 4 * 16384 + 4 * 8192 + 6 * 16384 + 1024;
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<8, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<8, 1, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<8, 1, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int sp : {1, 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      if (sp == 1) bench<8, 1, false, 1><<<128, 256, smem>>>(256, 0, g, d, 0);
      else bench<8, 1, false, 4><<<128, 256, smem>>>(256, 0, g, d, 0);
      cudaDeviceSynchronize();
    }
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%d warp(s) spinning on mbarrier.try_wait: %.1f cycles per MMA\n", sp, h / (256 * 16.0));
  }
  for (int rep = 0; rep < 2; ++rep) {
    bench<8, 1, true><<<128, 256, smem>>>(256, 0, g, d, 0);
    cudaDeviceSynchronize();
  }
  {
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("kernel stage layout, random e4m3 operands: %.1f cycles per MMA\n", h / (256 * 16.0));
  }
  const int iters = 256;
  for (int rep = 0; rep < 2; ++rep) {
    bench<8, 1><<<128, 256, smem>>>(iters, 0, g, d, 0);
    cudaDeviceSynchronize();
  }
  {
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("kernel stage layout (A A B B per 48 KB), commit per 8: %.1f cycles per MMA\n", h / (iters * 16.0));
  }
  
  for (int ce : {4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      if (ce == 4) bench<4><<<128, 256, smem>>>(iters, 0, g, d, 0);
      else if (ce == 8) bench<8><<<128, 256, smem>>>(iters, 0, g, d, 0);
      else bench<16><<<128, 256, smem>>>(iters, 0, g, d, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("commit (multicast arrive) every %2d MMAs: %.1f cycles per MMA\n", ce, h / (iters * 16.0));
  }
  for (int mode = 0; mode < 6; ++mode) {
    const int copy_kb = mode < 3 ? 0 : 96, tl = (mode % 3 == 0) ? 0 : (mode % 3 == 1 ? 1 : 4);
    for (int rep = 0; rep < 2; ++rep) {
      bench<0><<<128, 256, smem>>>(iters, copy_kb, g, d, tl);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("copy %3d KB / 16 MMAs, TMEM ld/st rounds %d per 16 MMAs: %.1f cycles per MMA (M256 N128 e4m3 K32)\n", copy_kb, tl, h / (iters * 16.0));
  }
  return 0;
}
