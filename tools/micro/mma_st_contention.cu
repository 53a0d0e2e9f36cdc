// Does concurrent tcgen05.st traffic (dequant warps) slow tcgen05.mma issue/completion?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
template <bool TS, bool WARP = false>
__global__ void __launch_bounds__(512, 1) k(int n, int iters, int st_warps, volatile int* stop, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { done = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp == 15) {
    if (WARP || (threadIdx.x & 31) == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
      const uint32_t base = su32(sm);
      uint32_t ph = 0; long long tissue = 0, ttot = 0;
      for (int it = 0; it < iters; ++it) {
        long long t0 = clock64();
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = desc(base + 16384 + (kk / 4) * 16384 + (kk % 4) * 32);
          if (TS && WARP) asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 384), "r"(tm + kk * 8), "l"(bd), "r"(idesc), "r"(kk) : "memory");
          else if (TS) asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 384), "r"(tm + kk * 8), "l"(bd), "r"(idesc), "r"(kk) : "memory");
          else { const uint64_t ad = desc(base + (kk / 4) * 8192 + (kk % 4) * 32);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm + 384), "l"(ad), "l"(bd), "r"(idesc), "r"(kk) : "memory"); }
        }
        if (WARP) asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&bar)) : "memory");
        else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        long long t1 = clock64();
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(&bar)), "r"(ph) : "memory");
        ph ^= 1; tissue += t1 - t0; ttot += clock64() - t0;
      }
      if ((threadIdx.x & 31) == 0) { out[2 * blockIdx.x] = tissue / iters; out[2 * blockIdx.x + 1] = ttot / iters; done = 1; }
    }
  } else if (warp < st_warps) {
    uint32_t v[16]; for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
    const uint32_t addr = tm + ((uint32_t)((warp & 3) * 32) << 16) + 64 + (warp >> 2) * 64;
    while (!done) {
      for (int x = 0; x < 4; ++x)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(addr + x * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                       "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[0]++;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 148); unsigned long long h[2];
  int* stop; cudaMalloc(&stop, 4);
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(k<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int stw : {0, 4, 12}) for (int n : {16, 128}) {
    k<true><<<148, 512, 96 * 1024>>>(n, 300, stw, stop, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("TS N=%3d st_warps=%2d: issue %llu cycles, issue+complete %llu (%s)\n", n, stw, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    k<false><<<148, 512, 96 * 1024>>>(n, 300, stw, stop, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("SS N=%3d st_warps=%2d: issue %llu cycles, issue+complete %llu\n", n, stw, h[0], h[1]);
    k<true, true><<<148, 512, 96 * 1024>>>(n, 300, stw, stop, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("TS-warp N=%3d st_warps=%2d: issue %llu cycles, issue+complete %llu (%s)\n", n, stw, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
