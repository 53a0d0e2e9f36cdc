// Microbenchmark: latency of tcgen05.mma (kind::f16, M=128, N in {16,64,128,256})
// issued in a chunk of 8 (K=128) followed by tcgen05.commit -> mbarrier wait.
// A from TMEM (TS) vs A from SMEM (SS).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
template <bool TS>
__global__ void __launch_bounds__(128, 1) mma_kernel(int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t base = su32(sm);
    uint32_t ph = 0;
    long long tsum = 0;
    for (int it = 0; it < iters; ++it) {
      long long t0 = clock64();
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = desc(base + 16384 + (k / 4) * 16384 + (k % 4) * 32);
        if (TS) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 256), "r"(tm + k * 8), "l"(bd), "r"(idesc), "r"(k) : "memory");
        } else {
          const uint64_t ad = desc(base + (k / 4) * 8192 + (k % 4) * 32);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm + 256), "l"(ad), "l"(bd), "r"(idesc), "r"(k) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(&bar)), "r"(ph) : "memory");
      ph ^= 1;
      tsum += clock64() - t0;
    }
    out[blockIdx.x] = tsum / iters;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148); unsigned long long h[148];
  cudaFuncSetAttribute(mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int n : {16, 64, 128, 256}) {
    mma_kernel<true><<<148, 128, 96 * 1024>>>(n, 200, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("TS N=%3d: 8 MMAs (K=128) + commit + wait: %llu cycles (%s)\n", n, h[0], cudaGetErrorString(cudaGetLastError()));
    mma_kernel<false><<<148, 128, 96 * 1024>>>(n, 200, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("SS N=%3d: 8 MMAs (K=128) + commit + wait: %llu cycles (%s)\n", n, h[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
