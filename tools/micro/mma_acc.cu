// Microbenchmark: does one issuing thread pipeline tcgen05.mma (kind::f16, TS,
// M=128, K=16) across independent accumulators?  8 MMAs per chunk, K-steps dealt
// round-robin over ND accumulators; 4 chunks in flight.  Also: the same with the
// 8 MMAs of a chunk split over 2 chunks' accumulators.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
template <int ND>
__global__ void __launch_bounds__(128, 1) k(int n, int chunks, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t base = su32(sm);
    uint32_t ph[4] = {0, 0, 0, 0};
    long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      const int s = c & 3;
      if (c >= 4) {
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(&bar[s])), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
      }
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = desc(base + 32768 + (kk / 4) * 16384 + (kk % 4) * 32);
        const uint32_t d = tm + 256 + (kk % ND) * 64;
        asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(tm + s * 64 + kk * 8), "l"(bd), "r"(idesc), "r"(kk | c) : "memory");
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&bar[s])) : "memory");
    }
    for (int s = 0; s < 4; ++s)
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(&bar[s])), "r"(ph[s]) : "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 8 * 148); unsigned long long h[148];
  const int chunks = 400;
  auto run = [&](auto kern, const char* name, int n) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    kern<<<148, 128, 96 * 1024>>>(n, chunks, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("%s N=%d: %.1f cycles per 8-MMA chunk (%s)\n", name, n, (double)h[0] / chunks, cudaGetErrorString(e));
  };
  for (int n : {16, 32, 64}) {
    run(k<1>, "1 accumulator ", n);
    run(k<2>, "2 accumulators", n);
    run(k<4>, "4 accumulators", n);
  }
  return 0;
}
