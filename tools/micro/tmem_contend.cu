// Microbenchmark: does tcgen05.st traffic (dequant warps writing A tiles) slow
// down tcgen05.mma with A from TMEM (TS)?  NI issuer warps issue 8-MMA chunks
// (M=128, N=16, K=128) with a commit ring; G groups of 4 warps store 4 x16
// columns per lane per chunk (a 128x128 fp16 tile = 32 KB) + wait::st.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
template <int NI, int G, bool TS>
__global__ void __launch_bounds__(128 + 128 * 4, 1) k(int chunks, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2][4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i / 4][i % 4]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  long long t0 = clock64();
  if (warp < NI) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | (8u << 24);
    const uint32_t base = su32(sm);
    uint32_t ph[4] = {0, 0, 0, 0};
    for (int c = 0; c < chunks; ++c) {
      const int s = c & 3;
      if (c >= 4) {
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(&bar[warp][s])), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
      }
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = desc(base + 32768 + (kk / 4) * 16384 + (kk % 4) * 32);
        if (TS)
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 448 + warp * 32), "r"(tm + warp * 64 + kk * 8), "l"(bd), "r"(idesc), "r"(kk | c) : "memory");
        else {
          const uint64_t ad = desc(base + (kk / 4) * 8192 + (kk % 4) * 32);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm + 448 + warp * 32), "l"(ad), "l"(bd), "r"(idesc), "r"(kk | c) : "memory");
        }
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&bar[warp][s])) : "memory");
    }
    for (int s = 0; s < 4; ++s)
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(&bar[warp][s])), "r"(ph[s]) : "memory");
    if (lane == 0) out[blockIdx.x * 8 + warp] = clock64() - t0;
  } else if (warp >= 4 && warp < 4 + 4 * G) {
    const int q = warp & 3, grp = (warp - 4) >> 2;
    const uint32_t ta = tm + ((uint32_t)(q * 32) << 16) + 128 + grp * 64;
    uint32_t v[16];
#pragma unroll
    for (int w = 0; w < 16; ++w) v[w] = lane * 16 + w;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
          :: "r"(ta + (s & 3) * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[0] += c;
    }
    if (lane == 0 && q == 0) out[blockIdx.x * 8 + 4 + grp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 8 * 148 * 8); unsigned long long h[148 * 8];
  const int chunks = 400;
  auto run = [&](auto kern, int threads, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaMemset(d, 0, 8 * 148 * 8);
    kern<<<148, threads, 96 * 1024>>>(chunks, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s %s  mma0 %.0f mma1 %.0f  st-groups %.0f %.0f %.0f %.0f cycles/chunk\n", name, cudaGetErrorString(e),
           (double)h[0] / chunks, (double)h[1] / chunks, (double)h[4] / chunks, (double)h[5] / chunks, (double)h[6] / chunks, (double)h[7] / chunks);
  };
  run(k<2, 0, true>, 128, "TS: 2 issuers, no st");
  run(k<2, 4, true>, 128 + 512, "TS: 2 issuers + 4 st groups");
  run(k<0, 4, true>, 128 + 512, "4 st groups only");
  run(k<2, 0, false>, 128, "SS: 2 issuers, no st");
  run(k<2, 4, false>, 128 + 512, "SS: 2 issuers + 4 st groups");
  run(k<1, 4, true>, 128 + 512, "TS: 1 issuer + 4 st groups");
  return 0;
}
