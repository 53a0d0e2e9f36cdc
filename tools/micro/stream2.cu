// Microbenchmark: HBM streaming through a bulk-copy ring as the decode GEMM's
// producer would drive it -- 148 CTAs, one producer warp (elected lane), one
// consumer warp releasing stages.  Per stage: `nc` code copies of HBM data
// (stage / nc bytes each) + `nx` small copies of an L2-resident buffer (xb
// bytes each).  Reports HBM GB/s (code bytes only) and cycles per stage.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
template <int NP>
__global__ void __launch_bounds__(64 * NP, 1) stream(const uint8_t* src, const uint8_t* xsrc, size_t per_cta, int stage, int nc,
                                                int nx, int xb, int nst, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  const int sstride = stage + nx * xb;
  __shared__ uint64_t full_all[NP][32], empty_all[NP][32];
  const int pr = threadIdx.x / 64;
  uint64_t* full = full_all[pr];
  uint64_t* empty = empty_all[pr];
  if (threadIdx.x == 0) {
    for (int q = 0; q < NP; ++q)
      for (int s = 0; s < nst; ++s) { minit(&full_all[q][s], 1); minit(&empty_all[q][s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * per_cta + pr * (per_cta / NP);
  const int n = (int)(per_cta / NP / stage);
  const int warp = (threadIdx.x >> 5) & 1, lane = threadIdx.x & 31;
  uint8_t* sm = sm_raw + pr * nst * sstride;
  long long t0 = clock64();
  if (warp == 0) {
    int s = 0; uint32_t ph = 0;
    for (int c = 0; c < n; ++c) {
      mwait(&empty[s], ph ^ 1);
      if (lane == 0) {
        const uint32_t d = su32(sm + s * sstride);
        mexpect(&full[s], stage + nx * xb);
        const int piece = stage / nc;
        for (int q = 0; q < nc; ++q) bulk(d + q * piece, base + (size_t)c * stage + q * piece, piece, &full[s]);
        for (int q = 0; q < nx; ++q) bulk(d + stage + q * xb, xsrc + (size_t)((blockIdx.x * 7 + c * 3 + q) % 64) * xb, xb, &full[s]);
      }
      __syncwarp();
      if (++s == nst) { s = 0; ph ^= 1; }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (int c = 0; c < n; ++c) {
      mwait(&full[s], ph);
      __syncwarp();
      if (lane == 0) marrive(&empty[s]);
      if (++s == nst) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const size_t per_cta = 6 << 20;   // 6 MB per CTA (888 MB total)
  uint8_t* buf; cudaMalloc(&buf, per_cta * 148 + (1 << 20)); cudaMemset(buf, 1, per_cta * 148);
  uint8_t* xbuf; cudaMalloc(&xbuf, 64 * 16384); cudaMemset(xbuf, 2, 64 * 16384);
  unsigned long long* d; cudaMalloc(&d, 148 * 8); unsigned long long h[148];
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](int stage, int nc, int nx, int xb, int nst, int np = 1) {
    const int smem = np * nst * (stage + nx * xb);
    if (smem > 220 * 1024) return;
    auto k = np == 1 ? stream<1> : np == 2 ? stream<2> : stream<4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 64 * np, smem>>>(buf, xbuf, per_cta, stage, nc, nx, xb, nst, d);
    cudaEventRecord(a);
    k<<<148, 64 * np, smem>>>(buf, xbuf, per_cta, stage, nc, nx, xb, nst, d);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("np %d stage %6d nc %d nx %d xb %5d nst %2d: %7.1f GB/s  %6.1f cycles/stage/producer  (%s)\n", np, stage, nc, nx, xb, nst,
           per_cta * 148 / (ms * 1e-3) / 1e9, (double)h[0] / (per_cta / np / stage), cudaGetErrorString(e));
  };
  run(6144, 1, 0, 0, 16, 1);
  run(6144, 1, 0, 0, 8, 2);
  run(6144, 1, 0, 0, 4, 4);
  run(3072, 1, 0, 0, 16, 2);
  run(12288, 1, 0, 0, 8, 2);
  run(6144, 2, 0, 0, 8, 2);
  run(8192, 1, 0, 0, 12, 1);
  run(16384, 1, 0, 0, 8, 1);
  run(8192, 1, 0, 0, 6, 2);
  return 0;
}
