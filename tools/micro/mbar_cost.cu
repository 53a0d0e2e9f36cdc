// Microbenchmark: latency of mbarrier primitives as seen by one thread, with
// the rest of the CTA idle / polling other barriers / streaming bulk copies.
//   A: try_wait on a completed phase            B: test_wait on a completed phase
//   C: arrive                                   D: arrive + try_wait round trip through a second warp (ping-pong)
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
__device__ __forceinline__ void mtest(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
// bg: 0 idle, 1 16 warps polling a never-completing barrier, 2 one warp streaming bulk copies
template <int BG>
__global__ void __launch_bounds__(640, 1) k(const uint8_t* src, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done, never, ping, pong, sfull[8], sempty[8];
  __shared__ volatile int stop;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    minit(&done, 1); minit(&never, 1); minit(&ping, 1); minit(&pong, 1);
    for (int s = 0; s < 8; ++s) { minit(&sfull[s], 1); minit(&sempty[s], 1); }
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (wid == 0) {
    if (lane == 0) marrive(&done);   // phase 0 completes
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < 1000; ++i) mwait(&done, 0);
    long long t1 = clock64();
    for (int i = 0; i < 1000; ++i) mtest(&done, 0);
    long long t2 = clock64();
    for (int i = 0; i < 1000; ++i) { if (lane == 0) marrive(&never); __syncwarp(); }
    long long t3 = clock64();
    // ping-pong with warp 1
    for (int i = 0; i < 500; ++i) {
      if (lane == 0) marrive(&ping);
      mwait(&pong, i & 1);
    }
    long long t4 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; }
    stop = 1;
  } else if (wid == 1) {
    for (int i = 0; i < 500; ++i) {
      mwait(&ping, i & 1);
      if (lane == 0) marrive(&pong);
    }
  } else if (BG == 1 && wid >= 2 && wid < 18) {
    while (!stop) {
      uint32_t ok;
      asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(su32(&never)), "r"(1u) : "memory");
    }
  } else if (BG == 2 && wid == 2) {
    int s = 0; uint32_t ph = 0;
    const uint8_t* base = src + blockIdx.x * (size_t)(64 << 20) / 148;
    for (int c = 0; !stop && c < 100000; ++c) {
      mwait(&sempty[s], ph ^ 1);
      if (lane == 0) { mexpect(&sfull[s], 16384); bulk(su32(sm + s * 16384), base + (size_t)(c % 256) * 16384, 16384, &sfull[s]); }
      __syncwarp();
      if (++s == 8) { s = 0; ph ^= 1; }
    }
  } else if (BG == 2 && wid == 3) {
    int s = 0; uint32_t ph = 0;
    for (int c = 0; !stop && c < 100000; ++c) {
      mwait(&sfull[s], ph);
      if (lane == 0) marrive(&sempty[s]);
      __syncwarp();
      if (++s == 8) { s = 0; ph ^= 1; }
    }
  }
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  uint8_t* buf; cudaMalloc(&buf, 64 << 20);
  unsigned long long* d; cudaMalloc(&d, 64); unsigned long long h[4];
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    kern<<<148, 640, 8 * 16384>>>(buf, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("%-28s try_wait(done) %6.1f  test_wait(done) %6.1f  arrive %6.1f  ping-pong round trip %6.1f cycles (%s)\n", name,
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 500.0, cudaGetErrorString(e));
  };
  run(k<0>, "idle CTA");
  run(k<1>, "16 warps polling");
  run(k<2>, "bulk stream in background");
  return 0;
}
