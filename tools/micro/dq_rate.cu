// Microbenchmark: raw dequant + TMEM-store throughput of one SM, no barriers.
// G groups of 4 warps; each warp loops: load 12 code words + 4 scales from smem,
// dequantize 4 x 32 3-bit codes (the engine's dequant32<3>), tcgen05.st x16 x4,
// tcgen05.wait::st.  Reports cycles per 128x128 chunk for the SM (all groups).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2605_09281_b200/csrc/tq_ptx.cuh"
using namespace tqb;
template <int G, bool ST, bool DQ>
__global__ void __launch_bounds__(G * 128, 1) dq(int iters, unsigned long long* out, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, q = wid & 3, grp = wid >> 2;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x12345678u * i;
  if (wid == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase + ((uint32_t)(q * 32) << 16) + grp * 64;
  const uint32_t* wst = reinterpret_cast<const uint32_t*>(sm) + q * 32 + lane;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int so = (it & 7) * 1536;
    uint32_t words[4][3]; uint16_t sb[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int w = 0; w < 3; ++w) words[s][w] = wst[so + (s >> 1) * 768 + (s & 1) * 384 + w * 128];
      sb[s] = reinterpret_cast<const uint16_t*>(sm + 60000)[(s & 1) * 128 + q * 32 + lane] | 0x3c00;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      uint32_t v[16];
      if (DQ) { const DqConst c = make_dq(__ushort_as_half(sb[s])); dequant32<3>(words[s], c, v); }
      else {
#pragma unroll
        for (int w = 0; w < 16; ++w) v[w] = words[s][w % 3] + w;
      }
      if (ST) tc_st_32x32b_x16(tm + s * 16, v);
      else {
#pragma unroll
        for (int w = 0; w < 16; ++w) acc ^= v[w];
      }
    }
    if (ST) tc_wait_st();
  }
  long long dt = clock64() - t0;
  if (acc == 0x1234567u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = dt;
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 148 * 8); uint32_t* sink; cudaMalloc(&sink, 64);
  unsigned long long h[148];
  const int iters = 2000;
  auto run = [&](auto k, int G, const char* name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k<<<148, G * 128, 100 * 1024>>>(iters, d, sink); cudaDeviceSynchronize();
    k<<<148, G * 128, 100 * 1024>>>(iters, d, sink); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-28s G=%d %s: %.1f cycles/iter/group, %.1f cycles per chunk per SM\n", name, G, cudaGetErrorString(e),
           (double)h[0] / iters, (double)h[0] / iters / G);
  };
  run(dq<1, true, true>, 1, "dequant+st");
  run(dq<2, true, true>, 2, "dequant+st");
  run(dq<3, true, true>, 3, "dequant+st");
  run(dq<4, true, true>, 4, "dequant+st");
  run(dq<4, false, true>, 4, "dequant only");
  run(dq<4, true, false>, 4, "st only");
  run(dq<1, false, true>, 1, "dequant only");
  return 0;
}
