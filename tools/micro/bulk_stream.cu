// Microbenchmark: HBM streaming bandwidth of cp.async.bulk into a smem ring
// (one producer thread, consumer warps that only release stages) as a
// function of stage size and ring depth, 148 persistent CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_09281_b200/csrc/tq_ptx.cuh"

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

__global__ void __launch_bounds__(256, 1) stream_kernel(const uint8_t* src, size_t per_cta, int stage, int nst, unsigned long long* sink, int split, int run_len = 6, int jump = 32, size_t cta_stride = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * stage);
  uint64_t* empty = full + 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { minit(&full[s], 1); minit(&empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * (cta_stride ? cta_stride : per_cta);
  const int nchunks = (int)(per_cta / stage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && split >= 2) {
    // the engine's producer: converged warp, elect.sync, codes + scale slice in one asm
    // split 3: scale slices from a separate region (the GEMM's layout);
    // split 4: + 41 KB runs with 221 KB jumps between runs (units of m-blocks)
    int s = 0; uint32_t ph = 0;
    const uint8_t* sbase = src + ((size_t)1 << 30) + blockIdx.x * (per_cta / stage) * 256;
    for (int c = 0; c < nchunks; ++c) {
      mwait(&empty[s], ph ^ 1);
      size_t off = (size_t)c * stage;
      if (split == 4) off = ((size_t)(c / run_len) * jump + (c % run_len)) * stage;
      const uint8_t* s2 = split >= 3 ? sbase + (size_t)c * 256 : base + off + stage - 256;
      tqb::bulk_copy2_elect(&full[s], sm + s * stage, base + off, stage - 256,
                            sm + s * stage + stage - 256, s2, 256u);
      if (++s == nst) { s = 0; ph ^= 1; }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int c = 0; c < nchunks; ++c) {
        mwait(&empty[s], ph ^ 1);
        mexpect(&full[s], stage);
        if (split) {
          bulk(sm + s * stage, base + (size_t)c * stage, stage - 256, &full[s]);
          bulk(sm + s * stage + stage - 256, base + (size_t)c * stage + stage - 256, 256, &full[s]);
        } else {
          bulk(sm + s * stage, base + (size_t)c * stage, stage, &full[s]);
        }
        if (++s == nst) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    int s = 0; uint32_t ph = 0; unsigned acc = 0;
    for (int c = 0; c < nchunks; ++c) {
      mwait(&full[s], ph);
      acc += reinterpret_cast<const uint32_t*>(sm + s * stage)[lane + 32 * (warp - 4)];
      __syncwarp();
      if (lane == 0) marrive(&empty[s]);
      if (++s == nst) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678) atomicAdd(sink, 1ull);
  }
}

// plain LDG.128 streaming for comparison
__global__ void __launch_bounds__(512) ldg_kernel(const int4* src, size_t n, unsigned long long* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* buf; cudaMalloc(&buf, 2 * total); cudaMemset(buf, 1, 2 * total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = 148;
  setvbuf(stdout, nullptr, _IONBF, 0);
  int stages[] = {6912};
  int depths[] = {10, 24};
  for (int split = 0; split < 4; ++split)
  for (int st : stages) for (int nd : depths) {
    size_t smem = (size_t)st * nd + 1024;
    if (smem > 220 * 1024) continue;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    size_t per = (total / grid) / st * st;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      stream_kernel<<<grid, 256, smem>>>(buf, per, st, nd, sink, split);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("split=%d bulk stage=%6d depth=%2d inflight=%4d KB  %7.1f GB/s  (%s)\n", split, st, nd, st * nd / 1024, per * grid / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  // decode-sized streams: 50 chunks per CTA (one GEMM launch at B=1)
  struct V { int split, nd, rl, jump; };
  V vs[] = {{3, 10, 50, 50}, {4, 10, 50, 50}, {4, 10, 6, 6}, {3, 10, 50, 50}, {4, 10, 6, 32}, {4, 10, 6, 7},
            {4, 10, 6, 12}};
  for (V v : vs) {
    const int st = 6912, nd = v.nd, split = v.split;
    size_t smem = (size_t)st * nd + 1024;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    size_t per = (size_t)50 * st;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      // CTA regions 6 MB apart (room for the jumps), alternate halves of the buffer per rep
      stream_kernel<<<grid, 256, smem>>>(buf + (rep % 2) * 900 * 1024 * 1024ull, per, st, nd, sink, split, v.rl, v.jump,
                                         (size_t)6 << 20);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("short split=%d depth=%2d run=%2d jump=%2d: 50 chunks/CTA  %.2f us  %7.1f GB/s\n", split, nd, v.rl, v.jump, best * 1e3, per * grid / best / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    ldg_kernel<<<148 * 4, 512>>>((const int4*)buf, total / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
  }
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("ldg.128 streaming %7.1f GB/s\n", total / ms / 1e6);
  return 0;
}
