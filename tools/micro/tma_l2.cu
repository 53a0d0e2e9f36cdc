// Microbenchmark: L2 -> SMEM bandwidth of 2D TMA tile loads (fp16, 64 cols,
// 128B swizzle) re-reading an L2-resident activation matrix, 148 CTAs.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* d, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(d)), "l"(m), "r"(c0), "r"(c1), "r"(su32(b)) : "memory");
}

__global__ void __launch_bounds__(128, 1) l2_kernel(const __grid_constant__ CUtensorMap map, int rows, int cols, int box_rows, int nbox, int nst, int iters, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int stage = box_rows * 128 * nbox;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * stage);
  uint64_t* empty = full + 32;
  if (threadIdx.x == 0) { for (int s = 0; s < nst; ++s) { minit(&full[s], 1); minit(&empty[s], 1); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kcs = cols / 64;
  const int tiles_r = rows / (box_rows * nbox);
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      const int t = (blockIdx.x * 7 + it) % (tiles_r * kcs);
      const int r0 = (t / kcs) * box_rows * nbox, c0 = (t % kcs) * 64;
      mwait(&empty[s], ph ^ 1);
      mexpect(&full[s], stage);
      for (int b = 0; b < nbox; ++b) tma2d(sm + s * stage + b * box_rows * 128, &map, c0, r0 + b * box_rows, &full[s]);
      if (++s == nst) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    int s = 0; uint32_t ph = 0; unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
      mwait(&full[s], ph);
      acc += reinterpret_cast<const uint32_t*>(sm + s * stage)[lane];
      __syncwarp();
      if (lane == 0) marrive(&empty[s]);
      if (++s == nst) { s = 0; ph ^= 1; }
    }
    if (acc == 0x1234567) atomicAdd(sink, 1u);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fn;
  unsigned* sink; cudaMalloc(&sink, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int rowsets[] = {1536, 12288};   // 12 MB and 96 MB of fp16 x 4096 cols
  for (int rows : rowsets) {
    const int cols = 4096;
    void* buf; cudaMalloc(&buf, (size_t)rows * cols * 2); cudaMemset(buf, 1, (size_t)rows * cols * 2);
    for (int box : {16, 64}) for (int nbox : {1, 3}) for (int nst : {4, 8}) {
      CUtensorMap m; memset(&m, 0, sizeof(m));
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)cols * 2};
      cuuint32_t bx[2] = {64, (cuuint32_t)box}; cuuint32_t es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int stage = box * 128 * nbox;
      size_t smem = (size_t)stage * nst + 1024;
      cudaFuncSetAttribute(l2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 4000;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        l2_kernel<<<148, 128, smem>>>(m, rows, cols, box, nbox, nst, iters, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("matrix %5.1f MB box=%2d x%d stages=%d: %7.1f GB/s (%s)\n", rows * cols * 2 / 1e6, box, nbox, nst, (double)stage * iters * 148 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(buf);
  }
  return 0;
}
