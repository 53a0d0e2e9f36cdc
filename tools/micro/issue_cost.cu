// Microbenchmark: single-thread issue cost of the code producer's per-chunk
// operations (mbarrier try_wait on a completed phase, arrive.expect_tx,
// cp.async.bulk of 6.6 KB + 256 B), one CTA, L2-resident source.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

// mode bit 0: wait on the (completed) previous phase of the stage before reuse
// mode bit 1: second 256-byte bulk copy per chunk
// mode bit 2: no copies at all (barrier ops only: arrive without tx)
__global__ void __launch_bounds__(128, 1) issue_kernel(const uint8_t* src, int nchunks, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int kSt = 6912, kN = 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kN * kSt);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kN; ++s) minit(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0;
    long long t0 = clock64(), tw = 0;
    for (int c = 0; c < nchunks; ++c) {
      if ((mode & 1) && c >= kN) {
        long long a = clock64();
        mwait(&full[s], ph ^ 1);   // the fill issued kN chunks ago
        tw += clock64() - a;
      }
      const uint8_t* g = src + (size_t)(c % 64) * kSt;
      if (mode & 4) {
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
      } else if (mode & 2) {
        mexpect(&full[s], kSt);
        bulk(sm + s * kSt, g, kSt - 256, &full[s]);
        bulk(sm + s * kSt + kSt - 256, g + kSt - 256, 256, &full[s]);
      } else {
        mexpect(&full[s], kSt);
        bulk(sm + s * kSt, g, kSt, &full[s]);
      }
      if (++s == kN) { s = 0; ph ^= 1; }
    }
    long long t1 = clock64();
    // drain
    for (int q = 0; q < kN; ++q) { mwait(&full[s], ph ^ 1); if (++s == kN) { s = 0; ph ^= 1; } }
    out[0] = t1 - t0;
    out[1] = tw;
    out[2] = clock64() - t0;
  }
}

int main() {
  uint8_t* buf; cudaMalloc(&buf, 64 * 6912); cudaMemset(buf, 1, 64 * 6912);
  long long* out; cudaMalloc(&out, 64);
  const int smem = 8 * 6912 + 1024;
  cudaFuncSetAttribute(issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"1 bulk, no wait", "1 bulk + wait", "2 bulks, no wait", "2 bulks + wait", "arrive only", "arrive + wait"};
  const int modes[] = {0, 1, 2, 3, 4, 5};
  for (int i = 0; i < 6; ++i) {
    long long h[3];
    for (int rep = 0; rep < 3; ++rep) {
      issue_kernel<<<1, 128, smem>>>(buf, 400, modes[i], out);
      cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    }
    printf("%-18s issue %6.1f cyc/chunk (of which wait %6.1f); incl. drain %6.1f cyc/chunk  %s\n", names[i], h[0] / 400.0,
           h[1] / 400.0, h[2] / 400.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
