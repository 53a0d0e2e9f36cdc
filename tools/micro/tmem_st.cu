// Microbenchmark: tcgen05.st (32x32b) issue->wait::st latency and throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NX>
__global__ void __launch_bounds__(512, 1) st_kernel(int iters, int nwarps_active, unsigned long long* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  uint32_t v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 16 + i;
  long long t0 = clock64();
  if (warp < nwarps_active) {
    const int q = warp & 3;
    const uint32_t addr = tm + ((uint32_t)(q * 32) << 16) + (warp >> 2) * 16 * NX;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int x = 0; x < NX; ++x)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(addr + x * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                       "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[0] += 1;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  const int iters = 2000;
  for (int nw : {1, 4, 8, 16}) {
    st_kernel<1><<<148, 512>>>(iters, nw, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("x16 x1  warps=%2d : %.1f cycles per (st+wait) iteration (%s)\n", nw, (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
    st_kernel<4><<<148, 512>>>(iters, nw, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("x16 x4  warps=%2d : %.1f cycles per (4 st+wait) iteration\n", nw, (double)h[0] / iters);
  }
  return 0;
}
