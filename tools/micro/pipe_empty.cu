// Microbenchmark: the gemm kernel's barrier pipeline with no payload.
// Roles as in tq_gemm.cu (3 dequant groups x 4 warps, epilogue 4, alloc, code
// producer, X producer, MMA issuer).  MODE selects how the MMA warp releases
// stages:  0 tcgen05.commit (elect) x2 per chunk   1 mbarrier.arrive x2
//          2 one tcgen05.commit per chunk to a shared "consumed" barrier
// Prints cycles per chunk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* b) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(b)) : "memory");
}
constexpr int CS = 13, AS = 6, XS = 6, NG = 3;
template <int MODE, bool LDS, bool UNITS, int FENCE = 1>
__global__ void __launch_bounds__(640, 1) pipe(int nch, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  __shared__ uint64_t c_full[CS], c_empty[CS], a_full[AS], a_empty[AS], x_full[XS], x_empty[XS], done, d_full[2], d_empty[2];
  __shared__ uint32_t tbase;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CS; ++s) { init(&c_full[s], 1); init(&c_empty[s], 4); }
    for (int s = 0; s < AS; ++s) { init(&a_full[s], 4); init(&a_empty[s], 1); }
    for (int s = 0; s < XS; ++s) { init(&x_full[s], 1); init(&x_empty[s], 1); }
    init(&done, 1); for (int s = 0; s < 2; ++s) { init(&d_full[s], 1); init(&d_empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (wid == 16) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (wid == 17) {            // code producer
    int s = 0; uint32_t ph = 0;
    for (int c = 0; c < nch; ++c) { wait(&c_empty[s], ph ^ 1); if (lane == 0) arrive(&c_full[s]); if (++s == CS) { s = 0; ph ^= 1; } }
  } else if (wid == 18) {     // X producer
    int s = 0; uint32_t ph = 0;
    for (int c = 0; c < nch; ++c) { wait(&x_empty[s], ph ^ 1); if (lane == 0) arrive(&x_full[s]); if (++s == XS) { s = 0; ph ^= 1; } }
  } else if (wid == 19) {     // MMA issuer
    int as = 0, xs = 0, lu = 0; uint32_t ap = 0, xp = 0;
    for (int c = 0; c < nch; ++c) {
      if (UNITS && c % 33 == 0) { wait(&d_empty[lu & 1], ((lu >> 1) & 1) ^ 1); }
      wait(&a_full[as], ap); wait(&x_full[xs], xp);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (MODE == 0) { commit_elect(&a_empty[as]); commit_elect(&x_empty[xs]); }
      else { if (lane == 0) { arrive(&a_empty[as]); arrive(&x_empty[xs]); } }
      if (++as == AS) { as = 0; ap ^= 1; }
      if (++xs == XS) { xs = 0; xp ^= 1; }
      if (UNITS && c % 33 == 32) { commit_elect(&d_full[lu & 1]); ++lu; }
    }
    if (MODE == 0) commit_elect(&done); else if (lane == 0) arrive(&done);
  } else if (wid < 4 * NG) {  // dequant groups
    const int grp = wid >> 2;
    int cs = 0, as = 0, rr = 0; uint32_t cp = 0, ap = 0;
    for (int c = 0; c < nch; ++c) {
      const bool mine = rr == grp; if (++rr == NG) rr = 0;
      if (mine) {
        wait(&c_full[cs], cp);
        uint32_t acc = 0;
        if (LDS) {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(dsm + cs * 7168) + (wid & 3) * 32 + lane;
#pragma unroll
          for (int k = 0; k < 16; ++k) acc += w[k * 128];
        }
        __syncwarp(); if (lane == 0) arrive(&c_empty[cs]);
        if (acc == 0x12345678u) out[1] = acc;
        wait(&a_empty[as], ap ^ 1);
        if (FENCE & 2) asm volatile("tcgen05.fence::after_thread_sync;");
        if (FENCE & 4) {
          uint32_t v[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = lane + k;
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
            :: "r"(tbase + (((wid & 3) * 32) << 16) + as * 64), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        if (FENCE & 1) asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp(); if (lane == 0) arrive(&a_full[as]);
      }
      if (++cs == CS) { cs = 0; cp ^= 1; }
      if (++as == AS) { as = 0; ap ^= 1; }
    }
  } else if (wid < 16) {      // epilogue
    if (UNITS) {
      const int nu = (nch + 32) / 33;
      for (int lu = 0; lu < nu; ++lu) {
        wait(&d_full[lu & 1], (lu >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t v0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v0) : "r"(tbase + (((wid & 3) * 32) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (v0 == 0x12345678u) out[2] = v0;
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp(); if (lane == 0) arrive(&d_empty[lu & 1]);
      }
    }
    wait(&done, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (wid == 16) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int nch = 33 * 90;
  auto run = [&](auto k, const char* name, int smem = 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 640, smem>>>(nch, d); cudaDeviceSynchronize();
    k<<<148, 640, smem>>>(nch, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-32s %s cycles/chunk %.1f\n", name, cudaGetErrorString(e), (double)h[0] / nch);
  };
  run(pipe<0, false, false>, "commit x2 per chunk");
  run(pipe<1, false, false>, "mbarrier.arrive x2 per chunk");
  run(pipe<0, false, false>, "commit x2, 220KB smem", 220 * 1024);
  run(pipe<0, true, false>, "commit x2, LDS, 220KB smem", 220 * 1024);
  run(pipe<0, true, true>, "commit x2, LDS, units, 220KB", 220 * 1024);
  run(pipe<0, false, true>, "commit x2, units", 0);
  run(pipe<0, true, true, 0>, "LDS units, no fences", 220 * 1024);
  run(pipe<0, true, true, 3>, "LDS units, both fences", 220 * 1024);
  run(pipe<0, true, true, 7>, "LDS units, fences + st x16", 220 * 1024);
  run(pipe<1, true, true, 0>, "arrive, LDS units, no fences", 220 * 1024);
  return 0;
}
