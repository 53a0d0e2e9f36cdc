// Microbenchmark: the v3 decode GEMM skeleton (no payload) -- 2 code + 2 activation
// producers, 2 dequant groups x 8 warps (tcgen05.st x16 per super-word), NI MMA
// issuers that each commit to the A-stage and X-stage barriers every step, 3 A
// stages, epilogue per 17-step part.  Knobs isolate what costs cycles per step.
//   NI      issuers (each commits every step)
//   ST      tcgen05.st per dequant warp per step (4 in the kernel, 0 = none)
//   XC      1: issuers also commit x_empty every step (2 commits / issuer / step)
//   MMA     K=16 MMAs per issuer per step (issued from TMEM A stage, B = smem zeros)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
constexpr int CS = 8, XS = 6, AS = 3;
template <int NI, int ST, int XC, int MMA>
__global__ void __launch_bounds__(896, 1) pipe(int nst, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  __shared__ uint64_t c_full[CS], c_empty[CS], x_full[XS], x_empty[XS], a_full[AS], a_empty[AS], d_full[4];
  __shared__ uint32_t tbase;
  __shared__ volatile uint32_t epi_seq[4];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CS; ++s) { init(&c_full[s], 1); init(&c_empty[s], 8); }
    for (int s = 0; s < XS; ++s) { init(&x_full[s], 1); init(&x_empty[s], XC ? NI : 1); }
    for (int s = 0; s < AS; ++s) { init(&a_full[s], 8); init(&a_empty[s], NI); }
    for (int s = 0; s < 4; ++s) { init(&d_full[s], 1); epi_seq[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(dsm)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  if (wid == 4) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const int seg = 17;
  const uint32_t tm = tbase;
  long long t0 = clock64();
  if (wid == 4 || wid == 5) {            // code producers
    const int pp = wid - 4; int cs = pp; uint32_t ph = 0;
    for (int j = pp; j < nst; j += 2) {
      wait(&c_empty[cs], ph ^ 1); if (lane == 0) arrive(&c_full[cs]); __syncwarp();
      cs += 2; if (cs >= CS) { cs -= CS; ph ^= 1; }
    }
  } else if (wid == 6 || wid == 7) {     // activation producers
    const int pp = wid - 6; int xs = pp; uint32_t ph = 0;
    for (int j = pp; j < nst; j += 2) {
      wait(&x_empty[xs], ph ^ 1); if (lane == 0) arrive(&x_full[xs]); __syncwarp();
      xs += 2; if (xs >= XS) { xs -= XS; ph ^= 1; }
    }
  } else if (wid < NI) {                 // issuers
    const int ii = wid;
    int as = 0, xs = 0; uint32_t ap = 0, xp = 0;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(32 >> 3) << 17) | (8u << 24);
    for (int j0 = 0, m = 0; j0 < nst; j0 += seg, ++m) {
      while (epi_seq[ii] < (uint32_t)m) __nanosleep(64);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int j = j0; j < j0 + seg && j < nst; ++j) {
        wait(&a_full[as], ap); wait(&x_full[xs], xp);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int kk = 0; kk < MMA; ++kk)
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 384 + ii * 32), "r"(tm + as * 128 + kk * 8), "l"(desc(su32(dsm) + (kk % 4) * 32)), "r"(idesc), "r"(kk) : "memory");
        commit(&a_empty[as]);
        if (XC || ii == 0) commit(&x_empty[xs]);
        if (++as == AS) { as = 0; ap ^= 1; }
        if (++xs == XS) { xs = 0; xp ^= 1; }
      }
      commit(&d_full[ii]);
    }
  } else if (wid >= 8 && wid < 12) {     // epilogue
    for (int j0 = 0, m = 0; j0 < nst; j0 += seg, ++m) {
      for (int ii = 0; ii < NI; ++ii) wait(&d_full[ii], m & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("bar.sync 1, 128;");
      if (wid == 8 && lane < NI) epi_seq[lane] = m + 1;
    }
  } else if (wid >= 12) {                // dequant groups
    const int dw = wid - 12, grp = dw >> 3;
    int cs = grp, as = grp; uint32_t cp = 0, ap = 0;
    for (int j = grp; j < nst; j += 2) {
      wait(&c_full[cs], cp);
      wait(&a_empty[as], ap ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int t = 0; t < ST; ++t) {
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = lane + k + t;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
          :: "r"(tm + (((wid & 3) * 32) << 16) + as * 128 + ((dw >> 2) & 1) * 64 + t * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      }
      if (ST) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      __syncwarp(); if (lane == 0) arrive(&c_empty[cs]);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp(); if (lane == 0) arrive(&a_full[as]);
      cs += 2; if (cs >= CS) { cs -= CS; cp ^= 1; }
      as += 2; if (as >= AS) { as -= AS; ap ^= 1; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (wid == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 256 * 8);
  unsigned long long h[148];
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int nst = 17 * 40;
  auto run = [&](auto k, const char* name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<148, 896, 64 * 1024>>>(nst, d); cudaDeviceSynchronize();
    k<<<148, 896, 64 * 1024>>>(nst, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-36s %s cycles/step %.1f\n", name, cudaGetErrorString(e), mx / nst);
  };
#define R(NI, ST, XC, MMA) run(pipe<NI, ST, XC, MMA>, "NI=" #NI " ST=" #ST " XC=" #XC " MMA=" #MMA)
  R(4, 4, 1, 0);   // the kernel's skeleton (abl=15)
  R(4, 4, 1, 4);   // + MMAs
  R(4, 0, 1, 0);
  R(4, 4, 0, 0);
  R(2, 4, 1, 0);
  R(1, 4, 1, 0);
  R(4, 0, 0, 0);
  R(2, 0, 0, 0);
  R(1, 0, 0, 0);
  R(4, 4, 0, 4);
  R(2, 4, 0, 8);
  return 0;
}
