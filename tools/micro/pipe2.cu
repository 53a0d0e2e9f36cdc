// Microbenchmark: the decode GEMM's barrier skeleton (no payload) -- producer,
// dequant groups, MMA issuers, epilogue -- as a function of the synchronisation
// design.  Prints cycles per pipeline step (148 CTAs, 1 per SM).
//   NG  dequant groups, GW warps per group (GW in {4, 8})
//   NI  MMA issuers (commit-released A / X stages)
//   ARR 0: every dequant warp arrives on a_full (count GW); 1: named barrier of
//       the group, then one arrival (count 1)
//   REL 0: code stage released by the dequant warps; 1: by the issuer's commit
//   HINT 1: waits with a suspend-time hint
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
template <int HINT>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  if (HINT)
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph), "r"(HINT) : "memory");
  else
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(b)) : "memory");
}
constexpr int CS = 16, XS = 8, AS = 4;
template <int NG, int GW, int NI, int ARR, int REL, int HINT>
__global__ void __launch_bounds__(1024, 1) pipe(int nst, unsigned long long* out) {
  __shared__ uint64_t c_full[CS], c_empty[CS], a_full[AS], a_empty[AS], x_full[XS], x_empty[XS], d_full[2], d_empty[2];
  __shared__ uint32_t tbase;
  constexpr int DQW = NG * GW;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int EPI = DQW, PROD = DQW + 4, MMA0 = DQW + 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CS; ++s) { init(&c_full[s], 1); init(&c_empty[s], REL ? 1 : (ARR ? 1 : GW)); }
    for (int s = 0; s < AS; ++s) { init(&a_full[s], ARR ? 1 : GW); init(&a_empty[s], 1); }
    for (int s = 0; s < XS; ++s) { init(&x_full[s], 1); init(&x_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { init(&d_full[s], NI); init(&d_empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (wid == PROD) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory"); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const int seg = 34;
  long long t0 = clock64();
  if (wid == PROD) {
    int cs = 0, xs = 0; uint32_t cp = 0, xp = 0;
    for (int j = 0; j < nst; ++j) {
      wait<HINT>(&c_empty[cs], cp ^ 1); if (lane == 0) arrive(&c_full[cs]);
      wait<HINT>(&x_empty[xs], xp ^ 1); if (lane == 0) arrive(&x_full[xs]);
      __syncwarp();
      if (++cs == CS) { cs = 0; cp ^= 1; }
      if (++xs == XS) { xs = 0; xp ^= 1; }
    }
  } else if (wid >= MMA0 && wid < MMA0 + NI) {
    const int ii = wid - MMA0;
    int as = ii, xs = ii, cs = ii; uint32_t ap = 0, xp = 0, cp = 0;
    int m = 0;
    for (int j0 = 0; j0 < nst; j0 += seg, ++m) {
      wait<HINT>(&d_empty[m & 1], ((m >> 1) & 1) ^ 1);
      int j = j0 + ((ii - j0) % NI + NI) % NI;
      for (; j < j0 + seg && j < nst; j += NI) {
        wait<HINT>(&a_full[as], ap); wait<HINT>(&x_full[xs], xp);
        asm volatile("tcgen05.fence::after_thread_sync;");
        commit(&a_empty[as]); commit(&x_empty[xs]);
        if (REL) commit(&c_empty[cs]);
        as += NI; if (as >= AS) { as -= AS; ap ^= 1; }
        xs += NI; if (xs >= XS) { xs -= XS; xp ^= 1; }
        cs += NI; if (cs >= CS) { cs -= CS; cp ^= 1; }
      }
      commit(&d_full[m & 1]);
    }
  } else if (wid < DQW) {
    const int grp = wid / GW;
    int cs = grp, as = grp; uint32_t cp = 0, ap = 0;
    for (int j = grp; j < nst; j += NG) {
      if (ARR && (wid % GW) != 0) {
      } else {
        wait<HINT>(&c_full[cs], cp);
      }
      if (ARR) asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(GW * 32) : "memory");
      if (!REL) {
        __syncwarp();
        if (ARR) { if (wid % GW == 0 && lane == 0) arrive(&c_empty[cs]); }
        else if (lane == 0) arrive(&c_empty[cs]);
      }
      if (!(ARR && (wid % GW) != 0)) wait<HINT>(&a_empty[as], ap ^ 1);
      if (ARR) asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(GW * 32) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = lane + k;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
        :: "r"(tbase + (((wid & 3) * 32) << 16) + as * 64), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (ARR) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(GW * 32) : "memory");
        if (wid % GW == 0 && lane == 0) arrive(&a_full[as]);
      } else {
        __syncwarp(); if (lane == 0) arrive(&a_full[as]);
      }
      cs += NG; if (cs >= CS) { cs -= CS; cp ^= 1; }
      as += NG; if (as >= AS) { as -= AS; ap ^= 1; }
    }
  } else if (wid >= EPI && wid < EPI + 4) {
    int m = 0;
    for (int j0 = 0; j0 < nst; j0 += seg, ++m) {
      wait<HINT>(&d_full[m & 1], (m >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t v0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v0) : "r"(tbase + (((wid & 3) * 32) << 16) + 300));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (v0 == 0x12345678u) out[200] = v0;
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp(); if (lane == 0) arrive(&d_empty[m & 1]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (wid == PROD) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 256 * 8);
  unsigned long long h[148];
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int nst = 34 * 60;
  auto run = [&](auto k, int threads, const char* name) {
    k<<<148, threads>>>(nst, d); cudaDeviceSynchronize();
    k<<<148, threads>>>(nst, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-44s %s cycles/step %.1f\n", name, cudaGetErrorString(e), mx / nst);
  };
#define RUN(NG, GW, NI, ARR, REL, HINT) run(pipe<NG, GW, NI, ARR, REL, HINT>, (NG * GW + 5 + NI) * 32, "NG=" #NG " GW=" #GW " NI=" #NI " ARR=" #ARR " REL=" #REL " HINT=" #HINT)
  RUN(2, 8, 2, 0, 0, 0);   // the decode kernel as written
  RUN(2, 8, 2, 1, 0, 0);
  RUN(2, 8, 2, 0, 1, 0);
  RUN(2, 8, 2, 1, 1, 0);
  RUN(2, 4, 2, 0, 0, 0);
  RUN(2, 4, 2, 0, 1, 0);
  RUN(4, 4, 2, 0, 1, 0);
  RUN(1, 4, 1, 0, 1, 0);
  RUN(1, 8, 1, 0, 1, 0);
  RUN(2, 4, 1, 0, 1, 0);
  RUN(2, 8, 2, 0, 0, 1000);
  RUN(2, 8, 2, 0, 0, 100000);
  RUN(2, 4, 2, 0, 1, 100000);
  return 0;
}
