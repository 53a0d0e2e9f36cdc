// Microbenchmark: decode GEMV on the warp-level tensor path (mma.sync m16n8k16,
// f16 x f16 -> f32) with the 3-bit dequant in registers, no TMEM / tcgen05.
// One CTA per SM, W warps; each warp repeatedly takes 16 weight rows x 128 K:
// 6 code words + 2 scales from shared memory, dequant32<3> into A fragments
// (K permuted so a lane's 32-code super-word feeds its fragment slots), then
// 8 x NT HMMAs against x fragments (8-byte LDS each).  Prints cycles per
// 128 x 256 "step" (32K weights) per SM.  Also: pure HMMA issue rate.
#include <cstdint>
#include <cstdio>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../paper_2605_09281_b200/csrc/tq_ptx.cuh"

using namespace tqb;

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NT, bool DQ>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out, float* sink) {
    __shared__ uint32_t codes[2 * 3 * 128 * 2];     // one 128 x 128 3-bit chunk: 2 atoms x 2 halves x 3 words x 128 rows
    __shared__ uint16_t scales[128];
    __shared__ __align__(16) __half xs[NT * 8 * 128];
    for (int i = threadIdx.x; i < 2 * 3 * 128 * 2; i += blockDim.x) codes[i] = 0x12345678u * (i + 1);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) scales[i] = 0x2000;
    for (int i = threadIdx.x; i < NT * 8 * 128; i += blockDim.x) xs[i] = __float2half(0.01f * (i % 7));
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int r0 = (warp & 7) * 16 + g;   // rows r0, r0 + 8 of the chunk
    float acc[NT][4] = {};
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        // lane q: super-word q = (atom q >> 1, half q & 1)
        const uint32_t* base = codes + (q >> 1) * (2 * 3 * 128) + (q & 1) * 3 * 128;
        uint32_t w0[3], w1[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            w0[j] = base[j * 128 + r0];
            w1[j] = base[j * 128 + r0 + 8];
        }
        uint32_t A0[16], A1[16];
        if (DQ) {
            const DqConst c0 = make_dq(__ushort_as_half(scales[r0]));
            const DqConst c1 = make_dq(__ushort_as_half(scales[r0 + 8]));
            dequant32<3>(w0, c0, A0);
            dequant32<3>(w1, c1, A1);
        } else {
#pragma unroll
            for (int p = 0; p < 16; ++p) {
                A0[p] = w0[p % 3] + p;
                A1[p] = w1[p % 3] + p;
            }
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint32_t a[4] = {A0[2 * s], A1[2 * s], A0[2 * s + 1], A1[2 * s + 1]};
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const uint2 b = *reinterpret_cast<const uint2*>(xs + (n * 8 + g) * 128 + q * 32 + 4 * s);
                hmma(acc[n], a, b.x, b.y);
            }
        }
    }
    const long long t1 = clock64();
    float v = 0.f;
#pragma unroll
    for (int n = 0; n < NT; ++n) v += acc[n][0] + acc[n][1] + acc[n][2] + acc[n][3];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = v;
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int NT, bool DQ>
void run(int warps) {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 148 * 1024 * 4);
    const int iters = 2000;
    k<NT, DQ><<<148, warps * 32>>>(iters, d, sink);
    k<NT, DQ><<<148, warps * 32>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // per iteration the CTA covers warps x 16 rows x 128 K; a step is 128 rows x 256 K = 32K weights
    const double weights_per_iter = warps * 16.0 * 128.0;
    const double cyc_per_step = double(h[0]) / iters * (32768.0 / weights_per_iter);
    printf("%s NT=%d (N=%3d tokens) warps=%2d: %.0f cycles per 128x256 step per SM (%s)\n", DQ ? "dequant+hmma" : "hmma only   ",
           NT, NT * 8, warps, cyc_per_step, cudaGetErrorString(e));
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    for (int w : {8, 16}) {
        run<1, false>(w);
        run<1, true>(w);
        run<2, true>(w);
        run<4, true>(w);
        run<4, false>(w);
        run<8, true>(w);
    }
    return 0;
}
