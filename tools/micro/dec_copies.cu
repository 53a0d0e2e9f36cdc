// Microbenchmark: the decode GEMM's copy pipeline alone.  Per step a CTA bulk-copies
// 12 KB of codes + a 512 B scale slice (code producers, even / odd steps) and XB bytes
// of activation rows (activation producers, even / odd steps) into an S-stage ring;
// 8 consumer warps only wait and release.  148 persistent CTAs, `steps` steps each.
// Prints cycles per step per SM and the implied HBM rate -- the floor the decode GEMM
// can reach before any dequant / MMA work.
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "../../paper_2605_09281_b200/csrc/tq_ptx.cuh"

using namespace tqb;

__global__ void __launch_bounds__(384, 1) k(const uint8_t* codes, const uint8_t* scales, const uint8_t* xs, int steps, int xb,
                                           int nst, int sb, int use_sc, unsigned long long* out, int xsplit) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * sb);
    uint64_t* empty = full + 32;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(&full[i], 2);
            mbar_init(&empty[i], 8);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    const uint8_t* cbase = codes + static_cast<size_t>(blockIdx.x) * steps * 12288;
    if (wid >= 8) {
        const int pw = wid - 8, par = pw & 1;
        const bool cp = pw < 2;
        int st = par;
        uint32_t ph = 0;
        for (int j = par; j < steps; j += 2) {
            mbar_wait(&empty[st], ph ^ 1u);
            uint8_t* dst = sm + st * sb;
            if (elect_one()) {
                if (cp) {
                    mbar_arrive_expect_tx(&full[st], 12288 + (use_sc ? 512 : 0));
                    bulk_copy_g2s(dst, cbase + static_cast<size_t>(j) * 12288, 12288, &full[st]);
                    if (use_sc) bulk_copy_g2s(dst + 12288, scales + (static_cast<size_t>(blockIdx.x) * steps + j) * 512, 512, &full[st]);
                } else {
                    mbar_arrive_expect_tx(&full[st], xb);
                    // xsplit pieces: the activation rows of a step as 1 or 4 (one per 64-K atom) copies
                    for (int q = 0; q < xsplit && xb; ++q)
                        bulk_copy_g2s(dst + 13312 + q * (xb / xsplit), xs + static_cast<size_t>(j % 16) * 32768 + q * 8192,
                                      xb / xsplit, &full[st]);
                }
            }
            __syncwarp();
            st += 2;
            if (st >= nst) {
                st -= nst;
                ph ^= 1u;
            }
        }
    } else {
        int st = 0;
        uint32_t ph = 0;
        for (int j = 0; j < steps; ++j) {
            mbar_wait(&full[st], ph);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == nst) {
                st = 0;
                ph ^= 1u;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    const int maxsteps = 1024;
    uint8_t *codes, *scales, *xs;
    cudaMalloc(&codes, static_cast<size_t>(148) * maxsteps * 12288);
    cudaMalloc(&scales, static_cast<size_t>(148) * maxsteps * 512);
    cudaMalloc(&xs, 16 * 32768);
    cudaMemset(codes, 1, static_cast<size_t>(148) * maxsteps * 12288);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    unsigned long long h[148];
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    uint8_t* flush;
    cudaMalloc(&flush, 512 << 20);
    auto run = [&](int steps, int xb, int nst, int use_sc, int xsplit = 1) {
        const int sb = 13312 + 16384;
        const int smem = nst * sb + 1024;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float best = 1e9f;
        for (int r = 0; r < 3; ++r) {
            cudaMemset(flush, r, 512 << 20);
            cudaEventRecord(a);
            k<<<148, 384, smem>>>(codes, scales, xs, steps, xb, nst, sb, use_sc, d, xsplit);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        const double bytes = 148.0 * steps * (12288 + (use_sc ? 512 : 0) + xb);
        printf("steps %4d xb %5d x-copies %d scales %d stages %2d: %7.2f us  %6.0f cycles/step (CTA 0)  %7.1f GB/s  (%s)\n",
               steps, xb, xsplit, use_sc, nst, best * 1e3, double(h[0]) / steps, bytes / (best * 1e-3) / 1e9,
               cudaGetErrorString(e));
    };
    for (int steps : {26, 103})
        for (int xs : {1, 4}) {
            run(steps, 4096, 7, 1, xs);
            run(steps, 16384, 7, 1, xs);
        }
    run(26, 1024, 7, 1, 4);
    run(26, 1024, 7, 1, 1);
    return 0;
}
