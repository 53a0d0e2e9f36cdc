// sm_100a kernels of the paper's comparison layouts:
// GPU ports of the reference's bench baselines (ref: infer.cpp:187-339, the
// bench harness infer.cpp:371-426) so the fused 2D layout's overhead and
// dispatch structure can be measured against them on the same hardware.
//
//   lr_right_kernel   one (token, expert) right-factor multiply of the
//                     element-wise layout: mid[j] = sigma_j * <V_q[j] / s_k, x_b>
//                     (baseline_elementwise_forward, infer.cpp:207-215); with a
//                     token grid dimension it is the 1D layout's shared
//                     projection (baseline_1d_forward, infer.cpp:245-246).
//   lr_left_kernel    one (token, expert) output multiply: acc_b += g * U . mid
//                     (infer.cpp:216-222 / 258-264).
//   dequant_all_kernel  the dequant_only layout: every resident expert's
//                     residual materialised as fp16 (infer.cpp:409-411 calls
//                     dequantize() for every expert, quant.cpp:285-323).
//
// Numerics: f32 accumulation (the reference accumulates in f64); outputs are
// checked against the reference within the tolerances in tests/.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tq_internal.h"
#include "tq_ptx.cuh"

namespace tqb {

constexpr int kLrThreads = 256;

// mid[b * mid_ld + j] = scale[j] * sum_c A[j * a_ld + c] * x[b * x_ld + c]
// grid (rows of A, tokens); A f32 row-major; one CTA reduces one row for one token
__global__ void __launch_bounds__(kLrThreads) lr_right_kernel(const float* __restrict__ A, int64_t a_ld,
                                                               const float* __restrict__ x, int64_t x_ld, int n,
                                                               const float* __restrict__ scale,
                                                               float* __restrict__ mid, int64_t mid_ld) {
    __shared__ float part[kLrThreads / 32];
    const int j = blockIdx.x, b = blockIdx.y;
    const float* a = A + static_cast<int64_t>(j) * a_ld;
    const float* xb = x + static_cast<int64_t>(b) * x_ld;
    float acc = 0.0f;
    for (int c = threadIdx.x * 4; c < n; c += kLrThreads * 4) {
        if (c + 3 < n && ((reinterpret_cast<uintptr_t>(a + c) | reinterpret_cast<uintptr_t>(xb + c)) & 15) == 0) {
            const float4 av = *reinterpret_cast<const float4*>(a + c);
            const float4 xv = *reinterpret_cast<const float4*>(xb + c);
            acc = fmaf(av.x, xv.x, acc);
            acc = fmaf(av.y, xv.y, acc);
            acc = fmaf(av.z, xv.z, acc);
            acc = fmaf(av.w, xv.w, acc);
        } else {
            for (int q = c; q < c + 4 && q < n; ++q) acc = fmaf(a[q], xb[q], acc);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int w = 0; w < kLrThreads / 32; ++w) s += part[w];
        mid[static_cast<int64_t>(b) * mid_ld + j] = scale ? s * scale[j] : s;
    }
}

// acc[c] += g * sum_j U[c * r + j] * mid[j]   (U: o x r f32 row-major)
__global__ void __launch_bounds__(kLrThreads) lr_left_kernel(const float* __restrict__ U, int o, int r,
                                                              const float* __restrict__ mid, const float* __restrict__ gate,
                                                              float* __restrict__ acc) {
    __shared__ float s_mid[256];
    for (int j = threadIdx.x; j < r && j < 256; j += blockDim.x) s_mid[j] = mid[j];
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= o) return;
    const float* u = U + static_cast<int64_t>(c) * r;
    float d = 0.0f;
    for (int j = 0; j < r; ++j) d = fmaf(u[j], s_mid[j], d);
    acc[c] += gate[0] * d;
}

// W[w][row][col] (fp16) = (code * s' - zero * s') * 2^-k for every resident
// weight: one CTA per (64-column code block, m-block, weight), thread = row.
// Reads the engine's repacked layout (tq_runtime.cpp repack_qmat): code block
// [w][mb][kb] of BITS x 2 halves x 128 rows of u32 super-words, scale slabs
// [w][mb][group][128] (prescaled s'), ext blocks [w][mb] whose first G
// columns hold -zero * s' (fp16, rounded once at load).
template <int BITS>
__global__ void __launch_bounds__(128) dequant_all_kernel(const DequantAllArgs a) {
    const int kb = blockIdx.x, mb = blockIdx.y, w = blockIdx.z, r = threadIdx.x;
    const int64_t row = static_cast<int64_t>(mb) * kBM + r;
    if (row >= a.o) return;
    constexpr int kBlk = code_block_bytes(BITS);
    const uint32_t* blk = reinterpret_cast<const uint32_t*>(
        a.codes + static_cast<int64_t>(w) * a.weight_stride + (static_cast<int64_t>(mb) * a.kb_total + kb) * kBlk);
    const int64_t wm = static_cast<int64_t>(w) * a.mb_count + mb;
    const uint16_t* ext = reinterpret_cast<const uint16_t*>(a.ext_blocks + wm * a.ext_bytes);
    const float oscale = a.w_outscale[w];
    __half* out = a.out + (static_cast<int64_t>(w) * a.o + row) * a.i;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int col0 = kb * 64 + 32 * h;
        if (col0 >= a.i) break;
        const int g = col0 / a.group_size;   // a 32-column super-word lies in one group (group_size % 32 == 0)
        const uint16_t sb = a.scales[(wm * a.groups + g) * kBM + r];
        uint32_t v[16];
        if constexpr (BITS == kDenseBits) {
            // codebook residuals resolved to fp16 weights at load: the block IS the weights
            (void)sb;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = blk[(h * 16 + q) * kBM + r];
        } else {
            uint32_t words[BITS];
#pragma unroll
            for (int q = 0; q < BITS; ++q) words[q] = blk[(h * BITS + q) * kBM + r];
            dequant32<BITS>(words, make_dq(__ushort_as_half(sb)), v);
        }
        // ext column g (block g/64): u32 word ((g%64)/32*16 + (g%32)/2) of row r, half g%2
        const int gb = g >> 6, gc = g & 63;
        const uint16_t zb = ext[static_cast<int64_t>(gb) * (code_block_bytes(kDenseBits) / 2) +
                                ((((gc >> 5) * 16 + ((gc & 31) >> 1)) * kBM + r) * 2 + (gc & 1))];
        const float z = __half2float(__ushort_as_half(zb));
        __align__(16) __half o16[32];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const __half2 p = *reinterpret_cast<const __half2*>(&v[q]);
            o16[2 * q] = __float2half_rn((__low2float(p) + z) * oscale);
            o16[2 * q + 1] = __float2half_rn((__high2float(p) + z) * oscale);
        }
        const int ncol = static_cast<int>(a.i - col0 < 32 ? a.i - col0 : 32);
        if (ncol == 32 && (reinterpret_cast<uintptr_t>(out + col0) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) reinterpret_cast<int4*>(out + col0)[q] = reinterpret_cast<const int4*>(o16)[q];
        } else {
            for (int q = 0; q < ncol; ++q) out[col0 + q] = o16[q];
        }
    }
}

cudaError_t launch_lr_right(const float* A, int64_t a_ld, int rows, const float* x, int64_t x_ld, int tokens, int n,
                            const float* scale, float* mid, int64_t mid_ld, cudaStream_t stream) {
    if (rows <= 0 || tokens <= 0) return cudaSuccess;
    lr_right_kernel<<<dim3(rows, tokens), kLrThreads, 0, stream>>>(A, a_ld, x, x_ld, n, scale, mid, mid_ld);
    return cudaGetLastError();
}

cudaError_t launch_lr_left(const float* U, int o, int r, const float* mid, const float* gate, float* acc,
                           cudaStream_t stream) {
    if (o <= 0) return cudaSuccess;
    if (r > 256) return cudaErrorInvalidValue;
    lr_left_kernel<<<(o + kLrThreads - 1) / kLrThreads, kLrThreads, 0, stream>>>(U, o, r, mid, gate, acc);
    return cudaGetLastError();
}

cudaError_t launch_dequant_all(const DequantAllArgs& a, int bits, cudaStream_t stream) {
    if (a.n_weights <= 0) return cudaSuccess;
    if (a.group_size % 32 != 0) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>(a.kb_total), static_cast<unsigned>(a.mb_count),
                    static_cast<unsigned>(a.n_weights));
    switch (bits) {
        case 2: dequant_all_kernel<2><<<grid, 128, 0, stream>>>(a); break;
        case 3: dequant_all_kernel<3><<<grid, 128, 0, stream>>>(a); break;
        case 4: dequant_all_kernel<4><<<grid, 128, 0, stream>>>(a); break;
        case 8: dequant_all_kernel<8><<<grid, 128, 0, stream>>>(a); break;
        case kDenseBits: dequant_all_kernel<kDenseBits><<<grid, 128, 0, stream>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace tqb
