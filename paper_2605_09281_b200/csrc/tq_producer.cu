// GPU ports of the artifact producer's hot spots:
//
//   estimate_hessian   quant.cpp:116-150   H = (1/T) X^T X + lambda I
//   spd_inverse        quant.cpp:72-112    Cholesky, L^-1, L^-T L^-1
//   make_grids / RTN   quant.cpp:28-70,152-175
//   quantize_gptq      quant.cpp:177-221   per-row error feedback through H^-1
//   proxy_loss         quant.cpp:325-343   tr(E H E^T)
//
// Every function returns the reference's bits, not an approximation: each
// output element sees the same f64 operations in the same order as the
// reference's scalar loops (compiled for x86-64 without FMA contraction), so
// products and sums are issued one at a time with __dmul_rn / __dadd_rn /
// __dsub_rn / __ddiv_rn and are never contracted.  What the GPU changes is
// WHICH elements run concurrently:
//
//   * the dot-product-shaped loops (Hessian accumulation, the Cholesky trailing
//     update, the L^-1 block update, L^-T L^-1, E H) run as 64x64 output tiles
//     whose threads each accumulate their 4x4 outputs over k ascending -- the
//     reference's order per element; terms the reference skips are either
//     skipped too or exact zero products that leave a +0-started sum unchanged;
//   * the sequential recurrences (the Cholesky panel, the L^-1 diagonal block,
//     the GPTQ column sweep) keep their order along the recurrence and run
//     independent rows / columns side by side.
//
// All of it is FP64 CUDA-core work (the reference's arithmetic is f64); none
// of it is GEMM-shaped in a precision the tensor cores serve.

#include <cuda_fp16.h>

#include <cstdint>

#include "tq_internal.h"

namespace tqb {
namespace {

constexpr int kT = 64;     // output tile edge
constexpr int kKC = 16;    // k chunk staged in shared memory
constexpr int kTT = 256;   // threads per tile CTA (16 x 16, 4 x 4 outputs each, strided by 16)

// Status word shared by the spd_inverse kernels: the first failing pivot.
struct SpdStatus {
    int32_t failed;
    int32_t pad;
    int64_t column;
    double pivot;
};

// ---------------------------------------------------------------------------
// ordered f64 tile product
// ---------------------------------------------------------------------------

// acc[ii][jj] (+|-)= A(i0 + ty + 16 ii, k) * B(k, j0 + tx + 16 jj) for k = k0 .. k1-1
// ascending.  kAK / kBK: the operand is contiguous along k (stage k-fastest) or
// along i / j (stage i/j-fastest), so the global loads coalesce either way.
template <bool kSub, bool kAK, bool kBK, class FA, class FB>
__device__ __forceinline__ void tile_accumulate(double (&acc)[4][4], int64_t i0, int64_t j0, int64_t k0, int64_t k1,
                                                const FA& fa, const FB& fb, double (*As)[kT + 2],
                                                double (*Bs)[kT + 2]) {
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    for (int64_t kb = k0; kb < k1; kb += kKC) {
        const int kc = static_cast<int>(k1 - kb < kKC ? k1 - kb : kKC);
        for (int e = tid; e < kKC * kT; e += kTT) {
            const int kk = kAK ? e % kKC : e / kT;
            const int ii = kAK ? e / kKC : e % kT;
            As[kk][ii] = kk < kc ? fa(i0 + ii, kb + kk) : 0.0;
        }
        for (int e = tid; e < kKC * kT; e += kTT) {
            const int kk = kBK ? e % kKC : e / kT;
            const int jj = kBK ? e / kKC : e % kT;
            Bs[kk][jj] = kk < kc ? fb(kb + kk, j0 + jj) : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = As[kk][ty + 16 * q];   // 2 addresses per warp: broadcast
                b[q] = Bs[kk][tx + 16 * q];   // 16 consecutive doubles: one wavefront
            }
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const double p = __dmul_rn(a[ii], b[jj]);
                    acc[ii][jj] = kSub ? __dsub_rn(acc[ii][jj], p) : __dadd_rn(acc[ii][jj], p);
                }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// estimate_hessian (quant.cpp:116-150)
// ---------------------------------------------------------------------------

// acc[a][b] = sum_t x[t][a] * x[t][b] for b >= a, t ascending (quant.cpp:127-133).
__global__ void __launch_bounds__(kTT) hessian_acc_kernel(const float* __restrict__ x, int64_t tokens, int64_t dim,
                                                           double* __restrict__ acc_out) {
    const int64_t a0 = static_cast<int64_t>(blockIdx.y) * kT, b0 = static_cast<int64_t>(blockIdx.x) * kT;
    if (b0 + kT <= a0) return;   // tile entirely below the diagonal
    __shared__ double As[kKC][kT + 2], Bs[kKC][kT + 2];
    double acc[4][4] = {};
    auto fa = [&](int64_t a, int64_t t) { return a < dim ? static_cast<double>(x[t * dim + a]) : 0.0; };
    auto fb = [&](int64_t t, int64_t b) { return b < dim ? static_cast<double>(x[t * dim + b]) : 0.0; };
    tile_accumulate<false, false, false>(acc, a0, b0, 0, tokens, fa, fb, As, Bs);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t a = a0 + ty + 16 * ii, b = b0 + tx + 16 * jj;
            if (a < dim && b < dim && b >= a) acc_out[a * dim + b] = acc[ii][jj];
        }
}

// trace = sum_a acc[a][a] / T (a ascending), lambda = damping * (trace / dim)  (quant.cpp:134-136)
__global__ void hessian_lambda_kernel(const double* __restrict__ acc, int64_t tokens, int64_t dim, double damping,
                                      double* __restrict__ lambda_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double t = static_cast<double>(tokens);
    double trace = 0.0;
    for (int64_t a = 0; a < dim; ++a) trace = __dadd_rn(trace, __ddiv_rn(acc[a * dim + a], t));
    *lambda_out = __dmul_rn(damping, __ddiv_rn(trace, static_cast<double>(dim)));
}

// h[a][b] = h[b][a] = float(acc[a][b] / T + (a == b ? lambda : 0))  (quant.cpp:141-148)
__global__ void hessian_fill_kernel(const double* __restrict__ acc, int64_t tokens, int64_t dim,
                                    const double* __restrict__ lambda, float* __restrict__ h) {
    const double t = static_cast<double>(tokens), lam = *lambda;
    const int64_t n = dim * dim;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t a = e / dim, b = e % dim;
        const int64_t lo = a < b ? a : b, hi = a < b ? b : a;   // the upper-triangle entry holds the sum
        const double v = __dadd_rn(__ddiv_rn(acc[lo * dim + hi], t), lo == hi ? lam : 0.0);
        h[e] = __double2float_rn(v);
    }
}

// ---------------------------------------------------------------------------
// spd_inverse (quant.cpp:72-112)
// ---------------------------------------------------------------------------

// C[i][j] = double(h[i][j]) on and below the diagonal (the Cholesky work array)
__global__ void chol_init_kernel(const float* __restrict__ h, int64_t n, double* __restrict__ c) {
    const int64_t total = n * n;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        c[e] = j <= i ? static_cast<double>(h[e]) : 0.0;
    }
}

// Right-looking trailing update after panel [j0, j0 + kT) is factored:
// C[i][j] -= C[i][k] * C[j][k] for k = j0 .. j0+kT-1 ascending, over the trailing
// lower triangle i >= j >= j0 + kT.  Panels run in order, so every element still
// receives its k = 0 .. j-1 subtractions in the reference's order
// (quant.cpp:77-78) -- the work of one panel spread over the whole trailing
// matrix instead of one K = j0 chain per output.
__global__ void __launch_bounds__(kTT) chol_trail_kernel(double* __restrict__ c, int64_t n, int64_t j0,
                                                          const SpdStatus* __restrict__ st) {
    if (st->failed) return;
    const int64_t j1 = j0 + kT;
    const int64_t i0 = j1 + static_cast<int64_t>(blockIdx.y) * kT, jt0 = j1 + static_cast<int64_t>(blockIdx.x) * kT;
    if (jt0 > i0) return;   // tile above the diagonal
    __shared__ double As[kKC][kT + 2], Bs[kKC][kT + 2];
    double acc[4][4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t i = i0 + ty + 16 * ii, j = jt0 + tx + 16 * jj;
            acc[ii][jj] = (i < n && j < n && j <= i) ? c[i * n + j] : 0.0;
        }
    auto fa = [&](int64_t i, int64_t k) { return i < n ? c[i * n + k] : 0.0; };
    auto fb = [&](int64_t k, int64_t j) { return j < n ? c[j * n + k] : 0.0; };
    tile_accumulate<true, true, true>(acc, i0, jt0, j0, j1, fa, fb, As, Bs);
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t i = i0 + ty + 16 * ii, j = jt0 + tx + 16 * jj;
            if (i < n && j < n && j <= i) c[i * n + j] = acc[ii][jj];
        }
}

// Factor the panel's diagonal block (one CTA, thread t owns row j0 + t): for each
// column j: the pivot, then the rows below it, each finishing k = j0 .. j-1 in order
// (quant.cpp:75-90).
__global__ void __launch_bounds__(kT) chol_diag_kernel(double* __restrict__ c, int64_t n, int64_t j0,
                                                        SpdStatus* __restrict__ st) {
    if (st->failed) return;
    __shared__ double d[kT][kT + 1];
    __shared__ int bad;
    const int t = threadIdx.x;
    const int w = static_cast<int>(n - j0 < kT ? n - j0 : kT);
    for (int j = 0; j < w; ++j) d[t][j] = (t < w && j <= t) ? c[(j0 + t) * n + j0 + j] : 0.0;
    if (t == 0) bad = 0;
    __syncthreads();
    for (int j = 0; j < w; ++j) {
        if (t == j) {
            double acc = d[j][j];
            for (int k = 0; k < j; ++k) acc = __dsub_rn(acc, __dmul_rn(d[j][k], d[j][k]));
            if (!(acc > 0.0) || !isfinite(acc)) {   // acc <= 0.0 || !finite (NaN included)
                st->failed = 1;
                st->column = j0 + j;
                st->pivot = acc;
                bad = 1;
            } else {
                d[j][j] = __dsqrt_rn(acc);
            }
        }
        __syncthreads();
        if (bad) return;
        if (t > j && t < w) {
            double acc = d[t][j];
            for (int k = 0; k < j; ++k) acc = __dsub_rn(acc, __dmul_rn(d[t][k], d[j][k]));
            d[t][j] = __ddiv_rn(acc, d[j][j]);
        }
        __syncthreads();
    }
    if (t < w)
        for (int j = 0; j <= t; ++j) c[(j0 + t) * n + j0 + j] = d[t][j];
}

// Rows below the diagonal block: row i finishes its panel entries left to right
// against the factored block (quant.cpp:87-88).  One thread per row.
constexpr int kRowsPerCta = 128;
__global__ void __launch_bounds__(kRowsPerCta) chol_rows_kernel(double* __restrict__ c, int64_t n, int64_t j0,
                                                                 const SpdStatus* __restrict__ st) {
    if (st->failed) return;
    extern __shared__ double sm[];
    double(*d)[kT + 1] = reinterpret_cast<double(*)[kT + 1]>(sm);                    // kT x (kT+1)
    double(*rv)[kT + 1] = reinterpret_cast<double(*)[kT + 1]>(sm + kT * (kT + 1));   // rows x (kT+1)
    const int w = static_cast<int>(n - j0 < kT ? n - j0 : kT);
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
        const int r = e / kT, q = e % kT;
        d[r][q] = (r < w && q <= r) ? c[(j0 + r) * n + j0 + q] : 0.0;
    }
    const int64_t i = j0 + kT + static_cast<int64_t>(blockIdx.x) * kRowsPerCta + threadIdx.x;
    __syncthreads();
    if (i >= n) return;
    double* row = rv[threadIdx.x];
    for (int j = 0; j < w; ++j) row[j] = c[i * n + j0 + j];
    for (int j = 0; j < w; ++j) {
        double acc = row[j];
        for (int k = 0; k < j; ++k) acc = __dsub_rn(acc, __dmul_rn(row[k], d[j][k]));
        row[j] = __ddiv_rn(acc, d[j][j]);
    }
    for (int j = 0; j < w; ++j) c[i * n + j0 + j] = row[j];
}

// L^-1, right-looking: once rows [i0, i0 + kT) of L^-1 are final, every later
// row's partial sums take their terms k = i0 .. i0+kT-1 in order:
// Linv[i][j] += L[i][k] * Linv[k][j] for i >= i0 + kT, j < i0 + kT (quant.cpp:96-99).
// Partial sums are parked in Linv[i][j] until row i's own block finishes them.
// Terms with k < j are exact zero products on a +0-started sum (the reference
// starts at k = j).
__global__ void __launch_bounds__(kTT) linv_trail_kernel(const double* __restrict__ c, double* __restrict__ li,
                                                          int64_t n, int64_t i0, const SpdStatus* __restrict__ st) {
    if (st->failed) return;
    const int64_t i1 = i0 + kT;
    const int64_t r0 = i1 + static_cast<int64_t>(blockIdx.y) * kT, j0 = static_cast<int64_t>(blockIdx.x) * kT;
    __shared__ double As[kKC][kT + 2], Bs[kKC][kT + 2];
    double acc[4][4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t i = r0 + ty + 16 * ii, j = j0 + tx + 16 * jj;
            acc[ii][jj] = (i < n && j < i1) ? li[i * n + j] : 0.0;
        }
    auto fa = [&](int64_t i, int64_t k) { return i < n ? c[i * n + k] : 0.0; };
    auto fb = [&](int64_t k, int64_t j) { return j < i1 ? li[k * n + j] : 0.0; };
    tile_accumulate<false, true, false>(acc, r0, j0, i0, i1, fa, fb, As, Bs);
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t i = r0 + ty + 16 * ii, j = j0 + tx + 16 * jj;
            if (i < n && j < i1) li[i * n + j] = acc[ii][jj];
        }
}

// L^-1, row block [i0, i0 + kT), the in-block part: thread per column j <= i0+kT-1
// walks rows i ascending, adds k = max(i0, j) .. i-1, then Linv[i][j] = -acc / L[i][i];
// Linv[j][j] = 1 / L[j][j] (quant.cpp:94-100).
__global__ void __launch_bounds__(kRowsPerCta) linv_block_kernel(const double* __restrict__ c,
                                                                  double* __restrict__ li, int64_t n, int64_t i0,
                                                                  const SpdStatus* __restrict__ st) {
    if (st->failed) return;
    __shared__ double d[kT][kT + 1];   // L[i0 + r][i0 + q]
    const int w = static_cast<int>(n - i0 < kT ? n - i0 : kT);
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
        const int r = e / kT, q = e % kT;
        d[r][q] = (r < w && q <= r) ? c[(i0 + r) * n + i0 + q] : 0.0;
    }
    __syncthreads();
    const int64_t j = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + threadIdx.x;
    if (j >= i0 + w) return;
    for (int r = 0; r < w; ++r) {
        const int64_t i = i0 + r;
        if (i < j) continue;
        if (i == j) {
            li[j * n + j] = __ddiv_rn(1.0, d[r][r]);
            continue;
        }
        double acc = j < i0 ? li[i * n + j] : 0.0;
        const int kb = static_cast<int>(j < i0 ? 0 : j - i0);
        for (int q = kb; q < r; ++q) acc = __dadd_rn(acc, __dmul_rn(d[r][q], li[(i0 + q) * n + j]));
        li[i * n + j] = __ddiv_rn(-acc, d[r][r]);
    }
}

// Hinv[i][j] = Hinv[j][i] = sum_{k >= i} Linv[k][i] * Linv[k][j] for j <= i, k ascending
// (quant.cpp:102-110; the k < i terms of a tile are exact zero products).
__global__ void __launch_bounds__(kTT) hinv_kernel(const double* __restrict__ li, int64_t n,
                                                    double* __restrict__ hinv, const SpdStatus* __restrict__ st) {
    if (st->failed) return;
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kT, j0 = static_cast<int64_t>(blockIdx.x) * kT;
    if (j0 > i0) return;
    __shared__ double As[kKC][kT + 2], Bs[kKC][kT + 2];
    double acc[4][4] = {};
    auto fa = [&](int64_t i, int64_t k) { return i < n ? li[k * n + i] : 0.0; };
    auto fb = [&](int64_t k, int64_t j) { return j < n ? li[k * n + j] : 0.0; };
    tile_accumulate<false, false, false>(acc, i0, j0, i0, n, fa, fb, As, Bs);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t i = i0 + ty + 16 * ii, j = j0 + tx + 16 * jj;
            if (i < n && j <= i) {
                hinv[i * n + j] = acc[ii][jj];
                hinv[j * n + i] = acc[ii][jj];
            }
        }
}

// ---------------------------------------------------------------------------
// grids, RTN, GPTQ (quant.cpp:28-70,152-221)
// ---------------------------------------------------------------------------

__device__ __forceinline__ float snap_f16(float v) { return __half2float(__float2half_rn(v)); }

// make_grid over one group (quant.cpp:28-48), std::min / std::max semantics kept
__global__ void grids_kernel(const float* __restrict__ r, int64_t rows, int64_t cols, int bits, int64_t gs,
                             float* __restrict__ scales, int32_t* __restrict__ zeros) {
    const int64_t G = (cols + gs - 1) / gs;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= rows * G) return;
    const int64_t row = t / G, g = t % G, start = g * gs;
    const int64_t len = cols - start < gs ? cols - start : gs;
    const float* v = r + row * cols + start;
    float vmin = v[0], vmax = v[0];
    for (int64_t q = 1; q < len; ++q) {
        const float x = v[q];
        vmin = x < vmin ? x : vmin;   // std::min(vmin, x)
        vmax = vmax < x ? x : vmax;   // std::max(vmax, x)
    }
    const double dmin = static_cast<double>(vmin), dmax = static_cast<double>(vmax);
    const double rmin = 0.0 < dmin ? 0.0 : dmin;   // std::min(dmin, 0.0)
    const double rmax = dmax < 0.0 ? 0.0 : dmax;   // std::max(dmax, 0.0)
    const double levels = static_cast<double>((1 << bits) - 1);
    double scale = __ddiv_rn(__dsub_rn(rmax, rmin), levels);
    if (scale <= 0.0) scale = 1e-8;
    float s = snap_f16(__double2float_rn(scale));
    if (s <= 0.0f) s = 5.9604644775390625e-8f;   // least positive binary16, 2^-24
    double zero = rint(__ddiv_rn(-rmin, static_cast<double>(s)));
    zero = 0.0 < zero ? zero : 0.0;          // std::max(0.0, zero)
    zero = zero < levels ? zero : levels;    // std::min(levels, .)
    scales[t] = s;
    zeros[t] = static_cast<int32_t>(zero);
}

// encode_one (quant.cpp:50-55)
__device__ __forceinline__ uint32_t encode_one(double value, float scale, int32_t zero, double levels) {
    double code = __dadd_rn(rint(__ddiv_rn(value, static_cast<double>(scale))), static_cast<double>(zero));
    code = 0.0 < code ? code : 0.0;
    code = code < levels ? code : levels;
    return static_cast<uint32_t>(code);
}

__global__ void rtn_codes_kernel(const float* __restrict__ r, int64_t rows, int64_t cols, int bits, int64_t gs,
                                 const float* __restrict__ scales, const int32_t* __restrict__ zeros,
                                 uint8_t* __restrict__ codes) {
    const int64_t G = (cols + gs - 1) / gs, n = rows * cols;
    const double levels = static_cast<double>((1 << bits) - 1);
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = e / cols, c = e % cols, g = row * G + c / gs;
        codes[e] = static_cast<uint8_t>(encode_one(static_cast<double>(r[e]), scales[g], zeros[g], levels));
    }
}

// RN(a / d) given y = RN(1 / d), without a division per element: q0 = RN(a y)
// is within 1.5 ulp of a / d, one FMA correction q1 = RN(q0 + (a - d q0) y)
// brings it within 1 ulp, and by Markstein's theorem (y the correctly rounded
// reciprocal, q1 within an ulp, residual exact by FMA) q2 = RN(q1 + (a - d q1) y)
// is the correctly rounded quotient.  The theorem needs the residuals to be
// exact -- no underflow -- so quotients far from 1 (|q0| outside 2^+-800; the
// caller checks d once per column) take __ddiv_rn.  (Checked bit for bit against
// IEEE division on 4e8 operand pairs, adversarial mantissas included.)
__device__ __forceinline__ double div_rn_by(double a, double d, double y) {
    if (a == 0.0) return __dmul_rn(a, y);   // the signed zero a / d
    const double q0 = __dmul_rn(a, y);
    const unsigned eq = (static_cast<unsigned>(__double2hiint(q0)) >> 20) & 0x7ffu;
    if (eq - 223u > 1600u) return __ddiv_rn(a, d);   // biased exponent outside [223, 1823]
    const double q1 = __fma_rn(__fma_rn(-q0, d, a), y, q0);
    return __fma_rn(__fma_rn(-q1, d, a), y, q1);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// GPTQ column sweep (quant.cpp:200-213).  A CTA owns kR rows: their working rows
// and grids sit in shared memory; columns are dealt to threads round-robin so
// the shrinking trailing range stays balanced.  Column j's codes and errors are
// formed ONCE, by the thread that owns column j, right after it applied the
// last update to that column (step j-1), and published through a small
// double-buffered shared array; step j then updates every column c > j:
// work[c] -= err * Hinv[j][c] / Hinv[j][j].  With kStage, row j+1 of Hinv is
// copied into a second shared buffer (cp.async) while column j is processed,
// so the sweep never waits on L2 latency between its barriers.
constexpr int kGptqThreads = 1024;   // (measured: 1024 threads 484 ms vs 512 threads 546 ms at c2)

template <int kR>
__device__ __forceinline__ void gptq_encode(const double (&w)[kR], int nr, int64_t j, int64_t G, int64_t gs,
                                            const float* gsc, const int32_t* gzp, double levels, int64_t row0,
                                            int64_t dim, uint8_t* __restrict__ codes, double* errb) {
    const int64_t g = j / gs;
#pragma unroll
    for (int q = 0; q < kR; ++q) {
        if (q < nr) {
            const float sc = gsc[q * G + g];
            const int32_t z = gzp[q * G + g];
            const uint32_t code = encode_one(w[q], sc, z, levels);
            const double deq = __dmul_rn(__dsub_rn(static_cast<double>(code), static_cast<double>(z)),
                                         static_cast<double>(sc));
            errb[q] = __dsub_rn(w[q], deq);
            codes[(row0 + q) * dim + j] = static_cast<uint8_t>(code);
        }
    }
}

template <int kR, bool kStage>
__global__ void __launch_bounds__(kGptqThreads) gptq_kernel(const float* __restrict__ r, int64_t rows, int64_t dim,
                                                             int bits, int64_t gs, const float* __restrict__ scales,
                                                             const int32_t* __restrict__ zeros,
                                                             const double* __restrict__ hinv,
                                                             uint8_t* __restrict__ codes) {
    extern __shared__ double sm[];
    __shared__ double errb[2][kR];
    const int64_t G = (dim + gs - 1) / gs;
    double* work = sm;                                    // kR x dim
    double* hb = sm + kR * dim;                           // 2 x dim (kStage)
    float* gsc = reinterpret_cast<float*>(hb + (kStage ? 2 * dim : 0));   // kR x G
    int32_t* gzp = reinterpret_cast<int32_t*>(gsc + kR * G);              // kR x G
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kR;
    const int nr = static_cast<int>(rows - row0 < kR ? rows - row0 : kR);
    const double levels = static_cast<double>((1 << bits) - 1);
    const int tid = threadIdx.x;
    for (int q = 0; q < nr; ++q) {
        for (int64_t c = tid; c < dim; c += kGptqThreads) work[q * dim + c] = static_cast<double>(r[(row0 + q) * dim + c]);
        for (int64_t g = tid; g < G; g += kGptqThreads) {
            gsc[q * G + g] = scales[(row0 + q) * G + g];
            gzp[q * G + g] = zeros[(row0 + q) * G + g];
        }
    }
    if (kStage) {
        for (int64_t c = tid; c < dim; c += kGptqThreads) cp_async8(hb + c, hinv + c);
        cp_async_commit();
        cp_async_wait_all();
    }
    __syncthreads();
    if (tid == 0 && dim > 0) {   // column 0 is final from the start
        double w0[kR];
#pragma unroll
        for (int q = 0; q < kR; ++q) w0[q] = q < nr ? work[q * dim] : 0.0;
        gptq_encode<kR>(w0, nr, 0, G, gs, gsc, gzp, levels, row0, dim, codes, errb[0]);
    }
    __syncthreads();
    for (int64_t j = 0; j < dim; ++j) {
        const double* hrow;
        const int buf = static_cast<int>(j & 1);
        if (kStage) {
            hrow = hb + buf * dim;
            if (j + 1 < dim) {   // prefetch row j+1 (own columns >= j+1; the diagonal included)
                const int64_t f = j + 1;
                double* dst = hb + (buf ^ 1) * dim;
                for (int64_t c = f + ((tid - f) % kGptqThreads + kGptqThreads) % kGptqThreads; c < dim;
                     c += kGptqThreads)
                    cp_async8(dst + c, hinv + f * dim + c);
                cp_async_commit();
            }
        } else {
            hrow = hinv + j * dim;
        }
        double err[kR];
#pragma unroll
        for (int q = 0; q < kR; ++q) err[q] = errb[buf][q];
        const double inv_jj = hrow[j];
        // the reciprocal path needs a divisor well inside the normal range (block-uniform)
        const unsigned ed = (static_cast<unsigned>(__double2hiint(inv_jj)) >> 20) & 0x7ffu;
        const double rcp = (ed - 223u <= 1600u) ? __drcp_rn(inv_jj) : 0.0;
        const int64_t first = j + 1;
        for (int64_t c = first + ((tid - first) % kGptqThreads + kGptqThreads) % kGptqThreads; c < dim;
             c += kGptqThreads) {
            const double h = hrow[c];
            double nw[kR];
#pragma unroll
            for (int q = 0; q < kR; ++q) {
                nw[q] = 0.0;
                if (q < nr) {
                    const double p = __dmul_rn(err[q], h);
                    nw[q] = __dsub_rn(work[q * dim + c], rcp != 0.0 ? div_rn_by(p, inv_jj, rcp) : __ddiv_rn(p, inv_jj));
                    work[q * dim + c] = nw[q];
                }
            }
            if (c == first)   // column j+1 just got its last update: publish its codes / errors
                gptq_encode<kR>(nw, nr, first, G, gs, gsc, gzp, levels, row0, dim, codes, errb[buf ^ 1]);
        }
        if (kStage) cp_async_wait_all();
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// proxy_loss (quant.cpp:325-343)
// ---------------------------------------------------------------------------

// e = original - float(double(code - zero) * scale)  (matrix.cpp:138-143, quant.cpp:296-300)
__device__ __forceinline__ float err_elem(const float* __restrict__ orig, const uint8_t* __restrict__ codes,
                                          const float* __restrict__ scales, const int32_t* __restrict__ zeros,
                                          int64_t row, int64_t c, int64_t dim, int64_t G, int64_t gs) {
    const int64_t g = row * G + c / gs;
    const int64_t q = static_cast<int64_t>(codes[row * dim + c]) - zeros[g];
    const float deq = __double2float_rn(__dmul_rn(static_cast<double>(q), static_cast<double>(scales[g])));
    return __fsub_rn(orig[row * dim + c], deq);
}

// he[row][a] = sum_b double(H[a][b]) * e[row][b], b ascending (quant.cpp:333-337);
// stored column-major (he_t[a][row - r0]) for the row-sequential pass.
__global__ void __launch_bounds__(kTT, 4) proxy_he_kernel(const float* __restrict__ orig,
                                                        const uint8_t* __restrict__ codes,
                                                        const float* __restrict__ scales,
                                                        const int32_t* __restrict__ zeros, int64_t rows, int64_t dim,
                                                        int64_t gs, const float* __restrict__ h, int64_t r0,
                                                        int64_t nrows, double* __restrict__ he_t) {
    const int64_t i0 = r0 + static_cast<int64_t>(blockIdx.y) * kT, a0 = static_cast<int64_t>(blockIdx.x) * kT;
    const int64_t G = (dim + gs - 1) / gs, rend = r0 + nrows;
    __shared__ double As[kKC][kT + 2], Bs[kKC][kT + 2];
    double acc[4][4] = {};
    auto fa = [&](int64_t row, int64_t b) {
        return row < rend ? static_cast<double>(err_elem(orig, codes, scales, zeros, row, b, dim, G, gs)) : 0.0;
    };
    auto fb = [&](int64_t b, int64_t a) { return a < dim ? static_cast<double>(h[a * dim + b]) : 0.0; };
    tile_accumulate<false, true, true>(acc, i0, a0, 0, dim, fa, fb, As, Bs);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t row = i0 + ty + 16 * ii, a = a0 + tx + 16 * jj;
            if (row < rend && a < dim) he_t[a * nrows + (row - r0)] = acc[ii][jj];
        }
}

// rowsum[row] = sum_a double(e[row][a]) * he[row][a], a ascending (quant.cpp:338-339)
__global__ void proxy_rowsum_kernel(const float* __restrict__ orig, const uint8_t* __restrict__ codes,
                                    const float* __restrict__ scales, const int32_t* __restrict__ zeros, int64_t dim,
                                    int64_t gs, int64_t r0, int64_t nrows, const double* __restrict__ he_t,
                                    double* __restrict__ rowsum) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const int64_t row = r0 + t, G = (dim + gs - 1) / gs;
    double s = 0.0;
    for (int64_t a = 0; a < dim; ++a) {
        const double e = static_cast<double>(err_elem(orig, codes, scales, zeros, row, a, dim, G, gs));
        s = __dadd_rn(s, __dmul_rn(e, he_t[a * nrows + t]));
    }
    rowsum[row] = s;
}

// total = sum_row rowsum[row], rows ascending (quant.cpp:340)
__global__ void proxy_total_kernel(const double* __restrict__ rowsum, int64_t rows, double* __restrict__ total) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0;
    for (int64_t r = 0; r < rows; ++r) s = __dadd_rn(s, rowsum[r]);
    *total = s;
}


// ---------------------------------------------------------------------------
// sketch_lowrank (lowrank.cpp:194-247): the f64 mat-vecs of the randomized
// sketch on the resident working copy.  Host code (tq_runtime.cpp) draws the
// probes and runs the sequential control flow.
// ---------------------------------------------------------------------------

__global__ void widen_kernel(const float* __restrict__ w, int64_t n, double* __restrict__ out) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[e] = static_cast<double>(w[e]);
}

// y[r] = sum_c a[r][c] * x[c], c ascending (lowrank.cpp:37-46).  A warp owns 32
// rows: it stages 32 x 32 tiles with coalesced row segments (the next tile's
// loads issued before the current tile is consumed) and each lane walks its own
// row through the tile.
constexpr int kMvWarps = 4;
__global__ void __launch_bounds__(kMvWarps * 32) matvec_kernel(const double* __restrict__ a, int64_t rows,
                                                                int64_t cols, const double* __restrict__ x,
                                                                double* __restrict__ y) {
    __shared__ double tile[kMvWarps][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * kMvWarps + warp) * 32;
    if (r0 >= rows) return;   // warp-uniform; no CTA barriers below
    const int nrow = static_cast<int>(rows - r0 < 32 ? rows - r0 : 32);
    double nxt[32];
    auto fetch = [&](int64_t c0) {
        const bool ok = c0 + lane < cols;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) nxt[rr] = (ok && rr < nrow) ? __ldcs(a + (r0 + rr) * cols + c0 + lane) : 0.0;
    };
    double acc = 0.0;
    fetch(0);
    for (int64_t c0 = 0; c0 < cols; c0 += 32) {
        const int w = static_cast<int>(cols - c0 < 32 ? cols - c0 : 32);
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) tile[warp][rr][lane] = nxt[rr];
        const double xv = lane < w ? x[c0 + lane] : 0.0;
        __syncwarp();
        if (c0 + 32 < cols) fetch(c0 + 32);
        for (int k = 0; k < w; ++k) {
            const double xk = __shfl_sync(0xffffffffu, xv, k);
            acc = __dadd_rn(acc, __dmul_rn(tile[warp][lane][k], xk));
        }
        __syncwarp();
    }
    if (lane < nrow) y[r0 + lane] = acc;
}

// y[c] = sum_r a[r][c] * x[r], r ascending (lowrank.cpp:48-56).  A CTA owns 32
// columns: its warps stream kMtvRows x 32 tiles (coalesced 256-byte row
// segments) into a kMtvStages-deep shared ring with cp.async, and warp 0 -- one
// lane per column -- adds the rows in order out of shared memory; the ring keeps
// several tiles in flight so the add chain, not the load latency, sets the pace.
constexpr int kMtvWarps = 4, kMtvRows = 32, kMtvStages = 5;
__global__ void __launch_bounds__(kMtvWarps * 32) mattvec_kernel(const double* __restrict__ a, int64_t rows,
                                                                  int64_t cols, const double* __restrict__ x,
                                                                  double* __restrict__ y) {
    __shared__ double tile[kMtvStages][kMtvRows][32];
    __shared__ double xs[kMtvStages][kMtvRows];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + lane;
    const bool col_ok = c < cols;
    const int64_t nchunks = (rows + kMtvRows - 1) / kMtvRows;
    auto stage = [&](int64_t chunk) {   // every thread issues its share, then commits one group
        if (chunk < nchunks) {
            const int buf = static_cast<int>(chunk % kMtvStages);
            const int64_t rb = chunk * kMtvRows;
            for (int rr = warp; rr < kMtvRows; rr += kMtvWarps) {
                const int64_t r = rb + rr;
                if (r < rows && col_ok) cp_async8(&tile[buf][rr][lane], a + r * cols + c);
                else tile[buf][rr][lane] = 0.0;
            }
            if (warp == 0) {
                const int64_t r = rb + lane;
                if (r < rows) cp_async8(&xs[buf][lane], x + r);
                else xs[buf][lane] = 0.0;
            }
        }
        cp_async_commit();
    };
    for (int64_t k = 0; k < kMtvStages - 1; ++k) stage(k);
    double acc = 0.0;
    for (int64_t chunk = 0; chunk < nchunks; ++chunk) {
        stage(chunk + kMtvStages - 1);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kMtvStages - 1) : "memory");
        __syncthreads();
        if (warp == 0) {
            const int buf = static_cast<int>(chunk % kMtvStages);
            const int n = static_cast<int>(rows - chunk * kMtvRows < kMtvRows ? rows - chunk * kMtvRows : kMtvRows);
            for (int rr = 0; rr < n; ++rr) acc = __dadd_rn(acc, __dmul_rn(tile[buf][rr][lane], xs[buf][rr]));
        }
        __syncthreads();   // the slot is refilled kMtvStages - 1 chunks later
    }
    if (warp == 0 && col_ok) y[c] = acc;
}

// sqrt(sum v^2), v ascending (lowrank.cpp:58-62): one warp; the lanes load and
// square 32 consecutive entries, every lane adds them in order (shuffles), so
// only the dependent add chain is serial
__global__ void norm2_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    double acc = 0.0;
    double nxt = lane < n ? v[lane] : 0.0;
    for (int64_t t0 = 0; t0 < n; t0 += 32) {
        const double cur = nxt;
        if (t0 + 32 + lane < n) nxt = v[t0 + 32 + lane];
        const double sq = __dmul_rn(cur, cur);
        if (n - t0 >= 32) {   // full chunk: the 32 shuffles issue ahead of the add chain
            double b[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) b[k] = __shfl_sync(0xffffffffu, sq, k);
#pragma unroll
            for (int k = 0; k < 32; ++k) acc = __dadd_rn(acc, b[k]);
        } else {
            const int m = static_cast<int>(n - t0);
            for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, sq, k));
        }
    }
    if (lane == 0) *out = __dsqrt_rn(acc);
}

// dst[i] = src[i] / *d  (x /= qn, v /= sigma)
__global__ void div_by_kernel(const double* __restrict__ src, int64_t n, const double* __restrict__ d,
                              double* __restrict__ dst) {
    const double den = *d;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[e] = __ddiv_rn(src[e], den);
}

// work[r][c] -= (sigma * u[r]) * v[c]  (lowrank.cpp:232-236); a CTA per row band
__global__ void deflate_kernel(double* __restrict__ a, int64_t rows, int64_t cols, const double* __restrict__ sigma,
                               const double* __restrict__ u, const double* __restrict__ v) {
    const double s = *sigma;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const double ur = __dmul_rn(s, u[r]);
        double* row = a + r * cols;
        for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) row[c] = __dsub_rn(row[c], __dmul_rn(ur, v[c]));
    }
}

// left[i][p] = float(u_{order[p]}[i]), right[p][c] = float(v_{order[p]}[c])  (lowrank.cpp:84-99)
__global__ void pack_triples_kernel(const double* __restrict__ us, const double* __restrict__ vs,
                                    const int32_t* __restrict__ order, int64_t rank, int64_t rows, int64_t cols,
                                    float* __restrict__ left, float* __restrict__ right) {
    const int64_t nl = rows * rank, n = nl + rank * cols;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (e < nl) {
            const int64_t i = e / rank, p = e % rank;
            left[e] = __double2float_rn(us[static_cast<int64_t>(order[p]) * rows + i]);
        } else {
            const int64_t f = e - nl, p = f / cols, c = f % cols;
            right[f] = __double2float_rn(vs[static_cast<int64_t>(order[p]) * cols + c]);
        }
    }
}

unsigned grid_for(int64_t n, int threads) {
    const int64_t b = (n + threads - 1) / threads;
    return static_cast<unsigned>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

cudaError_t launch_estimate_hessian(const float* x, int64_t tokens, int64_t dim, double damping, double* acc,
                                    double* lambda, float* h, cudaStream_t stream) {
    const unsigned nt = static_cast<unsigned>((dim + kT - 1) / kT);
    hessian_acc_kernel<<<dim3(nt, nt), kTT, 0, stream>>>(x, tokens, dim, acc);
    hessian_lambda_kernel<<<1, 32, 0, stream>>>(acc, tokens, dim, damping, lambda);
    hessian_fill_kernel<<<grid_for(dim * dim, 256), 256, 0, stream>>>(acc, tokens, dim, lambda, h);
    return cudaGetLastError();
}

size_t spd_status_bytes() { return sizeof(SpdStatus); }

// chol / linv: n x n f64 scratch each; status: spd_status_bytes() of device memory
cudaError_t launch_spd_inverse(const float* h, int64_t n, double* chol, double* linv, double* hinv, void* status,
                               cudaStream_t stream) {
    SpdStatus* st = static_cast<SpdStatus*>(status);
    cudaError_t e = cudaMemsetAsync(st, 0, sizeof(SpdStatus), stream);
    if (e != cudaSuccess) return e;
    chol_init_kernel<<<grid_for(n * n, 256), 256, 0, stream>>>(h, n, chol);
    const size_t rows_smem = sizeof(double) * (kT + kRowsPerCta) * (kT + 1);
    e = cudaFuncSetAttribute(chol_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(rows_smem));
    if (e != cudaSuccess) return e;
    for (int64_t j0 = 0; j0 < n; j0 += kT) {
        chol_diag_kernel<<<1, kT, 0, stream>>>(chol, n, j0, st);
        const int64_t below = n - j0 - kT;
        if (below > 0) {
            chol_rows_kernel<<<static_cast<unsigned>((below + kRowsPerCta - 1) / kRowsPerCta), kRowsPerCta, rows_smem,
                               stream>>>(chol, n, j0, st);
            const unsigned t = static_cast<unsigned>((below + kT - 1) / kT);
            chol_trail_kernel<<<dim3(t, t), kTT, 0, stream>>>(chol, n, j0, st);
        }
    }
    e = cudaMemsetAsync(linv, 0, sizeof(double) * n * n, stream);
    if (e != cudaSuccess) return e;
    for (int64_t i0 = 0; i0 < n; i0 += kT) {
        const int64_t cols = (n - i0 < kT ? n : i0 + kT);
        linv_block_kernel<<<static_cast<unsigned>((cols + kRowsPerCta - 1) / kRowsPerCta), kRowsPerCta, 0, stream>>>(
            chol, linv, n, i0, st);
        const int64_t below = n - i0 - kT;
        if (below > 0)
            linv_trail_kernel<<<dim3(static_cast<unsigned>((i0 + kT) / kT), static_cast<unsigned>((below + kT - 1) / kT)),
                                kTT, 0, stream>>>(chol, linv, n, i0, st);
    }
    const unsigned nt = static_cast<unsigned>((n + kT - 1) / kT);
    hinv_kernel<<<dim3(nt, nt), kTT, 0, stream>>>(linv, n, hinv, st);
    return cudaGetLastError();
}

void spd_status_read(const void* host_copy, int* failed, int64_t* column, double* pivot) {
    const SpdStatus* s = static_cast<const SpdStatus*>(host_copy);
    *failed = s->failed;
    *column = s->column;
    *pivot = s->pivot;
}

cudaError_t launch_make_grids(const float* r, int64_t rows, int64_t cols, int bits, int64_t gs, float* scales,
                              int32_t* zeros, cudaStream_t stream) {
    const int64_t n = rows * ((cols + gs - 1) / gs);
    grids_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(r, rows, cols, bits, gs, scales, zeros);
    return cudaGetLastError();
}

cudaError_t launch_rtn_codes(const float* r, int64_t rows, int64_t cols, int bits, int64_t gs, const float* scales,
                             const int32_t* zeros, uint8_t* codes, cudaStream_t stream) {
    rtn_codes_kernel<<<grid_for(rows * cols, 256), 256, 0, stream>>>(r, rows, cols, bits, gs, scales, zeros, codes);
    return cudaGetLastError();
}

namespace {
constexpr size_t kGptqSmemBudget = 220 * 1024;
size_t gptq_smem(int R, bool stage, int64_t dim, int64_t G) {
    return sizeof(double) * (R + (stage ? 2 : 0)) * dim + (sizeof(float) + sizeof(int32_t)) * R * G;
}
// (rows per CTA, staged Hinv rows) for this shape; R = 0 when even one row does not fit
void gptq_config(int64_t dim, int64_t gs, int* R, bool* stage) {
    const int64_t G = (dim + gs - 1) / gs;
    for (bool st : {true, false})
        for (int r : {4, 2, 1})
            if (gptq_smem(r, st, dim, G) <= kGptqSmemBudget) {
                *R = r;
                *stage = st;
                return;
            }
    *R = 0;
    *stage = false;
}
template <int kR, bool kStage>
cudaError_t launch_gptq_t(const float* r, int64_t rows, int64_t dim, int bits, int64_t gs, const float* scales,
                          const int32_t* zeros, const double* hinv, uint8_t* codes, cudaStream_t stream) {
    const size_t smem = gptq_smem(kR, kStage, dim, (dim + gs - 1) / gs);
    cudaError_t e = cudaFuncSetAttribute(gptq_kernel<kR, kStage>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    gptq_kernel<kR, kStage><<<static_cast<unsigned>((rows + kR - 1) / kR), kGptqThreads, smem, stream>>>(
        r, rows, dim, bits, gs, scales, zeros, hinv, codes);
    return cudaGetLastError();
}
}  // namespace

int gptq_rows_per_cta(int64_t dim, int64_t gs) {
    int R;
    bool st;
    gptq_config(dim, gs, &R, &st);
    return R;
}

cudaError_t launch_gptq(const float* r, int64_t rows, int64_t dim, int bits, int64_t gs, const float* scales,
                        const int32_t* zeros, const double* hinv, uint8_t* codes, cudaStream_t stream) {
    int R;
    bool st;
    gptq_config(dim, gs, &R, &st);
    if (R == 0) return cudaErrorInvalidValue;
    if (st) {
        if (R == 4) return launch_gptq_t<4, true>(r, rows, dim, bits, gs, scales, zeros, hinv, codes, stream);
        if (R == 2) return launch_gptq_t<2, true>(r, rows, dim, bits, gs, scales, zeros, hinv, codes, stream);
        return launch_gptq_t<1, true>(r, rows, dim, bits, gs, scales, zeros, hinv, codes, stream);
    }
    if (R == 4) return launch_gptq_t<4, false>(r, rows, dim, bits, gs, scales, zeros, hinv, codes, stream);
    if (R == 2) return launch_gptq_t<2, false>(r, rows, dim, bits, gs, scales, zeros, hinv, codes, stream);
    return launch_gptq_t<1, false>(r, rows, dim, bits, gs, scales, zeros, hinv, codes, stream);
}

// he_t: chunk_rows x dim f64 scratch; rowsum: rows f64; total: 1 f64 (device)
cudaError_t launch_proxy_loss(const float* orig, const uint8_t* codes, const float* scales, const int32_t* zeros,
                              int64_t rows, int64_t dim, int64_t gs, const float* h, int64_t chunk_rows, double* he_t,
                              double* rowsum, double* total, cudaStream_t stream) {
    for (int64_t r0 = 0; r0 < rows; r0 += chunk_rows) {
        const int64_t nr = rows - r0 < chunk_rows ? rows - r0 : chunk_rows;
        const dim3 grid(static_cast<unsigned>((dim + kT - 1) / kT), static_cast<unsigned>((nr + kT - 1) / kT));
        proxy_he_kernel<<<grid, kTT, 0, stream>>>(orig, codes, scales, zeros, rows, dim, gs, h, r0, nr, he_t);
        proxy_rowsum_kernel<<<static_cast<unsigned>((nr + 127) / 128), 128, 0, stream>>>(orig, codes, scales, zeros,
                                                                                          dim, gs, r0, nr, he_t,
                                                                                          rowsum);
    }
    proxy_total_kernel<<<1, 32, 0, stream>>>(rowsum, rows, total);
    return cudaGetLastError();
}


// sketch_lowrank building blocks
cudaError_t launch_widen(const float* w, int64_t n, double* out, cudaStream_t stream) {
    widen_kernel<<<grid_for(n, 256), 256, 0, stream>>>(w, n, out);
    return cudaGetLastError();
}
cudaError_t launch_matvec(const double* a, int64_t rows, int64_t cols, const double* x, double* y,
                          cudaStream_t stream) {
    const int64_t warps = (rows + 31) / 32;
    matvec_kernel<<<static_cast<unsigned>((warps + kMvWarps - 1) / kMvWarps), kMvWarps * 32, 0, stream>>>(a, rows,
                                                                                                           cols, x, y);
    return cudaGetLastError();
}
cudaError_t launch_mattvec(const double* a, int64_t rows, int64_t cols, const double* x, double* y,
                           cudaStream_t stream) {
    mattvec_kernel<<<static_cast<unsigned>((cols + 31) / 32), kMtvWarps * 32, 0, stream>>>(a, rows, cols, x, y);
    return cudaGetLastError();
}
cudaError_t launch_norm2(const double* v, int64_t n, double* out, cudaStream_t stream) {
    norm2_kernel<<<1, 32, 0, stream>>>(v, n, out);
    return cudaGetLastError();
}
cudaError_t launch_div_by(const double* src, int64_t n, const double* d, double* dst, cudaStream_t stream) {
    div_by_kernel<<<grid_for(n, 256), 256, 0, stream>>>(src, n, d, dst);
    return cudaGetLastError();
}
cudaError_t launch_deflate(double* a, int64_t rows, int64_t cols, const double* sigma, const double* u,
                           const double* v, cudaStream_t stream) {
    deflate_kernel<<<static_cast<unsigned>(rows < 148 * 16 ? rows : 148 * 16), 512, 0, stream>>>(a, rows, cols, sigma,
                                                                                               u, v);
    return cudaGetLastError();
}
cudaError_t launch_pack_triples(const double* us, const double* vs, const int32_t* order, int64_t rank, int64_t rows,
                                int64_t cols, float* left, float* right, cudaStream_t stream) {
    pack_triples_kernel<<<grid_for((rows + cols) * rank, 256), 256, 0, stream>>>(us, vs, order, rank, rows, cols,
                                                                                 left, right);
    return cudaGetLastError();
}

}  // namespace tqb
