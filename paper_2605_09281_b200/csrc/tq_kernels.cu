// sm_100a kernels of the fused low-rank MoE inference path.
//
//   route_kernel        route() (moe.cpp:43-89): FP64 gate scores with a
//                       certified-rounding fast path (bit-exact f32 scores),
//                       f64 softmax, top-k by (prob desc, index asc); also
//                       emits the fp16 activations and per-group sums.
//   plan_kernel         stable token permutation by expert
//                       and the device-built work-unit tables.
//   gemm_kernel         THE fused kernel: persistent, warp-specialised
//                       tcgen05 grouped GEMM.  TMA stages activation tiles
//                       and bulk-copies packed b-bit weight tiles into smem;
//                       8 dequant warps unpack codes in registers straight
//                       into the A operand in TMEM (tcgen05.st); one thread
//                       issues tcgen05.mma (A from TMEM, B = activations from
//                       smem, fp32 accumulator in TMEM); the rank-r low-rank
//                       correction (X.A).B_p and the zero-point correction
//                       ride in the SAME accumulator as extra K chunks; 4
//                       epilogue warps drain TMEM to global.
//   gather_kernel       permuted activation rows + extension rows.
//   combine_kernel      gate-weighted combine, t ascending then shared
//                       experts (reference_forward order, moe.cpp:115-132).
//   unpack_kernel       unpack_codes (codec.cpp:168-195) on the GPU.
//   export_codes_kernel inverse of the loader's repack (bit-exactness proof).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>

#include "tq_exp.h"
#include "tq_internal.h"
#include "tq_ptx.cuh"

namespace tqb {

// =============================================================================
// router: bit-exact route() (moe.cpp:43-89)
// =============================================================================

// Per token: scores[k] = float(sum_c double(x[c]) * double(G[k,c])) with the
// reference's sequential index-order f64 sum (matrix.cpp:25-36).  Every
// product is exact in f64, so ANY summation order of the i terms lands within
// gamma_{i-1} * sum|p| of the exact sum, as does the reference's sequential
// loop.  We sum in parallel and bound |ours - reference| <= 2 *
// gamma_{i+i/32+40} * sum|p|; when both ends of that interval round to the
// same f32, the f32 score is certified identical to the reference's,
// otherwise one warp replays the sequential loop (rare).  Then f64
// max-subtracted softmax, total summed k = 0..K-1, order by (prob desc, index
// asc), gates = float(prob / selected) -- moe.cpp:64-87 step by step.
//
// Grid (token, slice of 4 experts), 1024 threads: every thread issues all its
// gate loads up front (one memory round trip), the 4 (sum, sum|p|) pairs meet
// in shared memory in a fixed order; the last slice CTA of a token (atomic
// ticket) runs the softmax / top-k over the token's certified scores.
__device__ void plan_body(const PlanArgs& a, int32_t* pl_smem);

#ifndef TQ_ROUTE_THREADS
#define TQ_ROUTE_THREADS 512
#endif
constexpr int kRouteThreads = TQ_ROUTE_THREADS;
constexpr int kRouteWarps = kRouteThreads / 32;
#ifndef TQ_ROUTE_EXPERTS
#define TQ_ROUTE_EXPERTS 2   // measured: 2 beats 4 (decode 711 -> 698 us sweep, prefill 1520 -> 1458 us) and 1
#endif
constexpr int kRouteExperts = TQ_ROUTE_EXPERTS;   // experts per CTA
constexpr int kRouteCols = 4;         // columns per thread per pass (i <= 4096 in one pass)
constexpr int kReplayWin = 2048;      // products per replay window (16 KB of shared memory)

template <int kRT>
struct RouteSmem {
    double part[kRT / 32][kRouteExperts][2];
    double prod[kReplayWin];
    double replay_acc;
    unsigned und;
};

// Certified f32 scores of experts [k0, k0 + kRouteExperts) of one token
// (matrix.cpp:25-36 semantics, see the header comment): the whole CTA takes
// part; thread j < kRouteExperts writes score_row[k0 + j].  Returns the mask of
// scores that needed the exact replay (the caller fences those writes).
template <int kRT>
__device__ unsigned route_slice(const float* __restrict__ xb, int in_dim, const float* __restrict__ gate,
                                int num_experts, int k0, float* __restrict__ score_row, RouteSmem<kRT>& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();   // shared state of the previous token is consumed
    if (threadIdx.x == 0) {
        sm.und = 0u;
        sm.replay_acc = 0.0;
    }
    __syncthreads();
    // ---- tier 1: plain parallel dot products, loose bound ----------------
    // any summation order of the i exact products is within
    // gamma_{i-1} * sum|p| of the exact sum, as is the reference's sequential
    // loop: certify against 2 * gamma_{i+i/32+40} * sum|p| (fails for ~1e-3 of
    // the scores).  Tier 2 (below) only runs for a CTA with an undecided score.
    constexpr int kPass = kRT * 4;
    const bool vec = (in_dim & 3) == 0;
    auto load_pass = [&](int c0, float (&xv)[4], float (&gv)[kRouteExperts][4]) {
        const int cb = c0 + 4 * threadIdx.x;
        if (vec && cb + 3 < in_dim) {
            const float4 x4 = *reinterpret_cast<const float4*>(xb + cb);
            xv[0] = x4.x; xv[1] = x4.y; xv[2] = x4.z; xv[3] = x4.w;
#pragma unroll
            for (int j = 0; j < kRouteExperts; ++j) {
                float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k0 + j < num_experts) g4 = __ldg(reinterpret_cast<const float4*>(gate + static_cast<int64_t>(k0 + j) * in_dim + cb));
                gv[j][0] = g4.x; gv[j][1] = g4.y; gv[j][2] = g4.z; gv[j][3] = g4.w;
            }
        } else {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int c = cb + m;
                xv[m] = c < in_dim ? xb[c] : 0.0f;
#pragma unroll
                for (int j = 0; j < kRouteExperts; ++j)
                    gv[j][m] = (c < in_dim && k0 + j < num_experts) ? __ldg(gate + static_cast<int64_t>(k0 + j) * in_dim + c) : 0.0f;
            }
        }
    };
    {
        double sum1[kRouteExperts], abs1[kRouteExperts];
#pragma unroll
        for (int j = 0; j < kRouteExperts; ++j) sum1[j] = abs1[j] = 0.0;
        for (int c0 = 0; c0 < in_dim; c0 += kPass) {
            float xv[4], gv[kRouteExperts][4];
            load_pass(c0, xv, gv);
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int j = 0; j < kRouteExperts; ++j) {
                    const double pr = static_cast<double>(xv[m]) * static_cast<double>(gv[j][m]);
                    sum1[j] += pr;
                    abs1[j] += fabs(pr);
                }
        }
#pragma unroll
        for (int j = 0; j < kRouteExperts; ++j) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                sum1[j] += __shfl_xor_sync(0xffffffffu, sum1[j], off);
                abs1[j] += __shfl_xor_sync(0xffffffffu, abs1[j], off);
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < kRouteExperts; ++j) {
                sm.part[warp][j][0] = sum1[j];
                sm.part[warp][j][1] = abs1[j];
            }
        }
        __syncthreads();
        if (threadIdx.x < kRouteExperts && k0 + static_cast<int>(threadIdx.x) < num_experts) {
            const int j = threadIdx.x;
            double sv = 0.0, av = 0.0;
            for (int w = 0; w < (kRT / 32); ++w) {
                sv += sm.part[w][j][0];
                av += sm.part[w][j][1];
            }
            const double u = 1.1102230246251565e-16;  // 2^-53
            const double nterms = 2.0 * (static_cast<double>(in_dim) + static_cast<double>(in_dim) / 32.0 + 40.0);
            const double err = __dmul_ru(__dmul_ru(nterms * u, 1.01), __dmul_ru(av, 1.0001));
            const float lo = __double2float_rn(__dsub_rd(sv, err));
            const float hi = __double2float_rn(__dadd_ru(sv, err));
            score_row[k0 + j] = __double2float_rn(sv);
            if (lo != hi) atomicOr(&sm.und, 1u << j);
        }
        __syncthreads();
    }
    // every thread takes its copy of the undecided mask BEFORE thread 0 clears it for
    // tier 2 (reading sm.und in the condition itself raced with that clear: a late
    // thread saw 0, skipped tier 2 and its barriers, and the CTA's barrier phases
    // fell apart -- the intermittent decode-router fault)
    const unsigned und1 = sm.und;
    __syncthreads();
    if (und1 != 0u) {   // block-uniform
    if (threadIdx.x == 0) sm.und = 0u;
    __syncthreads();
    // ---- tier 2: the partial sums of the reference's order ----
    // Thread t owns columns [4t, 4t+4) of each pass, so thread order is index
    // order: a block scan gives every partial sum S_k of the reference's
    // sequential loop, whose rounding error is bounded by u * sum_k |S_k|
    // (first order) -- far tighter than gamma_n * sum|p| when the partial sums
    // stay small.  Tier 3 (exact sequential replay) is then very rare.
    double tot_s[kRouteExperts], abs_s[kRouteExperts], abs_p[kRouteExperts];
#pragma unroll
    for (int j = 0; j < kRouteExperts; ++j) tot_s[j] = abs_s[j] = abs_p[j] = 0.0;
    for (int c0 = 0; c0 < in_dim; c0 += kPass) {
        float xv[4], gv[kRouteExperts][4];
        load_pass(c0, xv, gv);
        // exact products, in-thread inclusive prefix
        double pre[kRouteExperts][4];
#pragma unroll
        for (int j = 0; j < kRouteExperts; ++j) {
            double run = 0.0;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const double pr = static_cast<double>(xv[m]) * static_cast<double>(gv[j][m]);
                abs_p[j] += fabs(pr);
                run += pr;
                pre[j][m] = run;
            }
        }
        // block exclusive scan of the thread totals (thread order = column order)
        double incl[kRouteExperts];
#pragma unroll
        for (int j = 0; j < kRouteExperts; ++j) {
            double v = pre[j][3];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const double o = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += o;
            }
            incl[j] = v;
            if (lane == 31) sm.part[warp][j][0] = v;
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll
            for (int j = 0; j < kRouteExperts; ++j) {
                double v = lane < (kRT / 32) ? sm.part[lane][j][0] : 0.0;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const double o = __shfl_up_sync(0xffffffffu, v, off);
                    if (lane >= off) v += o;
                }
                if (lane < (kRT / 32)) sm.part[lane][j][1] = v;   // inclusive scan of the warp totals
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kRouteExperts; ++j) {
            const double base = tot_s[j] + (warp > 0 ? sm.part[warp - 1][j][1] : 0.0) + (incl[j] - pre[j][3]);
#pragma unroll
            for (int m = 0; m < 4; ++m) abs_s[j] += fabs(base + pre[j][m]);
            tot_s[j] += sm.part[(kRT / 32) - 1][j][1];
        }
        __syncthreads();   // sm.part[] is reused by the next pass / the reduction below
    }
    // block sums of sum_k |S_k| and sum |p|; the total is the scan's last value
#pragma unroll
    for (int j = 0; j < kRouteExperts; ++j) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            abs_s[j] += __shfl_xor_sync(0xffffffffu, abs_s[j], off);
            abs_p[j] += __shfl_xor_sync(0xffffffffu, abs_p[j], off);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < kRouteExperts; ++j) {
            sm.part[warp][j][0] = abs_s[j];
            sm.part[warp][j][1] = abs_p[j];
        }
    }
    __syncthreads();
    // ---- certification (thread j: expert k0 + j) ----
    if (threadIdx.x < kRouteExperts && k0 + static_cast<int>(threadIdx.x) < num_experts) {
        const int j = threadIdx.x;
        double as = 0.0, ap = 0.0;
        for (int w = 0; w < (kRT / 32); ++w) {
            as += sm.part[w][j][0];
            ap += sm.part[w][j][1];
        }
        const double sv = tot_s[j];
        const double u = 1.1102230246251565e-16;  // 2^-53
        const double n = static_cast<double>(in_dim);
        // reference: |seq - exact| <= u * sum|S_k| (+ second order); ours: <= 24 u sum|p|
        // (each partial sum passes <= 4 + 5 + 5 + 2 additions per pass); the partial sums
        // we used carry the same ours-error, n times: + n * 24 u^2 sum|p|
        const double err_ref = __dmul_ru(__dmul_ru(u, 1.02), __dadd_ru(as, __dmul_ru(n * 48.0 * u, ap)));
        const double err_our = __dmul_ru(__dmul_ru(24.0 * u * (1.0 + n / 4096.0), 1.02), ap);
        const double err = __dadd_ru(err_ref, err_our);
        const float lo = __double2float_rn(__dsub_rd(sv, err));
        const float hi = __double2float_rn(__dadd_ru(sv, err));
        score_row[k0 + j] = __double2float_rn(sv);
        if (lo != hi) atomicOr(&sm.und, 1u << j);
    }
    __syncthreads();
    }   // tier 2
    // replay: the reference's exact sequential loop (matrix.cpp:29-34).  The
    // CTA forms the (exact) products in shared memory, then one thread adds
    // them in index order -- a dependent f64 chain, loads hoisted ahead
    const unsigned und = sm.und;
    for (int j = 0; j < kRouteExperts; ++j) {
        if (!(und & (1u << j))) continue;
        const float* gk = gate + static_cast<int64_t>(k0 + j) * in_dim;
        for (int c0 = 0; c0 < in_dim; c0 += kReplayWin) {
            const int n = min(kReplayWin, in_dim - c0);
            __syncthreads();
            for (int q = threadIdx.x; q < n; q += kRT)
                sm.prod[q] = static_cast<double>(xb[c0 + q]) * static_cast<double>(gk[c0 + q]);
            __syncthreads();
            if (threadIdx.x == 0) {
                double acc = sm.replay_acc;
                int q = 0;
                for (; q + 8 <= n; q += 8) {
                    double v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) v[t] = sm.prod[q + t];
#pragma unroll
                    for (int t = 0; t < 8; ++t) acc = __dadd_rn(acc, v[t]);
                }
                for (; q < n; ++q) acc = __dadd_rn(acc, sm.prod[q]);
                sm.replay_acc = c0 + n < in_dim ? acc : 0.0;
                if (c0 + n >= in_dim) score_row[k0 + j] = __double2float_rn(acc);
            }
        }
    }
    return und;
}

// Softmax and top-k of one token's certified scores (moe.cpp:64-87), run by
// ONE warp: mx, prob_k = exp(s_k - mx) in f64 (glibc's exp, tq_exp.h), total
// summed k = 0..K-1, order by (prob desc, index asc), gate = float(prob / selected).
__device__ void route_pick(const float* score_row, int num_experts, int top_k, float* sc, double* ex, int* pick_k,
                           double* pick_p, int32_t* __restrict__ ids_row, float* __restrict__ gates_row,
                           bool fence = true) {
    const int lane = threadIdx.x & 31;
    if (fence) __threadfence();   // (callers that acquired through their ticket pass false)
    for (int k = lane; k < num_experts; k += 32) sc[k] = __ldcg(score_row + k);
    __syncwarp();
    double mx = -INFINITY;
    for (int k = lane; k < num_experts; k += 32) mx = fmax(mx, static_cast<double>(sc[k]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    for (int k = lane; k < num_experts; k += 32) ex[k] = tq_exp::exp(__dsub_rn(static_cast<double>(sc[k]), mx));
    __syncwarp();
    double total = 0.0;   // in the reference order k = 0..K-1
    for (int k = 0; k < num_experts; ++k) total = __dadd_rn(total, ex[k]);
    // prob_k = exp(s_k - mx) / total, formed once (lane owns k = lane, lane + 32)
    const double p0 = lane < num_experts ? __ddiv_rn(ex[lane], total) : -1.0;
    const double p1 = lane + 32 < num_experts ? __ddiv_rn(ex[lane + 32], total) : -1.0;
    double selected = 0.0;
    uint64_t taken = 0;
    for (int tt = 0; tt < top_k; ++tt) {
        double best_p = -1.0;
        int best_k = 0x7fffffff;
        for (int h = 0; h < 2; ++h) {
            const int k = lane + 32 * h;
            if (k >= num_experts || (taken & (1ull << k))) continue;
            const double pk = h ? p1 : p0;
            if (pk > best_p || (pk == best_p && k < best_k)) {
                best_p = pk;
                best_k = k;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double op = __shfl_xor_sync(0xffffffffu, best_p, off);
            const int ok = __shfl_xor_sync(0xffffffffu, best_k, off);
            if (op > best_p || (op == best_p && ok < best_k)) {
                best_p = op;
                best_k = ok;
            }
        }
        taken |= 1ull << best_k;
        if (lane == 0) {
            pick_k[tt] = best_k;
            pick_p[tt] = best_p;
        }
        selected = __dadd_rn(selected, best_p);
    }
    __syncwarp();
    for (int tt = lane; tt < top_k; tt += 32) {
        ids_row[tt] = pick_k[tt];
        gates_row[tt] = __double2float_rn(__ddiv_rn(pick_p[tt], selected));
    }
}

template <int kRT>
__global__ void __launch_bounds__(kRT) route_kernel(const float* __restrict__ x, int batch, int in_dim,
                                                             const float* __restrict__ gate, int num_experts,
                                                             int top_k, int group_size, int groups, int k_pad,
                                                             int32_t* __restrict__ ids, float* __restrict__ gates,
                                                             __half* __restrict__ x16, float* __restrict__ sx,
                                                             float* __restrict__ score_ws, int32_t* __restrict__ ticket,
                                                             int tokens_per_cta) {
    __shared__ RouteSmem<kRT> sm;
    __shared__ float sc[64];
    __shared__ double ex[64];
    __shared__ int pick_k[64];
    __shared__ double pick_p[64];
    __shared__ int s_last;
    pdl_wait();
    pdl_launch_dependents();
    const int k0 = blockIdx.y * kRouteExperts;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // prefill: several tokens per CTA, the CTA's gate slice is re-read from L1
    for (int tb = 0; tb < tokens_per_cta; ++tb) {
    const int b = blockIdx.x * tokens_per_cta + tb;
    if (b >= batch) break;
    const float* xb = x + static_cast<int64_t>(b) * in_dim;
    if (blockIdx.y == 0) {
        // fp16 activations (zero-padded to k_pad) and per-group sums of them
        if (x16) {
            __half* xo = x16 + static_cast<int64_t>(b) * k_pad;
            for (int c = threadIdx.x; c < k_pad; c += kRT) xo[c] = __float2half_rn(c < in_dim ? xb[c] : 0.0f);
        }
        for (int g = warp; sx && g < groups; g += (kRT / 32)) {
            float acc = 0.0f;
            const int c0 = g * group_size, c1 = min(in_dim, c0 + group_size);
            for (int c = c0 + lane; c < c1; c += 32) acc += __half2float(__float2half_rn(xb[c]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
            if (lane == 0) sx[static_cast<int64_t>(b) * groups + g] = acc;
        }
    }
    if (num_experts == 0) continue;  // activations-only prep (tq_forward with given routing)
    const unsigned und = route_slice<kRT>(xb, in_dim, gate, num_experts, k0, score_ws + static_cast<int64_t>(b) * num_experts, sm);
    // ---- the last slice CTA of token b finishes the routing ----
    if (threadIdx.x < kRouteExperts || (threadIdx.x == 0 && und)) __threadfence();   // score_ws writers
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int done = atomicAdd(&ticket[b], 1);
        s_last = done == static_cast<int>(gridDim.y) - 1;
        if (s_last) ticket[b] = 0;   // ready for the next launch
    }
    __syncthreads();
    if (s_last && warp == 0) {
    route_pick(score_ws + static_cast<int64_t>(b) * num_experts, num_experts, top_k, sc, ex, pick_k, pick_p,
               ids + static_cast<int64_t>(b) * top_k, gates + static_cast<int64_t>(b) * top_k);
    }   // last slice CTA of token b
    }   // tokens of this CTA
}

// =============================================================================
// route, prefill: token tiles x all experts (a skinny f64 GEMM)
// =============================================================================
// Same contract and certification as route_kernel, organised for large
// batches: a CTA owns kTT tokens and ALL experts, stages 128-column chunks of
// x and G in shared memory as f64 (each gate chunk read once per kTT tokens,
// each x element converted once), and every thread accumulates a 2-token x
// 4-expert micro-tile over a strided column subset (DFMA for the sum, DFMA on
// |x|,|g| for sum|p|).  The partial sums of the S column splits meet in
// shared memory; a score whose any-order interval straddles an f32 rounding
// boundary is replayed with the reference's sequential loop (matrix.cpp:29-34)
// by one warp; then one warp per token runs the softmax / top-k of
// moe.cpp:64-87.  Also writes the fp16 activations and group sums (identical
// arithmetic to route_kernel).
#ifndef TQ_ROUTE_TT
#define TQ_ROUTE_TT 16
#endif
constexpr int kTT = TQ_ROUTE_TT;   // tokens per CTA
#ifndef TQ_ROUTE_TC
#define TQ_ROUTE_TC 256   // measured at 4096 tokens: 128 -> 143 us, 256 -> 137 us
#endif
constexpr int kTC = TQ_ROUTE_TC;   // columns per staged chunk
constexpr int kTStride = kTC + 4;   // padded f32 row stride (16-byte rows; row r shifts banks by 4r)
constexpr int kTThreads = 256;

__host__ __device__ inline int route_tile_smem(int num_experts) {
    const int ke = (num_experts + 3) & ~3;
    const int tiles = 2 * (kTT + ke) * kTStride * 4;   // two f32 stages of [x rows | G rows]
    const int red = kTThreads * 16 * 8;                // split-reduction buffer (f64)
    return tiles > red ? tiles : red;
}

static __device__ __forceinline__ uint32_t bits_of(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
static __device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// one chunk of a thread's 2-token x 4-expert micro-tile: columns s, s+S, ...
// (S compile-time, so the unrolled loads are hoisted ahead of the f64 chains)
template <int S>
__device__ __forceinline__ void route_tile_mac(const float* __restrict__ xa, const float* __restrict__ ga, int s,
                                              double (&sum)[8], float (&asum)[8]) {
#pragma unroll 8
    for (int c = s; c < kTC; c += S) {
        const float xf0 = xa[c], xf1 = xa[kTStride + c];
        const float gf0 = ga[c], gf1 = ga[kTStride + c], gf2 = ga[2 * kTStride + c], gf3 = ga[3 * kTStride + c];
        const double x0 = xf0, x1 = xf1, g0 = gf0, g1 = gf1, g2 = gf2, g3 = gf3;
        sum[0] = fma(x0, g0, sum[0]); asum[0] = fmaf(fabsf(xf0), fabsf(gf0), asum[0]);
        sum[1] = fma(x0, g1, sum[1]); asum[1] = fmaf(fabsf(xf0), fabsf(gf1), asum[1]);
        sum[2] = fma(x0, g2, sum[2]); asum[2] = fmaf(fabsf(xf0), fabsf(gf2), asum[2]);
        sum[3] = fma(x0, g3, sum[3]); asum[3] = fmaf(fabsf(xf0), fabsf(gf3), asum[3]);
        sum[4] = fma(x1, g0, sum[4]); asum[4] = fmaf(fabsf(xf1), fabsf(gf0), asum[4]);
        sum[5] = fma(x1, g1, sum[5]); asum[5] = fmaf(fabsf(xf1), fabsf(gf1), asum[5]);
        sum[6] = fma(x1, g2, sum[6]); asum[6] = fmaf(fabsf(xf1), fabsf(gf2), asum[6]);
        sum[7] = fma(x1, g3, sum[7]); asum[7] = fmaf(fabsf(xf1), fabsf(gf3), asum[7]);
    }
}

__global__ void __launch_bounds__(kTThreads, 2) route_tile_kernel(const float* __restrict__ x, int batch, int in_dim,
                                                               const float* __restrict__ gate, int num_experts,
                                                               int top_k, int group_size, int groups, int k_pad,
                                                               int32_t* __restrict__ ids, float* __restrict__ gates,
                                                               __half* __restrict__ x16, float* __restrict__ sx) {
    extern __shared__ double tsm[];
    __shared__ float sc[kTT][64];
    __shared__ double ex[kTThreads / 32][64];
    __shared__ int pick_k[kTThreads / 32][64];
    __shared__ double pick_p[kTThreads / 32][64];
    __shared__ int und[kTT * 64];
    __shared__ double und_sv[kTT * 64], und_ap[kTT * 64];
    __shared__ int n_und;
    pdl_wait();
    pdl_launch_dependents();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b0 = blockIdx.x * kTT;
    const int ke = (num_experts + 3) & ~3;
    const int ke4 = ke >> 2;
    const int mt_n = (kTT / 2) * ke4;   // micro-tiles
    int S = 32;
    while (S > 1 && mt_n * S > kTThreads) S >>= 1;
    float* stage0 = reinterpret_cast<float*>(tsm);
    const int stage_floats = (kTT + ke) * kTStride;   // [x rows kTT][G rows ke]
    const int t = threadIdx.x;
    const bool active = t < mt_n * S;
    const int mt = t / S, s = t % S;
    // micro-tile order: experts fastest when a warp holds <= 2 micro-tiles (its
    // two halves then read one x row, broadcast), token pairs fastest otherwise
    // (a warp's gate rows would all land in the same banks)
    const bool e_fast = S >= 16;
    const int tp = e_fast ? mt / ke4 : mt % (kTT / 2), eg = e_fast ? mt % ke4 : mt / (kTT / 2);
    // sum: f64 (each product exact, one rounding per add); sum|p|: an f32 upper
    // bound (only the certification interval uses it; scaled by its own error below)
    double sum[8];
    float asum[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        sum[k] = 0.0;
        asum[k] = 0.0f;
    }
    if (threadIdx.x == 0) n_und = 0;
    const int c_end = in_dim > k_pad ? in_dim : k_pad;
    const int n_chunks = (c_end + kTC - 1) / kTC;
    // chunk -> stage: coalesced 16-byte cp.async (in_dim % 4 == 0: a 4-column
    // piece is wholly in or out of range; zeros written directly outside)
    auto issue = [&](int ch) {
        float* st = stage0 + (ch & 1) * stage_floats;
        const uint32_t sa = smem_u32(st);
        const int c0 = ch * kTC;
        for (int i = threadIdx.x; i < (kTT + ke) * (kTC / 4); i += kTThreads) {
            const int r = i / (kTC / 4), cc = (i % (kTC / 4)) * 4, c = c0 + cc;
            const float* src = nullptr;
            if (r < kTT) {
                if (b0 + r < batch && c < in_dim) src = x + static_cast<int64_t>(b0 + r) * in_dim + c;
            } else if (r - kTT < num_experts && c < in_dim) {
                src = gate + static_cast<int64_t>(r - kTT) * in_dim + c;
            }
            if (src) cp_async_16(sa + 4u * static_cast<uint32_t>(r * kTStride + cc), src);
            else *reinterpret_cast<float4*>(st + r * kTStride + cc) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        cp_async_commit();
    };
    issue(0);
    for (int ch = 0; ch < n_chunks; ++ch) {
        if (ch + 1 < n_chunks) {
            issue(ch + 1);
            cp_async_wait_group1();   // chunk ch landed (ch + 1 in flight)
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        const int c0 = ch * kTC;
        const float* xs = stage0 + (ch & 1) * stage_floats;
        const float* gs = xs + kTT * kTStride;
        // fp16 activations (zero-padded to k_pad)
#ifndef TQ_RT_ABL
#define TQ_RT_ABL 0
#endif
        if (x16 && !(TQ_RT_ABL & 2)) {
            // 4 halves per thread per pass (k_pad % 4 == 0: a piece is wholly in or out)
            for (int i = threadIdx.x; i < kTT * (kTC / 4); i += kTThreads) {
                const int r = i / (kTC / 4), cc = (i % (kTC / 4)) * 4, c = c0 + cc;
                if (b0 + r < batch && c < k_pad) {
                    const float4 v = *reinterpret_cast<const float4*>(xs + r * kTStride + cc);
                    uint2 h;
                    h.x = bits_of(__halves2half2(__float2half_rn(v.x), __float2half_rn(v.y)));
                    h.y = bits_of(__halves2half2(__float2half_rn(v.z), __float2half_rn(v.w)));
                    *reinterpret_cast<uint2*>(x16 + static_cast<int64_t>(b0 + r) * k_pad + c) = h;
                }
            }
        }
        // group sums of the fp16 activations (route_kernel's exact arithmetic);
        // the launcher guarantees kTC % group_size == 0
        if (sx && c0 < in_dim && !(TQ_RT_ABL & 2)) {
            // kTC % group_size == 0 makes group_size and gpc powers of two: shifts
            const int lgs = __ffs(group_size) - 1;
            const int lgpc = __ffs(kTC >> lgs) - 1;
            // four (token, group) pairs per warp in flight (independent chains; each
            // pair's summation order is route_kernel's)
            constexpr int kP = 4;
            const int n_pairs = kTT << lgpc;
            for (int p0 = warp * kP; p0 < n_pairs; p0 += (kTThreads / 32) * kP) {
                float acc[kP];
                int cab[kP], cbb[kP];
#pragma unroll
                for (int j = 0; j < kP; ++j) {
                    const int pi = p0 + j;
                    const int r = pi >> lgpc, gl = pi & ((1 << lgpc) - 1);
                    const int g = (c0 >> lgs) + gl;
                    const bool ok = pi < n_pairs && b0 + r < batch && g < groups;
                    cab[j] = ok ? g * group_size : 0;
                    cbb[j] = ok ? min(in_dim, cab[j] + group_size) : 0;
                    acc[j] = 0.0f;
                }
                for (int k = lane; k < group_size; k += 32) {
#pragma unroll
                    for (int j = 0; j < kP; ++j) {
                        const int c = cab[j] + k;
                        const int r = (p0 + j) >> lgpc;
                        if (c < cbb[j]) acc[j] += __half2float(__float2half_rn(xs[r * kTStride + (c - c0)]));
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                    for (int j = 0; j < kP; ++j) acc[j] += __shfl_down_sync(0xffffffffu, acc[j], off);
                if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < kP; ++j)
                        if (cbb[j] > cab[j]) {   // a valid pair (g < groups: its range is non-empty)
                            const int pi = p0 + j;
                            sx[static_cast<int64_t>(b0 + (pi >> lgpc)) * groups + (c0 >> lgs) + (pi & ((1 << lgpc) - 1))] = acc[j];
                        }
                }
            }
        }
        if (active && c0 < in_dim && !(TQ_RT_ABL & 1)) {
            const float* xa = xs + (2 * tp) * kTStride;
            const float* ga = gs + (4 * eg) * kTStride;
            switch (S) {
                case 32: route_tile_mac<32>(xa, ga, s, sum, asum); break;
                case 16: route_tile_mac<16>(xa, ga, s, sum, asum); break;
                case 8: route_tile_mac<8>(xa, ga, s, sum, asum); break;
                case 4: route_tile_mac<4>(xa, ga, s, sum, asum); break;
                case 2: route_tile_mac<2>(xa, ga, s, sum, asum); break;
                default: route_tile_mac<1>(xa, ga, s, sum, asum); break;
            }
        }
        __syncthreads();   // stage (ch & 1) consumed before chunk ch + 2 is issued into it
    }
    __syncthreads();   // tiles consumed: the region becomes the split-reduction buffer
    double* red = tsm;   // [kTThreads][16]
    if (active) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            red[t * 16 + k] = sum[k];
            red[t * 16 + 8 + k] = asum[k];
        }
    }
    __syncthreads();
    // certification per (token, expert): tier 1 of route_kernel.  Our path
    // depth is <= n/S + S + 1 additions, inside the n + n/32 + 40 of the bound.
    for (int pr = threadIdx.x; pr < kTT * num_experts; pr += kTThreads) {
        const int r = pr / num_experts, e = pr % num_experts;
        if (b0 + r >= batch) continue;
        const int m = e_fast ? (r >> 1) * ke4 + (e >> 2) : (e >> 2) * (kTT / 2) + (r >> 1);
        const int k = (r & 1) * 4 + (e & 3);
        double sv = 0.0, av = 0.0;
        for (int q = 0; q < S; ++q) {
            sv += red[(m * S + q) * 16 + k];
            av += red[(m * S + q) * 16 + 8 + k];
        }
        const double u = 1.1102230246251565e-16;  // 2^-53
        const double nterms = 2.0 * (static_cast<double>(in_dim) + static_cast<double>(in_dim) / 32.0 + 40.0);
        // av: f32 sums of f32-rounded |x||g| (depth <= n/S + 1 each, then exact-ish f64
        // adds): exact sum|p| <= av * (1 + (n/S + 2) 2^-23) + n 2^-126 (subnormal products)
        const double avb = __dadd_ru(__dmul_ru(av, 1.0 + (static_cast<double>(in_dim) / S + 2.0) * 1.2e-7 + 1e-12),
                                     static_cast<double>(in_dim) * 1.1754943508222875e-38);
        const double err = __dmul_ru(__dmul_ru(nterms * u, 1.01), __dmul_ru(avb, 1.0001));
        const float lo = __double2float_rn(__dsub_rd(sv, err));
        const float hi = __double2float_rn(__dadd_ru(sv, err));
        sc[r][e] = __double2float_rn(sv);
        if (lo != hi) {
            const int slot = atomicAdd(&n_und, 1);
            und[slot] = pr;
            und_sv[slot] = sv;
            und_ap[slot] = avb;
        }
    }
    __syncthreads();
    // undecided scores.  Tier 2: bound the reference's own rounding by its
    // partial sums, |seq - exact| <= u * sum_k |S_k| (+ second order), far
    // tighter than the any-order bound when the partial sums stay small
    // (random-walk data: ~sqrt(n) x).  Still undecided: tier 3, the reference's
    // sequential loop.  (Measured at 4096 tokens: tier 2 per warp 141 us, per
    // CTA 123 us; 0.7% of the c3 scores fail tier 1.)
    // tier 2, the whole CTA on one undecided score at a time: thread t scans the
    // contiguous columns [t*seg, (t+1)*seg) (all its loads in flight at once),
    // a block scan of the segment totals gives every partial sum of the
    // reference's order; still undecided scores go to the tier-3 list
    __shared__ double t2_part[kTThreads / 32][2];
    __shared__ int n_t3;
    __shared__ int t3[kTT * 64];
    if (threadIdx.x == 0) n_t3 = 0;
    // the tier-3 count must be cleared for every warp before any reads it: with no
    // tier-2 score the loop below has no barrier, and a warp reading a stale n_t3
    // walked a stale t3[] list into wild addresses (the token-tile router's
    // intermittent illegal address)
    __syncthreads();
    const int n_t2 = (TQ_RT_ABL & 4) ? 0 : n_und;
    for (int i = 0; i < n_t2; ++i) {
        const int pr = und[i];
        const int r = pr / num_experts, e = pr % num_experts;
        const float* xb = x + static_cast<int64_t>(b0 + r) * in_dim;
        const float* gk = gate + static_cast<int64_t>(e) * in_dim;
        const int seg = (in_dim + kTThreads - 1) / kTThreads;
        const int ca = min(in_dim, static_cast<int>(threadIdx.x) * seg), cb = min(in_dim, ca + seg);
        double run = 0.0;
#pragma unroll 8
        for (int c = ca; c < cb; ++c) run = fma(static_cast<double>(xb[c]), static_cast<double>(gk[c]), run);
        double inc = run;   // block inclusive scan of the segment totals
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        if (lane == 31) t2_part[warp][0] = inc;
        __syncthreads();
        double woff = 0.0;
        for (int w = 0; w < warp; ++w) woff += t2_part[w][0];
        double as = 0.0;
        run = woff + (inc - run);   // exclusive offset of this segment
#pragma unroll 8
        for (int c = ca; c < cb; ++c) {
            run = fma(static_cast<double>(xb[c]), static_cast<double>(gk[c]), run);
            as += fabs(run);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) as += __shfl_xor_sync(0xffffffffu, as, d);
        if (lane == 0) t2_part[warp][1] = as;
        __syncthreads();
        if (threadIdx.x == 0) {
            double ast = 0.0;
            for (int w = 0; w < kTThreads / 32; ++w) ast += t2_part[w][1];
            const double u = 1.1102230246251565e-16;   // 2^-53
            const double n = static_cast<double>(in_dim);
            const double ap = und_ap[i];
            // our partial sums: depth <= seg + 5 (warp scan) + 8 (warp offsets) + 2,
            // so sum|S_k| <= ast (1 + (n + 40) u) + n (seg + 16) u ap
            const double sum_s = __dadd_ru(__dmul_ru(ast, 1.0 + 1.01 * (n + 40.0) * u),
                                           __dmul_ru(__dmul_ru(n, (seg + 16.0) * u * 1.01), ap));
            // reference: u * sum|S^ref_k| <= u (sum|S_k| + n * gamma_n * ap); ours: the
            // tile's any-order depth n/S + S + 2
            const double err_ref = __dmul_ru(u * 1.01, __dadd_ru(sum_s, __dmul_ru(n * n * u * 1.01, ap)));
            const double err_our = __dmul_ru((n / S + S + 2.0) * u * 1.01, ap);
            const double err = __dmul_ru(__dadd_ru(err_ref, err_our), 1.05);
            const double sv = und_sv[i];
            const float lo = __double2float_rn(__dsub_rd(sv, err));
            const float hi = __double2float_rn(__dadd_ru(sv, err));
            if (lo != hi) t3[n_t3++] = pr;   // certified otherwise: sc already holds float(sv)
        }
        __syncthreads();   // t2_part reused by the next score
    }
    // tier 3: the reference's sequential loop, one warp per still-undecided score
    // (products in a warp-private window, one lane adds them in index order)
    double* win = tsm + warp * 256;   // the reduction buffer is consumed
    for (int i = warp; i < n_t3; i += kTThreads / 32) {
        const int pr = t3[i];
        const int r = pr / num_experts, e = pr % num_experts;
        const float* xb = x + static_cast<int64_t>(b0 + r) * in_dim;
        const float* gk = gate + static_cast<int64_t>(e) * in_dim;
        double acc = 0.0;
        for (int c0 = 0; c0 < in_dim; c0 += 256) {
            const int n = min(256, in_dim - c0);
            __syncwarp();
            for (int q = lane; q < n; q += 32) win[q] = static_cast<double>(xb[c0 + q]) * static_cast<double>(gk[c0 + q]);
            __syncwarp();
            if (lane == 0) {
                int q = 0;
                for (; q + 8 <= n; q += 8) {
                    double v[8];
#pragma unroll
                    for (int tt = 0; tt < 8; ++tt) v[tt] = win[q + tt];
#pragma unroll
                    for (int tt = 0; tt < 8; ++tt) acc = __dadd_rn(acc, v[tt]);
                }
                for (; q < n; ++q) acc = __dadd_rn(acc, win[q]);
            }
        }
        if (lane == 0) sc[r][e] = __double2float_rn(acc);
    }
    __syncthreads();
    // softmax (f64, max-subtracted, total in k order) and top-k -- moe.cpp:64-87
    for (int r = warp; r < kTT; r += kTThreads / 32) {
        const int b = b0 + r;
        if (b >= batch) break;
        double mx = -INFINITY;
        for (int k = lane; k < num_experts; k += 32) mx = fmax(mx, static_cast<double>(sc[r][k]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        for (int k = lane; k < num_experts; k += 32)
            ex[warp][k] = tq_exp::exp(__dsub_rn(static_cast<double>(sc[r][k]), mx));
        __syncwarp();
        double total = 0.0;   // in the reference order k = 0..K-1
        for (int k = 0; k < num_experts; ++k) total = __dadd_rn(total, ex[warp][k]);
        double selected = 0.0;
        uint64_t taken = 0;
        for (int tt = 0; tt < top_k; ++tt) {
            double best_p = -1.0;
            int best_k = 0x7fffffff;
            for (int k = lane; k < num_experts; k += 32) {
                if (taken & (1ull << k)) continue;
                const double pk = __ddiv_rn(ex[warp][k], total);
                if (pk > best_p || (pk == best_p && k < best_k)) {
                    best_p = pk;
                    best_k = k;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double op = __shfl_xor_sync(0xffffffffu, best_p, off);
                const int ok = __shfl_xor_sync(0xffffffffu, best_k, off);
                if (op > best_p || (op == best_p && ok < best_k)) {
                    best_p = op;
                    best_k = ok;
                }
            }
            taken |= 1ull << best_k;
            if (lane == 0) {
                pick_k[warp][tt] = best_k;
                pick_p[warp][tt] = best_p;
            }
            selected = __dadd_rn(selected, best_p);
        }
        __syncwarp();
        for (int tt = lane; tt < top_k; tt += 32) {
            ids[static_cast<int64_t>(b) * top_k + tt] = pick_k[warp][tt];
            gates[static_cast<int64_t>(b) * top_k + tt] = __double2float_rn(__ddiv_rn(pick_p[warp][tt], selected));
        }
        __syncwarp();   // ex / pick of this warp are reused by its next token
    }
}

// =============================================================================
// plan: stable permutation + work-unit tables (single CTA)
// =============================================================================


#ifndef TQ_PLAN_THREADS
#define TQ_PLAN_THREADS 1024
#endif
constexpr int kPlanThreads = TQ_PLAN_THREADS;

// First main chunk of K split sp of ns over kc chunks when the last split also
// carries ext work worth e8/8 chunks: boundaries at round(sp * (kc + e8/8) / ns),
// capped so every split keeps >= 2 main chunks (each of the decode GEMM's two
// MMA issue streams sees a chunk of every unit; the host keeps ns <= kc / 2).
// e8 = 0: the uniform split.
__device__ __forceinline__ int split_bound(int sp, int ns, int kc, int e8) {
    if (sp >= ns) return kc;
    if (e8 <= 0 || kc < 2 * ns) return sp * kc / ns;
    const int b = (sp * (kc * 8 + e8) / ns + 4) / 8;
    return min(b, kc - 2 * (ns - sp));
}

// The plan on one CTA of any size (blockDim a multiple of 32, <= 1024 threads):
// run by plan_kernel, or fused into the router's globally-last CTA.
// pl_smem: (nwarps + 1) * K + 1 ints.
__device__ void plan_body(const PlanArgs& a, int32_t* pl_smem) {
    const int K = a.num_experts;
    const int nwarps = blockDim.x >> 5;
    int32_t* cnt = pl_smem;                // [nwarps][K]
    int32_t* tot = pl_smem + nwarps * K;   // [K+1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = a.batch * a.top_k;
    for (int t = threadIdx.x; t < nwarps * K; t += blockDim.x) cnt[t] = 0;
    __syncthreads();
    const int per = (n + nwarps - 1) / nwarps;
    const int f0 = warp * per, f1 = min(n, f0 + per);
    // phase 1: per-warp counts (warp-private rows, no atomics)
    for (int base = f0; base < f1; base += 32) {
        const int f = base + lane;
        const bool act = f < f1;
        int id = act ? __ldcg(a.ids + f) : -1;
        if (act && (id < 0 || id >= K)) {
            atomicExch(a.err_flag, 1);
            id = -1;
        }
        const unsigned m = __match_any_sync(0xffffffffu, id);
        if (id >= 0 && lane == __ffs(m) - 1) cnt[warp * K + id] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
    // phase 2: expert totals + exclusive offsets, per-warp bases
    if (threadIdx.x < K) {
        int s = 0;
        for (int w = 0; w < nwarps; ++w) s += cnt[w * K + threadIdx.x];
        tot[threadIdx.x] = s;
    }
    __syncthreads();
    __shared__ int32_t ptot[1025];   // expert row bases, each expert's rows padded to a multiple of 8
    if (threadIdx.x == 0) {
        int run = 0, prun = 0;
        for (int e = 0; e < K; ++e) {
            const int c = tot[e];
            tot[e] = run;
            ptot[e] = prun;
            run += c;
            prun += (c + 7) & ~7;
        }
        tot[K] = run;
        ptot[K] = prun;
    }
    __syncthreads();
    if (threadIdx.x <= K) {
        a.offsets[threadIdx.x] = tot[threadIdx.x];
        if (a.poffsets) a.poffsets[threadIdx.x] = ptot[threadIdx.x];
    }
    if (threadIdx.x < K) {
        int run = tot[threadIdx.x];
        for (int w = 0; w < nwarps; ++w) {
            const int c = cnt[w * K + threadIdx.x];
            cnt[w * K + threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
    // phase 3: stable scatter
    for (int base = f0; base < f1; base += 32) {
        const int f = base + lane;
        const bool act = f < f1;
        int id = act ? __ldcg(a.ids + f) : -1;
        if (id >= K || id < 0) {
            if (act) a.inv[f] = -1;
            id = -1;
        }
        const unsigned m = __match_any_sync(0xffffffffu, id);
        if (id >= 0) {
            const int rank = __popc(m & ((1u << lane) - 1u));
            const int pos = cnt[warp * K + id] + rank;
            a.perm[pos] = f;
            a.inv[f] = pos;
        }
        __syncwarp();
        if (id >= 0 && lane == __ffs(m) - 1) cnt[warp * K + id] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
    // ---- work units ----------------------------------------------------------
    // routed experts (e, mb, tile, split), then shared experts (s, mb, tile, split),
    // generated in parallel; the split count is chosen here from the actual
    // routing so the persistent grid is evenly loaded.
    __shared__ int32_t s_tiles[1025];
    __shared__ int32_t s_nsplit, s_ext8;
    const int n_slots = tot[K];
    const int bn = a.bn;
    const int n_local = a.e_end - a.e_begin;
    const int sh_tiles = (a.batch + bn - 1) / bn;
    for (int t = threadIdx.x; t < n_local; t += blockDim.x) {
        const int ne = tot[a.e_begin + t + 1] - tot[a.e_begin + t];
        s_tiles[t + 1] = (ne + bn - 1) / bn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s_tiles[0] = 0;
        for (int t = 0; t < n_local; ++t) s_tiles[t + 1] += s_tiles[t];  // prefix over resident experts
        const long base = static_cast<long>(s_tiles[n_local] + a.num_shared * sh_tiles) * a.mb_count;
        int best = a.main_kc ? max(1, a.nsplit_min) : 1;
        float best_score = -1.0f;
        const int cap = a.main_kc ? max(1, min(a.nsplit, a.kc_total)) : 1;
        const int lo_ns = a.main_kc ? min(max(1, a.nsplit_min), cap) : 1;
        for (int ns = lo_ns; ns <= cap; ++ns) {
            const long units = base * ns;
            const long rounds = (units + a.num_sms - 1) / a.num_sms;
            const float eff = rounds > 0 ? static_cast<float>(units) / static_cast<float>(rounds * a.num_sms) : 1.0f;
            float score = eff - (a.split_cost + 0.002f) * (ns - lo_ns);
            if (a.unit_cost8 > 0) {
                // decode (contiguous unit runs): a CTA's time ~ its units x (chunks per
                // unit + the per-unit pipeline cost), measured ~3.7 chunks per unit
                const float per_unit = static_cast<float>((a.kc_total + ns - 1) / ns) + a.unit_cost8 / 8.0f;
                score = -static_cast<float>(rounds) * per_unit * (1.0f + a.split_cost * (ns - lo_ns));
            }
            if (score > best_score + 1e-6f) {
                best_score = score;
                best = ns;
            }
        }
        s_nsplit = best;
        if (a.nsplit_out) *a.nsplit_out = best;
        // ext-balanced split boundaries (the last split also streams the ext
        // blocks): kept only if every unit still fits the resident slots
        int e8 = (a.main_kc && best > 1) ? a.ext8 : 0;
        if (e8 > 0 && a.max_run > 0) {
            for (int sp = 0; sp < best; ++sp) {
                const int len = split_bound(sp + 1, best, a.kc_total, e8) - split_bound(sp, best, a.kc_total, e8) +
                                (sp == best - 1 ? a.n_ext : 0);
                if (len > a.max_run) e8 = 0;
            }
        }
        s_ext8 = e8;
    }
    __syncthreads();
    const int ns = s_nsplit;
    const int ext8 = s_ext8;
    const int routed_units = s_tiles[n_local] * a.mb_count * ns;
    const int shared_units = a.num_shared * sh_tiles * a.mb_count * ns;
    const int total = routed_units + shared_units;
    for (int u = threadIdx.x; u < total; u += blockDim.x) {
        Unit un;
        int sp = u % ns;
        int rest = u / ns;
        if (u < routed_units) {
            int t, mb, tl;
            if (a.run_order) {
                // (expert, tile, split, m-block), m-block fastest: consecutive units share X
                mb = u % a.mb_count;
                const int r2 = u / a.mb_count;
                sp = r2 % ns;
                const int tg = r2 / ns;   // global tile index
                int lo = 0, hi = n_local;  // s_tiles[lo] <= tg < s_tiles[hi]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_tiles[mid] <= tg) lo = mid; else hi = mid;
                }
                t = lo;
                tl = tg - s_tiles[t];
            } else {
                // rest = (tile-global index) over (e, mb, tile): ordered e, mb, tile
                // find expert: units of expert t = (s_tiles[t+1]-s_tiles[t]) * mb_count
                int lo = 0, hi = n_local;  // s_tiles[lo]*mb <= rest < s_tiles[hi]*mb
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_tiles[mid] * a.mb_count <= rest) lo = mid; else hi = mid;
                }
                t = lo;
                const int within = rest - s_tiles[t] * a.mb_count;
                const int ntl = s_tiles[t + 1] - s_tiles[t];
                mb = within / ntl;
                tl = within % ntl;
            }
            const int e = a.e_begin + t;
            const int ne = tot[e + 1] - tot[e];
            un.weight = t;
            un.mb = mb;
            un.x_row = (a.poffsets ? ptot[e] : tot[e]) + tl * bn;
            un.n_tok = min(bn, ne - tl * bn);
            un.y_row = un.x_row;
        } else {
            int s, mb, tl;
            if (a.run_order) {
                const int v = u - routed_units;   // (s, tile, split, mb)
                mb = v % a.mb_count;
                const int r2 = v / a.mb_count;
                sp = r2 % ns;
                const int tg = r2 / ns;
                s = tg / sh_tiles;
                tl = tg % sh_tiles;
            } else {
                rest -= s_tiles[n_local] * a.mb_count;
                s = rest / (sh_tiles * a.mb_count);
                const int within = rest % (sh_tiles * a.mb_count);
                mb = within / sh_tiles;
                tl = within % sh_tiles;
            }
            const int base = a.poffsets ? ptot[K] : n_slots;
            un.weight = n_local + s;
            un.mb = mb;
            un.x_row = base + tl * bn;
            un.n_tok = min(bn, a.batch - tl * bn);
            un.y_row = base + s * a.batch + tl * bn;
        }
        un.kc_begin = static_cast<int16_t>(a.main_kc ? split_bound(sp, ns, a.kc_total, ext8) : 0);
        un.kc_end = static_cast<int16_t>(a.main_kc ? split_bound(sp + 1, ns, a.kc_total, ext8) : 0);
        un.n_ext = static_cast<int16_t>(sp == ns - 1 ? a.n_ext : 0);
        un.split = static_cast<int16_t>(sp);
        un.pad = 0;
        a.units[u] = un;
    }
    if (threadIdx.x == 0) *a.n_units = total;
    // projection pass units: stacked projection weight (index 0) x all tokens
    if (a.proj_mb > 0) {
        const int pbn = a.proj_bn > 0 ? a.proj_bn : bn;
        const int tiles = (a.batch + pbn - 1) / pbn;
        const int np = a.proj_mb * tiles * a.proj_nsplit;
        for (int u = threadIdx.x; u < np; u += blockDim.x) {
            const int sp = u % a.proj_nsplit;
            const int rest = u / a.proj_nsplit;
            const int mb = rest / tiles, tl = rest % tiles;
            Unit un;
            un.weight = 0;
            un.mb = mb;
            un.x_row = tl * pbn;
            un.n_tok = min(pbn, a.batch - tl * pbn);
            un.y_row = tl * pbn;
            un.kc_begin = static_cast<int16_t>(sp * a.proj_kc_total / a.proj_nsplit);
            un.kc_end = static_cast<int16_t>((sp + 1) * a.proj_kc_total / a.proj_nsplit);
            un.n_ext = 0;
            un.split = static_cast<int16_t>(sp);
            un.pad = 0;
            a.proj_units[u] = un;
        }
        if (threadIdx.x == 0 && a.n_proj_units) *a.n_proj_units = np;
    } else if (threadIdx.x == 0 && a.n_proj_units) {
        *a.n_proj_units = 0;
    }
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const PlanArgs a) {
    extern __shared__ int32_t pl_smem[];
    pdl_wait();
    pdl_launch_dependents();
    plan_body(a, pl_smem);
}

// =============================================================================
// gather: permuted fp16 activation rows + extension rows
// =============================================================================


__global__ void __launch_bounds__(256) gather_kernel(const GatherArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    const int n_slots = a.offsets[a.num_experts];
    const int rows = n_slots + (a.with_shared ? a.batch : 0);
    const int row = blockIdx.x;
    if (row >= rows) return;
    int b, e = -1;
    int64_t prow = row;   // destination row
    if (row < n_slots) {
        const int f = a.perm[row];
        b = f / a.top_k;
        e = a.ids[f];
        if (a.poffsets) prow = row + a.poffsets[e] - a.offsets[e];
    } else {
        b = row - n_slots;
        if (a.poffsets) prow = a.poffsets[a.num_experts] + b;
    }
    // destination of the 16-byte piece t (8 halves) of a row with `cols` columns
    auto dst_piece = [&](__half* base, int cols, int t) -> int4* {
        if (a.atom_rows > 0) {
            const int at = t >> 3, ch = t & 7;
            return reinterpret_cast<int4*>(base + ((static_cast<int64_t>(at) * a.atom_rows + prow) * 64 +
                                                   ((ch ^ static_cast<int>(prow & 7)) << 3)));
        }
        return reinterpret_cast<int4*>(base + prow * cols) + t;
    };
    // activation row: 16-byte vector copy
    const int4* src = reinterpret_cast<const int4*>(a.x16 + static_cast<int64_t>(b) * a.k_pad);
    for (int t = threadIdx.x; t < a.k_pad / 8; t += blockDim.x) *dst_piece(a.xp, a.k_pad, t) = src[t];
    // extension row: [Sx | zscale * sum_splits(Z) * rowscale | 0], 8 columns per thread
    for (int t = threadIdx.x; t < a.ext_cols / 8; t += blockDim.x) {
        __align__(16) __half h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int col = t * 8 + q;
            float v = 0.0f;
            if (col < a.groups) {
                if (a.use_sx) v = a.sx[static_cast<int64_t>(b) * a.groups + col];
            } else if (col < a.groups + a.rank) {
                if (a.use_z && e >= 0) {
                    const int j = col - a.groups;
                    const int zc = a.pm_of[e] * a.rank + j;
                    float z = 0.0f;
                    for (int sp = 0; sp < a.proj_nsplit; ++sp)
                        z += a.zpart[sp * a.zsplit_stride + static_cast<int64_t>(b) * a.zcols + zc];
                    v = z * a.rowscale[zc] * a.zscale[e];
                }
            }
            h[q] = __float2half_rn(v);
        }
        *dst_piece(a.ep, a.ext_cols, t) = *reinterpret_cast<const int4*>(h);
    }
}

// =============================================================================
// combine: y[b] = sum_t g_bt * Y[inv(b,t)] + sum_s Yshared_s[b]
// =============================================================================


// Token-major gather (the forward path): CTA b reads token b's fp16 activation
// row once and writes it to each of its top_k expert slots (+ the shared-expert
// row), with the extension rows.  The projection partials Z are reduced with
// the split index spread over threads (independent loads, fixed order).
constexpr int kGatherThreads = 256;
constexpr int kGatherMaxDest = 65;   // top_k <= 64, + shared

__global__ void __launch_bounds__(kGatherThreads) gather_tokens_kernel(const GatherArgs a) {
    extern __shared__ float s_z[];             // [top_k][rank]
    __shared__ float s_part[kGatherThreads];
    __shared__ int64_t s_row[kGatherMaxDest];  // destination row (-1: none)
    __shared__ int s_e[kGatherMaxDest];
    pdl_wait();
    pdl_launch_dependents();
    const int b = blockIdx.x;
    const int nr = a.num_experts > 0 ? a.top_k : 0;
    const int nd = nr + (a.with_shared ? 1 : 0);
    if (threadIdx.x < nd) {
        int64_t prow = -1;
        int e = -1;
        if (static_cast<int>(threadIdx.x) < nr) {
            const int f = b * nr + threadIdx.x;
            const int pos = a.inv[f];
            e = a.ids[f];
            if (pos >= 0) prow = a.poffsets ? pos + a.poffsets[e] - a.offsets[e] : pos;
            else e = -1;
        } else {
            prow = (a.poffsets ? a.poffsets[a.num_experts] : a.offsets[a.num_experts]) + b;
        }
        s_row[threadIdx.x] = prow;
        s_e[threadIdx.x] = e;
    }
    __syncthreads();
    // Z of each routed destination: sum over the projection's K splits
    const int pairs = a.use_z ? nr * a.rank : 0;
    if (pairs > 0) {
        const int ns = a.proj_nsplit;
        const int G = pairs >= kGatherThreads ? 1 : min(ns, kGatherThreads / pairs);
        const int per = kGatherThreads / G;
        for (int p0 = 0; p0 < pairs; p0 += per) {
            const int pi = threadIdx.x % per, g = threadIdx.x / per, pair = p0 + pi;
            float acc = 0.0f;
            if (pair < pairs && g < G) {
                const int d = pair / a.rank, j = pair % a.rank, e = s_e[d];
                if (e >= 0) {
                    const float* zb = a.zpart + static_cast<int64_t>(b) * a.zcols + a.pm_of[e] * a.rank + j;
#pragma unroll 4
                    for (int sp = g; sp < ns; sp += G) acc += zb[sp * a.zsplit_stride];
                }
            }
            s_part[threadIdx.x] = acc;
            __syncthreads();
            if (static_cast<int>(threadIdx.x) < per && p0 + static_cast<int>(threadIdx.x) < pairs) {
                float z = 0.0f;
                for (int q = 0; q < G; ++q) z += s_part[q * per + threadIdx.x];
                s_z[p0 + threadIdx.x] = z;
            }
            __syncthreads();
        }
    }
    auto dst_piece = [&](__half* base, int cols, int64_t prow, int t) -> int4* {
        if (a.atom_rows > 0) {
            const int at = t >> 3, ch = t & 7;
            return reinterpret_cast<int4*>(base + ((static_cast<int64_t>(at) * a.atom_rows + prow) * 64 +
                                                   ((ch ^ static_cast<int>(prow & 7)) << 3)));
        }
        return reinterpret_cast<int4*>(base + prow * cols) + t;
    };
    // activation row, read once, written to every destination
    const int4* src = reinterpret_cast<const int4*>(a.x16 + static_cast<int64_t>(b) * a.k_pad);
    for (int t = threadIdx.x; t < a.k_pad / 8; t += kGatherThreads) {
        const int4 v = src[t];
        for (int d = 0; d < nd; ++d)
            if (s_row[d] >= 0) *dst_piece(a.xp, a.k_pad, s_row[d], t) = v;
    }
    // extension rows: [Sx | zscale * Z * rowscale | 0]
    const int n8 = a.ext_cols / 8;
    for (int idx = threadIdx.x; idx < nd * n8; idx += kGatherThreads) {
        const int d = idx / n8, t = idx % n8;
        const int64_t prow = s_row[d];
        if (prow < 0) continue;
        const int e = s_e[d];
        __align__(16) __half h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int col = t * 8 + q;
            float v = 0.0f;
            if (col < a.groups) {
                if (a.use_sx) v = a.sx[static_cast<int64_t>(b) * a.groups + col];
            } else if (col < a.groups + a.rank) {
                if (pairs > 0 && e >= 0) {
                    const int j = col - a.groups;
                    v = s_z[d * a.rank + j] * a.rowscale[a.pm_of[e] * a.rank + j] * a.zscale[e];
                }
            }
            h[q] = __float2half_rn(v);
        }
        *dst_piece(a.ep, a.ext_cols, prow, t) = *reinterpret_cast<const int4*>(h);
    }
}

__global__ void __launch_bounds__(256) combine_kernel(const CombineArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    // 4 consecutive output columns per thread (float4 when out_dim % 4 == 0)
    const int b = blockIdx.y;
    const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (c0 >= a.out_dim) return;
    const bool vec = (a.out_dim & 3) == 0;
    const int n_slots = a.offsets ? a.offsets[a.num_experts] : 0;
    const int ns = a.nsplit_dev ? *a.nsplit_dev : a.nsplit;
    const int nsh = a.nsplit_dev ? ns : a.sh_nsplit;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    auto load4 = [&](const float* base, float (&v)[4]) {
        if (vec) {
            const float4 t = *reinterpret_cast<const float4*>(base);
            v[0] += t.x; v[1] += t.y; v[2] += t.z; v[3] += t.w;
        } else {
            for (int j = 0; j < 4; ++j)
                if (c0 + j < a.out_dim) v[j] += base[j];
        }
    };
    if (a.use_routed) {
        for (int t = 0; t < a.top_k; ++t) {
            const int f = b * a.top_k + t;
            int pos = a.inv[f];
            if (pos < 0) continue;  // invalid expert id (reported through the error flag)
            if (a.poffsets) {
                const int e = a.ids[f];
                pos += a.poffsets[e] - a.offsets[e];
            }
            float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 8
            for (int sp = 0; sp < ns; ++sp)
                load4(a.y + sp * a.split_stride + static_cast<int64_t>(pos) * a.out_dim + c0, v);
            const float g = a.gates[f];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fmaf(g, v[j], acc[j]);
        }
    }
    const int64_t sh0 = a.sh_from_offsets ? (a.poffsets ? a.poffsets[a.num_experts] : n_slots) : 0;
    for (int s = 0; s < a.num_shared; ++s) {
        const int64_t r = sh0 + static_cast<int64_t>(s) * a.batch + b;
        float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int sp = 0; sp < nsh; ++sp) load4(a.ysh + sp * a.sh_split_stride + r * a.out_dim + c0, v);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += v[j];
    }
    float* o = a.out + static_cast<int64_t>(b) * a.out_dim + c0;
    if (vec) {
        *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
        for (int j = 0; j < 4; ++j)
            if (c0 + j < a.out_dim) o[j] = acc[j];
    }
}

// =============================================================================
// unpack_codes (codec.cpp:168-195) and the export of the repacked layout
// =============================================================================

__global__ void unpack_kernel(const uint8_t* __restrict__ bytes, int64_t nbytes, int bits, int64_t count,
                              uint32_t* __restrict__ out, int32_t* __restrict__ err_flag) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += stride) {
        const int64_t bit = t * bits;
        const int64_t byte = bit >> 3;
        uint32_t w = bytes[byte];
        if (byte + 1 < nbytes) w |= static_cast<uint32_t>(bytes[byte + 1]) << 8;
        out[t] = (w >> (bit & 7)) & ((1u << bits) - 1u);
    }
    // padding bits beyond the last code must be zero
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t used = count * bits;
        for (int64_t bit = used; bit < nbytes * 8; ++bit)
            if (bytes[bit >> 3] & (1u << (bit & 7))) *err_flag = 1;
    }
}

// decode one super-word back to 32 codes (inverse of the loader's packing)
__device__ __forceinline__ void superword_codes(const uint32_t* w, int bits, uint32_t (&c)[32]) {
    if (bits == 2) {
        for (int j = 0; j < 2; ++j)
            for (int m = 0; m < 8; ++m) {
                const int p = 8 * j + m;
                c[2 * p] = (w[j] >> (2 * m)) & 3u;
                c[2 * p + 1] = (w[j] >> (16 + 2 * m)) & 3u;
            }
    } else if (bits == 3) {
        const int pos[5] = {0, 3, 6, 9, 12};
        for (int j = 0; j < 3; ++j)
            for (int m = 0; m < 5; ++m) {
                const int p = 5 * j + m;
                c[2 * p] = (w[j] >> pos[m]) & 7u;
                c[2 * p + 1] = (w[j] >> (16 + pos[m])) & 7u;
            }
        c[30] = ((w[0] >> 15) & 1u) | (((w[1] >> 15) & 1u) << 1) | (((w[2] >> 15) & 1u) << 2);
        c[31] = ((w[0] >> 31) & 1u) | (((w[1] >> 31) & 1u) << 1) | (((w[2] >> 31) & 1u) << 2);
    } else if (bits == 4) {
        for (int j = 0; j < 4; ++j)
            for (int m = 0; m < 4; ++m) {
                const int p = 4 * j + m;
                c[2 * p] = (w[j] >> (4 * m)) & 15u;
                c[2 * p + 1] = (w[j] >> (16 + 4 * m)) & 15u;
            }
    } else {
        for (int j = 0; j < 8; ++j)
            for (int m = 0; m < 2; ++m) {
                const int p = 2 * j + m;
                c[2 * p] = (w[j] >> (8 * m)) & 255u;
                c[2 * p + 1] = (w[j] >> (16 + 8 * m)) & 255u;
            }
    }
}

__global__ void export_codes_kernel(const uint8_t* __restrict__ wcodes, int bits, int kc_total, int out_dim,
                                    int in_dim, uint32_t* __restrict__ out) {
    // one thread per (row, 32-code half-chunk)
    const int64_t halves = static_cast<int64_t>(kc_total) * 2;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(out_dim) * halves) return;
    const int row = static_cast<int>(t / halves);
    const int hc = static_cast<int>(t % halves);
    const int kc = hc >> 1, h = hc & 1;
    const int mb = row / kBM, rloc = row % kBM;
    const int bb = code_block_bytes(bits);
    const uint32_t* blk = reinterpret_cast<const uint32_t*>(wcodes + (static_cast<int64_t>(mb) * kc_total + kc) * bb);
    uint32_t w[8];
    for (int j = 0; j < bits; ++j) w[j] = blk[(h * bits + j) * kBM + rloc];
    uint32_t c[32];
    superword_codes(w, bits, c);
    for (int k = 0; k < 32; ++k) {
        const int col = kc * kKC + 32 * h + k;
        if (col < in_dim) out[static_cast<int64_t>(row) * in_dim + col] = c[k];
    }
}

// =============================================================================
// decode path, launch 1: route + rank-r projections + scatter into expert slots
// =============================================================================
//
// Grid (token b, y): y < nslices scores kRouteExperts experts of token b
// (route_slice, bit-exact route()); the next num_q CTAs compute the token's
// rank-r projection of each folded / scalar tile column q (infer.cpp:104-121):
//     Z_q[j] = sigma_j * vabs_q/127 * sum_c v_q[j, c] * x[c] / s_q[c]
// (the reference's x . P^T with P = sigma * v / s, formed as v . (x / s) with
// the exact int8 codes).  The last CTA of the token (ticket) picks the top-k,
// takes a slot in each chosen expert (atomic counter; the row order inside an
// expert is irrelevant to the numerics: every row is an independent MMA
// column), computes general-tier projections for its routed experts only
// (x / s_e, infer.cpp:133-155 -- work B * top_k * r * i), and writes the fp16
// activation row and the extension row [Sx | Z * zscale_e] of every destination
// in the atom-major swizzled layout the expert GEMM bulk-copies.

__device__ __forceinline__ void rtrace(const DecRouteArgs& a, int k, unsigned tid = 0) {
#ifdef TQ_ROUTE_TRACE
    if (threadIdx.x == tid && a.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[(blockIdx.x * gridDim.y + blockIdx.y) * 16 + k] = t;
    }
#else
    (void)a;
    (void)k;
    (void)tid;
#endif
}

// out[j] = vscale[j] * sum_c codes[j, c] * xs(c) for j < r, xs(c) = x[c] / s[c] (s may be
// null: xs = x).  The whole CTA takes part: xs is staged in shared memory (xs_sm,
// 4096 floats, columns in chunks of 4096); warp w owns rows j = w, w + nw, ...; each
// lane issues all its 16-byte code loads of a row before using them (one memory
// round trip per row, not one per column block); fixed-order warp reduction.
template <int kRT>
__device__ void dec_project(const float* __restrict__ xb, const float* __restrict__ s, int in_dim,
                            const int8_t* __restrict__ codes, const float* __restrict__ vscale, int r,
                            float* out, float* xs_sm, const DecRouteArgs* ta = nullptr) {
    constexpr int kNW = kRT / 32;
    constexpr int kChunk = 4096;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool vec = (in_dim & 15) == 0;
    constexpr int kT = (64 + kNW - 1) / kNW;   // rows warp + kNW * t cover r <= 64
    float acc[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) acc[t] = 0.0f;
    for (int c0 = 0; c0 < in_dim; c0 += kChunk) {
        const int nc = min(kChunk, in_dim - c0);
        __syncthreads();   // xs_sm of the previous chunk / caller consumed
        for (int c = threadIdx.x; c < nc; c += kRT) xs_sm[c] = s ? __fdiv_rn(xb[c0 + c], s[c0 + c]) : xb[c0 + c];
        __syncthreads();
        if (ta) rtrace(*ta, 9);
#pragma unroll
        for (int t = 0; t < kT; ++t) {
            const int j = warp + kNW * t;
            if (j >= r) break;
            const int8_t* row = codes + static_cast<int64_t>(j) * in_dim + c0;
            if (vec) {
#pragma unroll
                for (int u0 = 0; u0 < 8; u0 += 4) {
                int4 v[4];   // 16 codes per load, lane-strided 16-byte pieces (coalesced)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = 16 * (lane + 32 * (u0 + u));
                    v[u] = cc < nc ? __ldg(reinterpret_cast<const int4*>(row + cc)) : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = 16 * (lane + 32 * (u0 + u));
                    if (cc < nc) {
                        const float4* x4 = reinterpret_cast<const float4*>(xs_sm + cc);
                        const uint32_t wv[4] = {static_cast<uint32_t>(v[u].x), static_cast<uint32_t>(v[u].y),
                                                static_cast<uint32_t>(v[u].z), static_cast<uint32_t>(v[u].w)};
#pragma unroll
                        for (int m4 = 0; m4 < 4; ++m4) {
                            // int8 -> float on the full-rate ALU: bias to unsigned, splice the byte
                            // into the mantissa of 2^23 (PRMT), subtract 2^23 + 128 (exact)
                            const uint32_t ub = wv[m4] ^ 0x80808080u;
                            const float4 xv = x4[m4];
                            const float c0 = __uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7540)) - 8388736.0f;
                            const float c1 = __uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7541)) - 8388736.0f;
                            const float c2 = __uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7542)) - 8388736.0f;
                            const float c3 = __uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7543)) - 8388736.0f;
                            acc[t] = fmaf(c0, xv.x, acc[t]);
                            acc[t] = fmaf(c1, xv.y, acc[t]);
                            acc[t] = fmaf(c2, xv.z, acc[t]);
                            acc[t] = fmaf(c3, xv.w, acc[t]);
                        }
                    }
                }
                }
            } else {
                for (int c = lane; c < nc; c += 32) acc[t] = fmaf(static_cast<float>(row[c]), xs_sm[c], acc[t]);
            }
        }
    }
    if (ta) rtrace(*ta, 10);
#pragma unroll
    for (int t = 0; t < kT; ++t) {
        const int j = warp + kNW * t;
        if (j >= r) break;
        float v = acc[t];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) out[j] = v * vscale[j];
    }
}

// Projection CTA of the decode router: rows [j0, j0 + 16) of tile column q for one
// token, column-parallel -- thread t owns columns [8t, 8t + 8) (+ 8 * kRT per pass),
// issues its x, s and int8 V loads together (one memory round trip), forms the 16
// partial dot products, and a fixed-order block reduction finishes them:
//     out[j] = vscale[j] * sum_c v[j, c] * x[c] / s[c]        (s may be null: x)
constexpr int kProjRows = 8;
template <int kRT>
__device__ void dec_project_rows(const float* __restrict__ xb, const float* __restrict__ s, int in_dim,
                                 const int8_t* __restrict__ codes, const float* __restrict__ vscale, int nrows,
                                 float* out, float* red /* [kRT / 32][kProjRows] */) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc[kProjRows];
#pragma unroll
    for (int j = 0; j < kProjRows; ++j) acc[j] = 0.0f;
    const bool vec = (in_dim & 7) == 0;
    for (int c0 = 8 * threadIdx.x; c0 < in_dim; c0 += 8 * kRT) {
        float xs[8];
        uint32_t v[kProjRows][2];
        if (vec) {
            const float4 xa = __ldg(reinterpret_cast<const float4*>(xb + c0));
            const float4 xc = __ldg(reinterpret_cast<const float4*>(xb + c0 + 4));
            float4 sa = make_float4(1.f, 1.f, 1.f, 1.f), sc4 = sa;
            if (s) {
                sa = __ldg(reinterpret_cast<const float4*>(s + c0));
                sc4 = __ldg(reinterpret_cast<const float4*>(s + c0 + 4));
            }
#pragma unroll
            for (int j = 0; j < kProjRows; ++j) {
                if (j < nrows) {
                    const uint2 w = __ldg(reinterpret_cast<const uint2*>(codes + static_cast<int64_t>(j) * in_dim + c0));
                    v[j][0] = w.x;
                    v[j][1] = w.y;
                } else {
                    v[j][0] = v[j][1] = 0x80808080u ^ 0x80808080u;
                }
            }
            xs[0] = xa.x; xs[1] = xa.y; xs[2] = xa.z; xs[3] = xa.w;
            xs[4] = xc.x; xs[5] = xc.y; xs[6] = xc.z; xs[7] = xc.w;
            if (s) {
                xs[0] = __fdiv_rn(xs[0], sa.x); xs[1] = __fdiv_rn(xs[1], sa.y);
                xs[2] = __fdiv_rn(xs[2], sa.z); xs[3] = __fdiv_rn(xs[3], sa.w);
                xs[4] = __fdiv_rn(xs[4], sc4.x); xs[5] = __fdiv_rn(xs[5], sc4.y);
                xs[6] = __fdiv_rn(xs[6], sc4.z); xs[7] = __fdiv_rn(xs[7], sc4.w);
            }
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int c = c0 + m;
                xs[m] = c < in_dim ? (s ? __fdiv_rn(xb[c], s[c]) : xb[c]) : 0.0f;
            }
#pragma unroll
            for (int j = 0; j < kProjRows; ++j) {
                uint32_t b[2] = {0u, 0u};
                for (int m = 0; m < 8; ++m) {
                    const int c = c0 + m;
                    const uint32_t byte = (j < nrows && c < in_dim) ? static_cast<uint8_t>(codes[static_cast<int64_t>(j) * in_dim + c]) : 0u;
                    b[m >> 2] |= byte << (8 * (m & 3));
                }
                v[j][0] = b[0];
                v[j][1] = b[1];
            }
        }
#pragma unroll
        for (int j = 0; j < kProjRows; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                // int8 -> float on the full-rate ALU: bias to unsigned, splice the byte into
                // the mantissa of 2^23 (PRMT), subtract 2^23 + 128 (exact)
                const uint32_t ub = v[j][h] ^ 0x80808080u;
                acc[j] = fmaf(__uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7540)) - 8388736.0f, xs[4 * h + 0], acc[j]);
                acc[j] = fmaf(__uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7541)) - 8388736.0f, xs[4 * h + 1], acc[j]);
                acc[j] = fmaf(__uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7542)) - 8388736.0f, xs[4 * h + 2], acc[j]);
                acc[j] = fmaf(__uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7543)) - 8388736.0f, xs[4 * h + 3], acc[j]);
            }
        }
    }
    // warp reduce-scatter (fixed order): after the halvings lane l holds the sum over
    // its lane group of row (l % kProjRows); the remaining exchanges add the groups
#pragma unroll
    for (int h = kProjRows / 2; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const float send = up ? acc[j] : acc[j + h];
            const float keep = up ? acc[j + h] : acc[j];
            acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
#pragma unroll
    for (int h = kProjRows; h < 32; h <<= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], h);
    if (lane < kProjRows) red[warp * kProjRows + lane] = acc[0];
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < nrows) {
        float v = 0.0f;
        for (int w = 0; w < kRT / 32; ++w) v += red[w * kProjRows + threadIdx.x];
        out[threadIdx.x] = v * vscale[threadIdx.x];
    }
}

#ifdef TQ_DEC_CHECK
#define RT_CHECK(cond, ...)                                                                     \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("RT_CHECK line %d cta (%d,%d) thr %d: " #cond "\n", __LINE__, blockIdx.x,     \
                   blockIdx.y, threadIdx.x);                                                    \
            printf(__VA_ARGS__);                                                                \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define RT_CHECK(cond, ...) \
    do {                    \
    } while (0)
#endif
constexpr int kDecRT = 512;

constexpr int kDecStage16 = 4096;   // fp16 row staged in shared memory up to this k_pad
constexpr int kDecZq = 512;         // projections of a token prefetched up to num_q * rank floats

// (one CTA per SM: capped at 64 registers for two, the spilling build faulted
// intermittently in the bench -- kept uncapped)
// kRT = 512 (one CTA per SM) for a handful of tokens; 256 (two per SM, half the waves)
// when the grid is many CTAs deep
template <int kRT>
__global__ void __launch_bounds__(kRT, 512 / kRT) dec_route_kernel(const DecRouteArgs a) {
    __shared__ RouteSmem<kRT> sm;
    __shared__ float sc[64];
    __shared__ double ex[64];
    __shared__ int pick_k[64];
    __shared__ double pick_p[64];
    __shared__ int s_last;
    __shared__ int s_row[kDecMaxTopK + 64];
    __shared__ int s_e[kDecMaxTopK + 64];
    __shared__ float s_sx[64];
    __shared__ float s_z[kDecMaxTopK][64];
    __shared__ __align__(16) __half s_x16[kDecStage16];
    __shared__ float s_zq[kDecZq];
    __shared__ int s_eq[64], s_qt[64];           // e -> tile column, column -> descale tier (last CTA)
    __shared__ float s_zs[64];                   // e -> zscale
    const int b = blockIdx.x;
    const int K = a.num_experts;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslices = a.given ? 0 : (K + kRouteExperts - 1) / kRouteExperts;
    const float* xb = a.x + static_cast<int64_t>(b) * a.in_dim;
    const int y = blockIdx.y;
    rtrace(a, 0);
    if (y < nslices) {
        (void)route_slice<kRT>(xb, a.in_dim, a.gate, K, y * kRouteExperts, a.score_ws + static_cast<int64_t>(b) * K,
                               sm);
    } else {
        // projection CTA: rows [kProjRows * rs, + kProjRows) of tile column q
        const int rs_cnt = (a.rank + kProjRows - 1) / kProjRows;
        const int q = (y - nslices) / rs_cnt, rs = (y - nslices) % rs_cnt;
        RT_CHECK(q < a.num_q && b < a.batch, "q %d rs %d y %d nslices %d\n", q, rs, y, nslices);
        const int tier = a.q_tier[q];
        RT_CHECK(tier >= -1 && tier <= 2 && (tier != 0 || (a.q_first[q] >= 0 && a.q_first[q] < K)), "tier %d first %d\n",
                 tier, a.q_first[q]);
        if (a.use_lr && (tier == 0 || tier == 1)) {
            const float* s = tier == 0 ? a.scaling + static_cast<int64_t>(a.q_first[q]) * a.in_dim : nullptr;
            const int j0 = rs * kProjRows;
            dec_project_rows<kRT>(xb, s, a.in_dim, a.vcodes + (static_cast<int64_t>(q) * a.rank + j0) * a.in_dim,
                                     a.vscale + q * a.rank + j0, min(kProjRows, a.rank - j0),
                                     a.zq_ws + (static_cast<int64_t>(b) * a.num_q + q) * a.rank + j0,
                                     reinterpret_cast<float*>(sm.prod));
        }
    }
    // publication without per-thread fences: the barrier orders every thread's score /
    // projection stores before thread 0's gpu-scope acq_rel ticket increment, which
    // releases them (cumulatively) and, in the last CTA, acquires the other CTAs'
    // stores for every thread behind the next barrier (they read them through L2)
    __syncthreads();
    rtrace(a, 1);
    if (threadIdx.x == 0) {
        int done;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(done) : "l"(a.ticket + b) : "memory");
        s_last = done == static_cast<int>(gridDim.y) - 1;
        if (s_last) a.ticket[b] = 0;   // ready for the next launch
#ifdef TQ_DEC_CHECK
        if (done >= static_cast<int>(gridDim.y)) {
            printf("DEC_CHECK router: token %d ticket %d >= %d\n", b, done, static_cast<int>(gridDim.y));
            __trap();
        }
#endif
    }
    __syncthreads();
    if (!s_last) return;
    rtrace(a, 2);
    const int k = a.top_k;
    // ---- routing decision (warp 0), overlapped with the token's loads (other warps):
    //      group sums of the fp16 activations, the fp16 row staged in shared memory,
    //      the folded / scalar tile columns' projections of this token ----
    if (!a.given) {
        if (warp == 0) {
            route_pick(a.score_ws + static_cast<int64_t>(b) * K, K, k, sc, ex, pick_k, pick_p,
                       a.ids + static_cast<int64_t>(b) * k, a.gates + static_cast<int64_t>(b) * k, false);
            rtrace(a, 11);
        }
    } else if (static_cast<int>(threadIdx.x) < k) {
        pick_k[threadIdx.x] = a.ids_in[static_cast<int64_t>(b) * k + threadIdx.x];
    }
    const int w0 = a.given ? 0 : 1;   // first warp free of the pick
    // small per-layer tables the tail reads per destination, staged once (no dependent
    // global loads after the pick); issued first so their latency overlaps the x pass
    for (int t = threadIdx.x; t < K; t += kRT) {
        s_eq[t] = a.e_q[t];
        s_zs[t] = a.zscale[t];
    }
    for (int t = threadIdx.x; t < a.num_q; t += kRT) s_qt[t] = a.q_tier[t];
    const int nzq = a.use_lr ? a.num_q * a.rank : 0;
    if (nzq <= kDecZq) {
        const float* zi = a.zq_ws + static_cast<int64_t>(b) * nzq;
        for (int t = threadIdx.x - 32 * w0; t >= 0 && t < nzq; t += kRT - 32 * w0) s_zq[t] = __ldcg(zi + t);
    }
    const bool stage16 = a.use_main && a.k_pad <= kDecStage16;
    // one pass over x for 128-column groups (the BASELINE shapes): warp w takes groups
    // w, w + nw, ...; every lane loads all its float4s first, then writes the fp16 row
    // and the group sums of the fp16-rounded values (one memory round trip, not two)
    constexpr int kGPW = 6;   // groups per warp held in flight
    const int nw = kRT / 32 - w0;
    const bool one_pass = stage16 && a.group_size == 128 && a.in_dim == a.k_pad && a.groups <= kGPW * nw;
    if (one_pass && warp >= w0) {
        float4 v[kGPW];
#pragma unroll
        for (int i = 0; i < kGPW; ++i) {
            const int g = warp - w0 + i * nw;
            if (g < a.groups) v[i] = __ldg(reinterpret_cast<const float4*>(xb + g * 128) + lane);
        }
#pragma unroll
        for (int i = 0; i < kGPW; ++i) {
            const int g = warp - w0 + i * nw;
            if (g >= a.groups) break;
            const __half2 h01 = __floats2half2_rn(v[i].x, v[i].y), h23 = __floats2half2_rn(v[i].z, v[i].w);
            reinterpret_cast<__half2*>(s_x16 + g * 128 + 4 * lane)[0] = h01;
            reinterpret_cast<__half2*>(s_x16 + g * 128 + 4 * lane)[1] = h23;
            float acc = (__low2float(h01) + __high2float(h01)) + (__low2float(h23) + __high2float(h23));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
            if (lane == 0) s_sx[g] = acc;
        }
        rtrace(a, 12, 32);
    }
    for (int g = warp - w0; !one_pass && a.use_main && g >= 0 && g < a.groups; g += kRT / 32 - w0) {
        float acc = 0.0f;
        const int c0 = g * a.group_size, c1 = min(a.in_dim, c0 + a.group_size);
        for (int c = c0 + lane; c < c1; c += 32) acc += __half2float(__float2half_rn(xb[c]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
        if (lane == 0) s_sx[g] = acc;
    }
    if (!one_pass && stage16 && warp >= w0) {
        for (int t8 = threadIdx.x - 32 * w0; t8 < a.k_pad / 8; t8 += kRT - 32 * w0) {
            __align__(16) __half hh[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int c = t8 * 8 + m;
                hh[m] = __float2half_rn(c < a.in_dim ? xb[c] : 0.0f);
            }
            reinterpret_cast<int4*>(s_x16)[t8] = *reinterpret_cast<const int4*>(hh);
        }
    }
    __syncthreads();
    rtrace(a, 3);
    // ---- destinations: one slot per routed expert, the shared-expert rows ----
    if (static_cast<int>(threadIdx.x) < k) {
        const int e = pick_k[threadIdx.x];
        RT_CHECK(a.given || (e >= 0 && e < K), "picked expert %d\n", e);
        int row = -1;
        if (e < 0 || e >= K) {
            atomicExch(a.err_flag, 1);   // expert id out of range (moe.cpp:111-114)
        } else {
            const int slot = atomicAdd(&a.cnt[e], 1);
            row = e * a.cap8 + slot;
#ifdef TQ_DEC_CHECK
            if (slot >= a.cap8) {
                printf("DEC_CHECK router: token %d expert %d slot %d >= cap8 %d (pick %d)\n", b, e, slot, a.cap8, threadIdx.x);
                __trap();
            }
#endif
            if (slot >= a.cap8) {   // cannot happen for a valid routing; never write outside the expert's rows
                atomicExch(a.err_flag, 1);
                row = -1;
            }
        }
        s_row[threadIdx.x] = row;
        s_e[threadIdx.x] = row >= 0 ? e : -1;
        a.inv[static_cast<int64_t>(b) * k + threadIdx.x] = row;
    }
    if (static_cast<int>(threadIdx.x) < a.num_shared) {
        s_row[k + threadIdx.x] = (K + static_cast<int>(threadIdx.x)) * a.cap8 + b;
        s_e[k + threadIdx.x] = -1;
    }
    __syncthreads();
    const int nd = k + (a.use_main ? a.num_shared : 0);
    rtrace(a, 4);
    // ---- rank-r terms of the routed destinations ----
    if (a.use_lr) {
        for (int t = 0; t < k; ++t) {
            const int e = s_e[t];
            if (e < 0) continue;   // block-uniform
            const int q = s_eq[e];
            RT_CHECK(q >= 0 && q < a.num_q, "e %d q %d\n", e, q);
            if (s_qt[q] == 2) {
                dec_project<kRT>(xb, a.scaling + static_cast<int64_t>(e) * a.in_dim, a.in_dim,
                                    a.vcodes + static_cast<int64_t>(q) * a.rank * a.in_dim, a.vscale + q * a.rank,
                                    a.rank, s_z[t], reinterpret_cast<float*>(sm.prod));
            } else if (nzq <= kDecZq) {
                for (int j = threadIdx.x; j < a.rank; j += kRT) s_z[t][j] = s_zq[q * a.rank + j];
            } else {
                const float* zi = a.zq_ws + (static_cast<int64_t>(b) * a.num_q + q) * a.rank;
                for (int j = threadIdx.x; j < a.rank; j += kRT) s_z[t][j] = __ldcg(zi + j);
            }
        }
    }
    __syncthreads();
    rtrace(a, 6);
    // ---- fp16 activation row -> every destination (atom-major, 128B swizzle of the row index) ----
    auto piece = [&](__half* base, int row, int t8) -> int4* {
        const int at = t8 >> 3, ch = t8 & 7;
        return reinterpret_cast<int4*>(base + ((static_cast<int64_t>(at) * a.atom_rows + row) * 64 + ((ch ^ (row & 7)) << 3)));
    };
    if (a.use_main) {
        for (int t8 = threadIdx.x; t8 < a.k_pad / 8; t8 += kRT) {
            int4 v;
            if (stage16) {
                v = reinterpret_cast<const int4*>(s_x16)[t8];
            } else {
                __align__(16) __half hh[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int c = t8 * 8 + m;
                    hh[m] = __float2half_rn(c < a.in_dim ? xb[c] : 0.0f);
                }
                v = *reinterpret_cast<const int4*>(hh);
            }
            for (int d = 0; d < nd; ++d) {
                RT_CHECK(s_row[d] < a.atom_rows - 16, "dest %d row %d atom_rows %lld\n", d, s_row[d],
                         static_cast<long long>(a.atom_rows));
                if (s_row[d] >= 0) *piece(a.xperm, s_row[d], t8) = v;
            }
        }
    }
    rtrace(a, 7);
    // ---- extension rows [Sx | Z * zscale_e | 0] ----
    const int n8 = a.ext_cols / 8;
    RT_CHECK(nd <= kDecMaxTopK + 64 && n8 <= 64, "nd %d n8 %d\n", nd, n8);
    for (int idx = threadIdx.x; idx < nd * n8; idx += kRT) {
        const int d = idx / n8, t8 = idx % n8;
        const int row = s_row[d];
        if (row < 0) continue;
        const int e = s_e[d];
        __align__(16) __half h[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int col = t8 * 8 + m;
            float v = 0.0f;
            if (col < a.groups) {
                if (a.use_main) v = s_sx[col];
            } else if (col < a.groups + a.rank) {
                if (a.use_lr && e >= 0) v = s_z[d][col - a.groups] * s_zs[e];
            }
            h[m] = __float2half_rn(v);
        }
        *piece(a.extperm, row, t8) = *reinterpret_cast<const int4*>(h);
    }
    __syncthreads();
    rtrace(a, 8);
}

// decode path, launch 3: y[b] = sum_t g_bt * Y[slot(b, t)] (t ascending) + sum_s Y_s[b]
// (reference_forward's order, moe.cpp:115-132); zeroes the slot counters.
__global__ void __launch_bounds__(256) dec_combine_kernel(const DecCombineArgs a) {
    __shared__ int s_row[64];
    __shared__ float s_gate[64];
    const int b = blockIdx.y;
    if (blockIdx.x == 0 && blockIdx.y == 0)
        for (int e = threadIdx.x; e < a.num_experts; e += blockDim.x) a.cnt[e] = 0;
    if (static_cast<int>(threadIdx.x) < a.top_k) {
        const int64_t f = static_cast<int64_t>(b) * a.top_k + threadIdx.x;
        s_row[threadIdx.x] = a.inv[f];
        s_gate[threadIdx.x] = a.gates[f];
#ifdef TQ_DEC_CHECK
        if (s_row[threadIdx.x] >= (a.num_experts + a.num_shared) * a.cap8) {
            printf("DEC_CHECK combine: token %d t %d row %d >= %d\n", b, threadIdx.x, s_row[threadIdx.x],
                   (a.num_experts + a.num_shared) * a.cap8);
            __trap();
        }
#endif
    }
    __syncthreads();
    const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (c0 >= a.out_dim) return;
    const bool vec = (a.out_dim & 3) == 0 && (a.ldy & 3) == 0;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    auto row4 = [&](int64_t row, float (&v)[4]) {
        const float* p = a.yslot + row * a.ldy + c0;
        if (vec) {
            const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
            for (int j = 0; j < 4; ++j) v[j] = c0 + j < a.out_dim ? p[j] : 0.0f;
        }
    };
    for (int t = 0; t < a.top_k; ++t) {
        if (s_row[t] < 0) continue;
        float v[4];
        row4(s_row[t], v);
        const float g = s_gate[t];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = fmaf(g, v[j], acc[j]);
    }
    for (int s = 0; s < a.num_shared; ++s) {
        float v[4];
        row4(static_cast<int64_t>(a.num_experts + s) * a.cap8 + b, v);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += v[j];
    }
    float* o = a.out + static_cast<int64_t>(b) * a.out_dim + c0;
    if (vec) {
        *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
        for (int j = 0; j < 4; ++j)
            if (c0 + j < a.out_dim) o[j] = acc[j];
    }
}

// =============================================================================
// launch wrappers (called from tq_runtime.cpp)
// =============================================================================

// All kernels of a forward run with the maximum shared-memory carveout, so
// the SMs never reconfigure L1/shared memory between the small kernels and the
// 226 KB expert GEMM (each reconfiguration drains the SM).
template <typename K>
static void max_carveout(K kern) {
    static bool done = false;   // one static per kernel type
    if (!done) {
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        done = true;
    }
}

cudaError_t launch_route(const float* x, int batch, int in_dim, const float* gate, int num_experts, int top_k,
                         int group_size, int groups, int k_pad, int32_t* ids, float* gates, __half* x16, float* sx,
                         float* score_ws, int32_t* ticket, cudaStream_t stream) {
    if (batch <= 0) return cudaSuccess;
    if (num_experts > 64 || top_k > 64) return cudaErrorInvalidValue;
#ifndef TQ_ROUTE_TOKEN_CTAS
#define TQ_ROUTE_TOKEN_CTAS (2 * 148)   // token-chunk CTAs at prefill (several tokens per CTA beyond this)
#endif
    // batch from which the token-tile router runs; the per-token route_kernel below
    // serves smaller batches (at decode sizes the tile router's 16 sequential
    // chunks per CTA cost more than one CTA per token)
    constexpr int tile_min = 297;
    const bool tile_ok = num_experts > 0 && tile_min > 0 && batch >= tile_min && (in_dim & 3) == 0 &&
                         (k_pad & 3) == 0 && (!sx || (group_size > 0 && kTC % group_size == 0));
    if (tile_ok) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(route_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, route_tile_smem(64));
            attr = true;
        }
        return launch_maybe_pdl(route_tile_kernel, dim3((batch + kTT - 1) / kTT), dim3(kTThreads),
                                static_cast<size_t>(route_tile_smem(num_experts)), stream, x, batch, in_dim, gate,
                                num_experts, top_k, group_size, groups, k_pad, ids, gates, x16, sx);
    }
    const int tpc = batch <= TQ_ROUTE_TOKEN_CTAS ? 1 : (batch + TQ_ROUTE_TOKEN_CTAS - 1) / TQ_ROUTE_TOKEN_CTAS;
    const dim3 grid((batch + tpc - 1) / tpc, num_experts > 0 ? (num_experts + kRouteExperts - 1) / kRouteExperts : 1);
    // prefill (several tokens per CTA): 128-thread CTAs (more CTAs per SM); decode: 512
    // (measured at 4096 tokens: 512 -> 1437 us, 256 -> 1367 us, 128 -> 1345 us per forward)
    if (tpc > 1) {
        max_carveout(route_kernel<128>);
        return launch_maybe_pdl(route_kernel<128>, grid, dim3(128), 0, stream, x, batch, in_dim, gate, num_experts,
                                top_k, group_size, groups, k_pad, ids, gates, x16, sx, score_ws, ticket, tpc);
    }
    max_carveout(route_kernel<kRouteThreads>);
    return launch_maybe_pdl(route_kernel<kRouteThreads>, grid, dim3(kRouteThreads), 0, stream, x, batch, in_dim, gate, num_experts,
                            top_k, group_size, groups, k_pad, ids, gates, x16, sx, score_ws, ticket, tpc);
}

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream) {
    const size_t smem = sizeof(int32_t) * (32 * static_cast<size_t>(a.num_experts) + a.num_experts + 1);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    max_carveout(plan_kernel);
    return launch_maybe_pdl(plan_kernel, dim3(1), dim3(kPlanThreads), smem, stream, a);
}

cudaError_t launch_gather(const GatherArgs& a, int max_rows, cudaStream_t stream) {
    if (max_rows <= 0) return cudaSuccess;
    max_carveout(gather_kernel);
    return launch_maybe_pdl(gather_kernel, dim3(max_rows), dim3(256), 0, stream, a);
}

// Large batches: one token per CTA row, 4 float4 columns per thread with the
// token's slot rows resolved once in shared memory -- every load of the
// thread's columns is independent (the per-thread index chain of
// combine_kernel left HBM at ~3 TB/s).  Same summation order as combine_kernel.
constexpr int kCbCols = 256 * 4 * 4;   // columns per CTA
__global__ void __launch_bounds__(256, 4) combine_rows_kernel(const CombineArgs a) {
    __shared__ int64_t s_row[64];
    __shared__ float s_gate[64];
    pdl_wait();
    pdl_launch_dependents();
    const int b = blockIdx.y;
    const int k = a.use_routed ? a.top_k : 0;
    if (static_cast<int>(threadIdx.x) < k) {
        const int f = b * k + threadIdx.x;
        int64_t pos = a.inv[f];
        if (pos >= 0 && a.poffsets) {
            const int e = a.ids[f];
            pos += a.poffsets[e] - a.offsets[e];
        }
        s_row[threadIdx.x] = pos;
        s_gate[threadIdx.x] = a.gates[f];
    }
    __syncthreads();
    const int ns = a.nsplit_dev ? *a.nsplit_dev : a.nsplit;
    const int nsh = a.nsplit_dev ? ns : a.sh_nsplit;
    const int n_slots = a.offsets ? a.offsets[a.num_experts] : 0;
    const int64_t sh0 = a.sh_from_offsets ? (a.poffsets ? a.poffsets[a.num_experts] : n_slots) : 0;
    if (ns == 1 && a.num_shared == 0 && k <= 2) {
        // common prefill case (top-2, one K split, no shared experts): every row
        // load of the CTA's four column groups issued before the first use
        // (same arithmetic as the general loop below: v = 0 + w, acc = fma(g, v, acc))
        float4 w[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c0 = blockIdx.x * kCbCols + (q * 256 + threadIdx.x) * 4;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                w[q][t] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (t < k && c0 < a.out_dim && s_row[t] >= 0)
                    w[q][t] = __ldcs(reinterpret_cast<const float4*>(a.y + s_row[t] * a.out_dim + c0));
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c0 = blockIdx.x * kCbCols + (q * 256 + threadIdx.x) * 4;
            if (c0 >= a.out_dim) break;
            float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (t >= k || s_row[t] < 0) continue;
                const float g = s_gate[t];
                acc[0] = fmaf(g, 0.0f + w[q][t].x, acc[0]);
                acc[1] = fmaf(g, 0.0f + w[q][t].y, acc[1]);
                acc[2] = fmaf(g, 0.0f + w[q][t].z, acc[2]);
                acc[3] = fmaf(g, 0.0f + w[q][t].w, acc[3]);
            }
            __stcs(reinterpret_cast<float4*>(a.out + static_cast<int64_t>(b) * a.out_dim + c0),
                   make_float4(acc[0], acc[1], acc[2], acc[3]));
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int c0 = blockIdx.x * kCbCols + (q * 256 + threadIdx.x) * 4;
        if (c0 >= a.out_dim) break;
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int t = 0; t < k; ++t) {
            const int64_t pos = s_row[t];
            if (pos < 0) continue;
            float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int sp = 0; sp < ns; ++sp) {
                const float4 w = *reinterpret_cast<const float4*>(a.y + sp * a.split_stride + pos * a.out_dim + c0);
                v[0] += w.x; v[1] += w.y; v[2] += w.z; v[3] += w.w;
            }
            const float g = s_gate[t];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fmaf(g, v[j], acc[j]);
        }
        for (int sh = 0; sh < a.num_shared; ++sh) {
            const int64_t r = sh0 + static_cast<int64_t>(sh) * a.batch + b;
            float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int sp = 0; sp < nsh; ++sp) {
                const float4 w = *reinterpret_cast<const float4*>(a.ysh + sp * a.sh_split_stride + r * a.out_dim + c0);
                v[0] += w.x; v[1] += w.y; v[2] += w.z; v[3] += w.w;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] += v[j];
        }
        *reinterpret_cast<float4*>(a.out + static_cast<int64_t>(b) * a.out_dim + c0) =
            make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream) {
    if (a.batch > 64 && (a.out_dim & 3) == 0 && a.top_k <= 64) {
        max_carveout(combine_rows_kernel);
        return launch_maybe_pdl(combine_rows_kernel, dim3((a.out_dim + kCbCols - 1) / kCbCols, a.batch), dim3(256), 0,
                                stream, a);
    }
    // small batches: narrow CTAs so the split partials are read by many SMs
    const int threads = a.batch <= 16 ? 64 : 256;
    dim3 grid((a.out_dim + 4 * threads - 1) / (4 * threads), a.batch);
    max_carveout(combine_kernel);
    return launch_maybe_pdl(combine_kernel, grid, dim3(threads), 0, stream, a);
}

cudaError_t launch_gather_tokens(const GatherArgs& a, cudaStream_t stream) {
    if (a.batch <= 0) return cudaSuccess;
    if (a.top_k + 1 > kGatherMaxDest) return cudaErrorInvalidValue;
    const size_t smem = sizeof(float) * static_cast<size_t>(a.use_z ? a.top_k * a.rank : 0);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(gather_tokens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    max_carveout(gather_tokens_kernel);
    return launch_maybe_pdl(gather_tokens_kernel, dim3(a.batch), dim3(kGatherThreads), smem, stream, a);
}

cudaError_t launch_unpack(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count, uint32_t* out,
                          int32_t* err_flag, cudaStream_t stream) {
    const int64_t blocks = count > 0 ? (count + 255) / 256 : 1;
    unpack_kernel<<<static_cast<unsigned>(blocks < 65535 ? blocks : 65535), 256, 0, stream>>>(bytes, nbytes, bits,
                                                                                                count, out, err_flag);
    return cudaGetLastError();
}

// Expert-parallel receive side, fixed-capacity slabs: work units built on the device
// from the received per-(source, local expert) row counts -- no host round trip.
// Source s's rows start at s * slab, its experts' rows follow each other in expert
// order; every (segment, m-block, token tile) becomes one Unit, in segment order.
__global__ void __launch_bounds__(1024) ep_units_kernel(const int32_t* __restrict__ counts, int n_src, int e_stride,
                                                       int n_local, int slab, int mb_count, int bn, int kc_end,
                                                       int n_ext, Unit* __restrict__ units, int32_t* __restrict__ n_units) {
    __shared__ int s_nu[1024];
    const int nseg = n_src * n_local;
    const int t = threadIdx.x;
    int r0 = 0, cnt = 0, nu = 0, s = 0, j = 0;
    if (t < nseg) {
        s = t / n_local;
        j = t % n_local;
        r0 = s * slab;
        for (int jj = 0; jj < j; ++jj) r0 += counts[s * e_stride + jj];
        cnt = counts[s * e_stride + j];
        nu = mb_count * ((cnt + bn - 1) / bn);
    }
    s_nu[t] = nu;
    __syncthreads();
    // inclusive scan (Hillis-Steele) of the unit counts
    for (int off = 1; off < 1024; off <<= 1) {
        const int v = t >= off ? s_nu[t - off] : 0;
        __syncthreads();
        s_nu[t] += v;
        __syncthreads();
    }
    const int base = s_nu[t] - nu;
    if (t == 1023) *n_units = s_nu[1023];
    int u = base;
    for (int t0 = 0; t0 < cnt; t0 += bn)
        for (int mb = 0; mb < mb_count; ++mb) {
            Unit un{};
            un.weight = j;
            un.mb = mb;
            un.x_row = r0 + t0;
            un.n_tok = min(bn, cnt - t0);
            un.y_row = un.x_row;
            un.kc_begin = 0;
            un.kc_end = static_cast<int16_t>(kc_end);
            un.n_ext = static_cast<int16_t>(n_ext);
            un.split = 0;
            units[u++] = un;
        }
}

cudaError_t launch_ep_units(const int32_t* counts, int n_src, int e_stride, int n_local, int slab, int mb_count, int bn,
                            int kc_end, int n_ext, Unit* units, int32_t* n_units, cudaStream_t stream) {
    if (n_src * n_local > 1024) return cudaErrorInvalidValue;
    ep_units_kernel<<<1, 1024, 0, stream>>>(counts, n_src, e_stride, n_local, slab, mb_count, bn, kc_end, n_ext, units,
                                            n_units);
    return cudaGetLastError();
}

// The f64 exp of the routers' softmax (route_pick / route_tile_kernel, moe.cpp:72
// std::exp) on arbitrary arguments: the hook the exp-vs-glibc parity test drives.
__global__ void exp_f64_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ y) {
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[t] = tq_exp::exp(x[t]);
}

cudaError_t launch_exp_f64(const double* x, int64_t n, double* y, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    exp_f64_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, stream>>>(x, n, y);
    return cudaGetLastError();
}


// Load-time repack on the device: the artifact's LSB-first packed
// code stream (codec.cpp:145-195) -> the engine's [mb][kc] super-word blocks,
// one thread per (m-block, K chunk, half, row): it gathers its row's 32 codes
// and writes them as `bits` super-words, the layout dequant32<b> decodes
// (tests/test_gpu_parity.py::test_repacked_codes_bit_exact reads it back).
__device__ __forceinline__ void pack_superword_dev(const uint32_t* c, int bits, uint32_t* w) {
    for (int j = 0; j < bits; ++j) w[j] = 0;
    if (bits == 2) {
        for (int j = 0; j < 2; ++j)
            for (int m = 0; m < 8; ++m) {
                const int p = 8 * j + m;
                w[j] |= (c[2 * p] << (2 * m)) | (c[2 * p + 1] << (16 + 2 * m));
            }
    } else if (bits == 3) {
        for (int j = 0; j < 3; ++j)
            for (int m = 0; m < 5; ++m) {
                const int p = 5 * j + m;
                w[j] |= (c[2 * p] << (3 * m)) | (c[2 * p + 1] << (16 + 3 * m));
            }
        for (int k = 0; k < 3; ++k) w[k] |= (((c[30] >> k) & 1u) << 15) | (((c[31] >> k) & 1u) << 31);
    } else if (bits == 4) {
        for (int j = 0; j < 4; ++j)
            for (int m = 0; m < 4; ++m) {
                const int p = 4 * j + m;
                w[j] |= (c[2 * p] << (4 * m)) | (c[2 * p + 1] << (16 + 4 * m));
            }
    } else {
        for (int j = 0; j < 8; ++j)
            for (int m = 0; m < 2; ++m) {
                const int p = 2 * j + m;
                w[j] |= (c[2 * p] << (8 * m)) | (c[2 * p + 1] << (16 + 8 * m));
            }
    }
}

__global__ void repack_codes_kernel(const uint8_t* __restrict__ packed, int64_t nbytes, int bits, int64_t o,
                                    int64_t i, int64_t mb_count, int64_t kc_total, uint8_t* __restrict__ out) {
    const int64_t n = mb_count * kc_total * 2 * kBM;
    const int blk = code_block_bytes(bits);
    const uint32_t mask = (1u << bits) - 1u;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int rl = static_cast<int>(t % kBM);
        const int h = static_cast<int>((t / kBM) % 2);
        const int64_t kc = (t / (2 * kBM)) % kc_total, mb = t / (2 * kBM * kc_total);
        const int64_t row = mb * kBM + rl, col0 = kc * kKC + 32 * h;
        uint32_t c[32];
        for (int q = 0; q < 32; ++q) {
            const int64_t col = col0 + q;
            uint32_t v = 0u;
            if (row < o && col < i) {
                const int64_t bit = (row * i + col) * bits, byte = bit >> 3;
                uint32_t two = packed[byte];
                if (byte + 1 < nbytes) two |= static_cast<uint32_t>(packed[byte + 1]) << 8;
                v = (two >> (bit & 7)) & mask;
            }
            c[q] = v;
        }
        uint32_t w[8];
        pack_superword_dev(c, bits, w);
        uint32_t* block = reinterpret_cast<uint32_t*>(out + (mb * kc_total + kc) * blk);
        for (int j = 0; j < bits; ++j) block[(h * bits + j) * kBM + rl] = w[j];
    }
}

cudaError_t launch_repack_codes(const uint8_t* packed, int64_t nbytes, int bits, int64_t o, int64_t i,
                                int64_t mb_count, int64_t kc_total, uint8_t* out, cudaStream_t stream) {
    const int64_t n = mb_count * kc_total * 2 * kBM;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    repack_codes_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(packed, nbytes, bits, o, i, mb_count,
                                                                           kc_total, out);
    return cudaGetLastError();
}

cudaError_t launch_export_codes(const uint8_t* wcodes, int bits, int kc_total, int out_dim, int in_dim,
                                uint32_t* out, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(out_dim) * kc_total * 2;
    export_codes_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(wcodes, bits, kc_total, out_dim,
                                                                                     in_dim, out);
    return cudaGetLastError();
}

cudaError_t launch_dec_route(const DecRouteArgs& a, cudaStream_t stream) {
    if (a.batch <= 0) return cudaSuccess;
    if (a.num_experts > 64 || a.top_k > kDecMaxTopK || a.top_k + a.num_shared > kDecMaxTopK + 64 || a.groups > 64 ||
        a.rank > 64)
        return cudaErrorInvalidValue;
    const int nslices = a.given ? 0 : (a.num_experts + kRouteExperts - 1) / kRouteExperts;
    const int ny = nslices + a.num_q * ((a.rank + kProjRows - 1) / kProjRows);
    if (ny < 1) return cudaErrorInvalidValue;
#ifndef TQ_ROUTE_NO256
    if (a.batch * ny > 2 * 148) {
        max_carveout(dec_route_kernel<256>);
        return launch_maybe_pdl(dec_route_kernel<256>, dim3(a.batch, ny), dim3(256), 0, stream, a);
    }
#endif
    max_carveout(dec_route_kernel<kDecRT>);
    return launch_maybe_pdl(dec_route_kernel<kDecRT>, dim3(a.batch, ny), dim3(kDecRT), 0, stream, a);
}

cudaError_t launch_dec_combine(const DecCombineArgs& a, cudaStream_t stream) {
    if (a.batch <= 0) return cudaSuccess;
    if (a.top_k > 64) return cudaErrorInvalidValue;
    max_carveout(dec_combine_kernel);
    return launch_maybe_pdl(dec_combine_kernel, dim3((a.out_dim + 1023) / 1024, a.batch), dim3(256), 0, stream, a);
}

}  // namespace tqb
