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
// loop.  We sum in parallel (vectorised, several accumulators, warp tree) and
// bound |ours - reference| <= 2 * gamma_{i+i/32+8} * sum|p|; when both ends of
// that interval round to the same f32, the f32 score is certified identical to
// the reference's, otherwise lane 0 replays the sequential loop (rare).  Then
// f64 max-subtracted softmax, total summed k = 0..K-1, order by (prob desc,
// index asc), gates = float(prob / selected) -- moe.cpp:64-87 step by step.
template <int TPB>
__global__ void __launch_bounds__(256) route_kernel(const float* __restrict__ x, int batch, int in_dim,
                                                   const float* __restrict__ gate, int num_experts, int top_k,
                                                   int group_size, int groups, int k_pad,
                                                   int32_t* __restrict__ ids, float* __restrict__ gates,
                                                   __half* __restrict__ x16, float* __restrict__ sx) {
    extern __shared__ __align__(16) float rs_smem[];
    float* xs = rs_smem;                          // TPB x in_dim
    float* scores = rs_smem + TPB * in_dim;       // TPB x num_experts
    const int b0 = blockIdx.x * TPB;
    const int nt = min(TPB, batch - b0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int t = 0; t < nt; ++t) {
        const float* xb = x + static_cast<int64_t>(b0 + t) * in_dim;
        for (int c = threadIdx.x; c < in_dim; c += blockDim.x) xs[t * in_dim + c] = xb[c];
    }
    __syncthreads();
    // fp16 activations (zero-padded to k_pad) and per-group sums of them
    for (int t = 0; t < nt; ++t) {
        const float* xr = xs + t * in_dim;
        if (x16) {
            __half* xo = x16 + static_cast<int64_t>(b0 + t) * k_pad;
            for (int c = threadIdx.x; c < k_pad; c += blockDim.x) xo[c] = __float2half_rn(c < in_dim ? xr[c] : 0.0f);
        }
        for (int g = warp; sx && g < groups; g += nwarps) {
            float acc = 0.0f;
            const int c0 = g * group_size, c1 = min(in_dim, c0 + group_size);
            for (int c = c0 + lane; c < c1; c += 32) acc += __half2float(__float2half_rn(xr[c]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
            if (lane == 0) sx[static_cast<int64_t>(b0 + t) * groups + g] = acc;
        }
    }
    if (num_experts == 0) return;  // activations-only prep (tq_forward with given routing)
    // certified scores
    const bool vec = (in_dim & 3) == 0;
    for (int k = warp; k < num_experts; k += nwarps) {
        const float* gk = gate + static_cast<int64_t>(k) * in_dim;
        double s[TPB], a[TPB];
#pragma unroll
        for (int t = 0; t < TPB; ++t) s[t] = a[t] = 0.0;
        if (vec) {
#pragma unroll 4
            for (int c = 4 * lane; c + 3 < in_dim; c += 128) {
                const float4 g4 = __ldg(reinterpret_cast<const float4*>(gk + c));
#pragma unroll
                for (int t = 0; t < TPB; ++t) {
                    if (t < nt) {
                        const float4 x4 = *reinterpret_cast<const float4*>(xs + t * in_dim + c);
                        const double p0 = static_cast<double>(x4.x) * g4.x, p1 = static_cast<double>(x4.y) * g4.y;
                        const double p2 = static_cast<double>(x4.z) * g4.z, p3 = static_cast<double>(x4.w) * g4.w;
                        s[t] += (p0 + p1) + (p2 + p3);
                        a[t] += (fabs(p0) + fabs(p1)) + (fabs(p2) + fabs(p3));
                    }
                }
            }
        } else {
            for (int cc = lane; cc < in_dim; cc += 32) {
                const float gv = gk[cc];
#pragma unroll
                for (int t = 0; t < TPB; ++t)
                    if (t < nt) {
                        const double p = static_cast<double>(xs[t * in_dim + cc]) * gv;
                        s[t] += p;
                        a[t] += fabs(p);
                    }
            }
        }
#pragma unroll
        for (int t = 0; t < TPB; ++t) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                s[t] += __shfl_down_sync(0xffffffffu, s[t], off);
                a[t] += __shfl_down_sync(0xffffffffu, a[t], off);
            }
        }
        // certification (lane 0 holds the sums); replay undecided scores
        const double u = 1.1102230246251565e-16;  // 2^-53
        const double nterms = 2.0 * (static_cast<double>(in_dim) + static_cast<double>(in_dim) / 32.0 + 8.0);
        unsigned undecided = 0;
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < TPB; ++t) {
                if (t >= nt) continue;
                const double err = __dmul_ru(__dmul_ru(nterms * u, 1.01), __dmul_ru(a[t], 1.0001));
                const float lo = __double2float_rn(__dsub_rd(s[t], err));
                const float hi = __double2float_rn(__dadd_ru(s[t], err));
                if (lo == hi) scores[t * num_experts + k] = __double2float_rn(s[t]);
                else undecided |= 1u << t;
            }
        }
        undecided = __shfl_sync(0xffffffffu, undecided, 0);
        while (undecided) {
            // the reference's exact sequential loop (matrix.cpp:29-34) for token t:
            // the warp streams the gate row through a per-warp smem window, lane 0 adds
            const int t = __ffs(undecided) - 1;
            undecided &= undecided - 1;
            // products are exact in f64, so the warp forms them; lane 0 keeps the sequential adds
            double* win = reinterpret_cast<double*>(rs_smem + ((TPB * (in_dim + num_experts) + 1) & ~1)) + warp * 64;
            const float* xr = xs + t * in_dim;
            double acc = 0.0;
            for (int c0 = 0; c0 < in_dim; c0 += 64) {
                __syncwarp();
                for (int j = lane; j < 64 && c0 + j < in_dim; j += 32)
                    win[j] = static_cast<double>(xr[c0 + j]) * static_cast<double>(gk[c0 + j]);
                __syncwarp();
                if (lane == 0) {
                    const int n = min(64, in_dim - c0);
                    for (int q = 0; q < n; ++q) acc = __dadd_rn(acc, win[q]);
                }
            }
            if (lane == 0) scores[t * num_experts + k] = __double2float_rn(acc);
        }
    }
    __syncthreads();
    for (int t = warp; t < nt; t += nwarps) {
        const float* sc = scores + t * num_experts;
        const int b = b0 + t;
        double mx = -INFINITY;
        for (int k = lane; k < num_experts; k += 32) mx = fmax(mx, static_cast<double>(sc[k]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        // every lane computes the total in the reference order k = 0..K-1
        double total = 0.0;
        for (int k = 0; k < num_experts; ++k) total = __dadd_rn(total, exp(static_cast<double>(sc[k]) - mx));
        double selected = 0.0;
        int picked[64];
        double pprob[64];
        for (int tt = 0; tt < top_k; ++tt) {
            double best_p = -1.0;
            int best_k = 0x7fffffff;
            for (int k = lane; k < num_experts; k += 32) {
                bool taken = false;
                for (int q = 0; q < tt; ++q) taken |= (picked[q] == k);
                if (taken) continue;
                const double pk = __ddiv_rn(exp(static_cast<double>(sc[k]) - mx), total);
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
            picked[tt] = best_k;
            pprob[tt] = best_p;
            selected = __dadd_rn(selected, best_p);
        }
        if (lane == 0) {
            for (int tt = 0; tt < top_k; ++tt) {
                ids[static_cast<int64_t>(b) * top_k + tt] = picked[tt];
                gates[static_cast<int64_t>(b) * top_k + tt] = __double2float_rn(__ddiv_rn(pprob[tt], selected));
            }
        }
    }
}

// =============================================================================
// plan: stable permutation + work-unit tables (single CTA)
// =============================================================================


constexpr int kPlanThreads = 1024;

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const PlanArgs a) {
    extern __shared__ int32_t pl_smem[];
    const int K = a.num_experts;
    int32_t* cnt = pl_smem;                // [32][K]
    int32_t* tot = pl_smem + 32 * K;       // [K+1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = a.batch * a.top_k;
    for (int t = threadIdx.x; t < 32 * K; t += blockDim.x) cnt[t] = 0;
    __syncthreads();
    const int per = (n + 31) / 32;
    const int f0 = warp * per, f1 = min(n, f0 + per);
    // phase 1: per-warp counts (warp-private rows, no atomics)
    for (int base = f0; base < f1; base += 32) {
        const int f = base + lane;
        const bool act = f < f1;
        int id = act ? a.ids[f] : -1;
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
        for (int w = 0; w < 32; ++w) s += cnt[w * K + threadIdx.x];
        tot[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int e = 0; e < K; ++e) {
            const int c = tot[e];
            tot[e] = run;
            run += c;
        }
        tot[K] = run;
    }
    __syncthreads();
    if (threadIdx.x <= K) a.offsets[threadIdx.x] = tot[threadIdx.x];
    if (threadIdx.x < K) {
        int run = tot[threadIdx.x];
        for (int w = 0; w < 32; ++w) {
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
        int id = act ? a.ids[f] : -1;
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
    __shared__ int32_t s_nsplit;
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
        int best = 1;
        float best_score = -1.0f;
        const int cap = a.main_kc ? max(1, min(a.nsplit, a.kc_total)) : 1;
        for (int ns = 1; ns <= cap; ++ns) {
            const long units = base * ns;
            const long rounds = (units + a.num_sms - 1) / a.num_sms;
            const float eff = rounds > 0 ? static_cast<float>(units) / static_cast<float>(rounds * a.num_sms) : 1.0f;
            const float score = eff - 0.01f * ns;
            if (score > best_score + 1e-6f) {
                best_score = score;
                best = ns;
            }
        }
        s_nsplit = best;
        if (a.nsplit_out) *a.nsplit_out = best;
    }
    __syncthreads();
    const int ns = s_nsplit;
    const int routed_units = s_tiles[n_local] * a.mb_count * ns;
    const int shared_units = a.num_shared * sh_tiles * a.mb_count * ns;
    const int total = routed_units + shared_units;
    for (int u = threadIdx.x; u < total; u += blockDim.x) {
        Unit un;
        int sp = u % ns;
        int rest = u / ns;
        if (u < routed_units) {
            // rest = (tile-global index) over (e, mb, tile): ordered e, mb, tile
            // find expert: units of expert t = (s_tiles[t+1]-s_tiles[t]) * mb_count
            int lo = 0, hi = n_local;  // s_tiles[lo]*mb <= rest < s_tiles[hi]*mb
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_tiles[mid] * a.mb_count <= rest) lo = mid; else hi = mid;
            }
            const int t = lo;
            const int within = rest - s_tiles[t] * a.mb_count;
            const int ntl = s_tiles[t + 1] - s_tiles[t];
            const int mb = within / ntl, tl = within % ntl;
            const int e = a.e_begin + t;
            const int ne = tot[e + 1] - tot[e];
            un.weight = t;
            un.mb = mb;
            un.x_row = tot[e] + tl * bn;
            un.n_tok = min(bn, ne - tl * bn);
            un.y_row = un.x_row;
        } else {
            rest -= s_tiles[n_local] * a.mb_count;
            const int s = rest / (sh_tiles * a.mb_count);
            const int within = rest % (sh_tiles * a.mb_count);
            const int mb = within / sh_tiles, tl = within % sh_tiles;
            un.weight = n_local + s;
            un.mb = mb;
            un.x_row = n_slots + tl * bn;
            un.n_tok = min(bn, a.batch - tl * bn);
            un.y_row = n_slots + s * a.batch + tl * bn;
        }
        un.kc_begin = static_cast<int16_t>(a.main_kc ? sp * a.kc_total / ns : 0);
        un.kc_end = static_cast<int16_t>(a.main_kc ? (sp + 1) * a.kc_total / ns : 0);
        un.n_ext = static_cast<int16_t>(sp == ns - 1 ? a.n_ext : 0);
        un.split = static_cast<int16_t>(sp);
        un.pad = 0;
        a.units[u] = un;
    }
    if (threadIdx.x == 0) *a.n_units = total;
    // projection pass units: stacked projection weight (index 0) x all tokens
    if (a.proj_mb > 0) {
        const int tiles = (a.batch + bn - 1) / bn;
        const int np = a.proj_mb * tiles * a.proj_nsplit;
        for (int u = threadIdx.x; u < np; u += blockDim.x) {
            const int sp = u % a.proj_nsplit;
            const int rest = u / a.proj_nsplit;
            const int mb = rest / tiles, tl = rest % tiles;
            Unit un;
            un.weight = 0;
            un.mb = mb;
            un.x_row = tl * bn;
            un.n_tok = min(bn, a.batch - tl * bn);
            un.y_row = tl * bn;
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

// =============================================================================
// gather: permuted fp16 activation rows + extension rows
// =============================================================================


__global__ void __launch_bounds__(256) gather_kernel(const GatherArgs a) {
    const int n_slots = a.offsets[a.num_experts];
    const int rows = n_slots + (a.with_shared ? a.batch : 0);
    const int row = blockIdx.x;
    if (row >= rows) return;
    int b, e = -1;
    if (row < n_slots) {
        const int f = a.perm[row];
        b = f / a.top_k;
        e = a.ids[f];
    } else {
        b = row - n_slots;
    }
    // activation row: 16-byte vector copy
    const int4* src = reinterpret_cast<const int4*>(a.x16 + static_cast<int64_t>(b) * a.k_pad);
    int4* dst = reinterpret_cast<int4*>(a.xp + static_cast<int64_t>(row) * a.k_pad);
    for (int t = threadIdx.x; t < a.k_pad / 8; t += blockDim.x) dst[t] = src[t];
    // extension row: [Sx | zscale * sum_splits(Z) * rowscale | 0]
    __half* er = a.ep + static_cast<int64_t>(row) * a.ext_cols;
    for (int col = threadIdx.x; col < a.ext_cols; col += blockDim.x) {
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
        er[col] = __float2half_rn(v);
    }
}

// =============================================================================
// combine: y[b] = sum_t g_bt * Y[inv(b,t)] + sum_s Yshared_s[b]
// =============================================================================


__global__ void __launch_bounds__(256) combine_kernel(const CombineArgs a) {
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
            const int pos = a.inv[f];
            if (pos < 0) continue;  // invalid expert id (reported through the error flag)
            float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int sp = 0; sp < ns; ++sp)
                load4(a.y + sp * a.split_stride + static_cast<int64_t>(pos) * a.out_dim + c0, v);
            const float g = a.gates[f];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fmaf(g, v[j], acc[j]);
        }
    }
    const int64_t sh0 = a.sh_from_offsets ? n_slots : 0;
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
// launch wrappers (called from tq_runtime.cpp)
// =============================================================================

cudaError_t launch_route(const float* x, int batch, int in_dim, const float* gate, int num_experts, int top_k,
                         int group_size, int groups, int k_pad, int32_t* ids, float* gates, __half* x16,
                         float* sx, cudaStream_t stream) {
    // tokens per CTA: share each gate row across several tokens at prefill,
    // spread tokens over many CTAs at decode
    int tpb = batch <= 32 ? 1 : (batch <= 1024 ? 2 : 8);
    while (tpb > 1 && sizeof(float) * static_cast<size_t>(tpb) * (in_dim + num_experts) > 160 * 1024) tpb >>= 1;
    const size_t smem = sizeof(float) * (static_cast<size_t>(tpb) * (in_dim + num_experts) + 2) + 8 * 64 * sizeof(double);
    const int grid = (batch + tpb - 1) / tpb;
    auto go = [&](auto kern) -> cudaError_t {
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        kern<<<grid, 256, smem, stream>>>(x, batch, in_dim, gate, num_experts, top_k, group_size, groups, k_pad,
                                          ids, gates, x16, sx);
        return cudaGetLastError();
    };
    if (tpb == 8) return go(route_kernel<8>);
    if (tpb == 4) return go(route_kernel<4>);
    if (tpb == 2) return go(route_kernel<2>);
    return go(route_kernel<1>);
}

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream) {
    const size_t smem = sizeof(int32_t) * (32 * static_cast<size_t>(a.num_experts) + a.num_experts + 1);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    plan_kernel<<<1, kPlanThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_gather(const GatherArgs& a, int max_rows, cudaStream_t stream) {
    if (max_rows <= 0) return cudaSuccess;
    gather_kernel<<<max_rows, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream) {
    dim3 grid((a.out_dim + 1023) / 1024, a.batch);
    combine_kernel<<<grid, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count, uint32_t* out,
                          int32_t* err_flag, cudaStream_t stream) {
    const int64_t blocks = count > 0 ? (count + 255) / 256 : 1;
    unpack_kernel<<<static_cast<unsigned>(blocks < 65535 ? blocks : 65535), 256, 0, stream>>>(bytes, nbytes, bits,
                                                                                                count, out, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_export_codes(const uint8_t* wcodes, int bits, int kc_total, int out_dim, int in_dim,
                                uint32_t* out, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(out_dim) * kc_total * 2;
    export_codes_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(wcodes, bits, kc_total, out_dim,
                                                                                     in_dim, out);
    return cudaGetLastError();
}

}  // namespace tqb
