// Decode-path fused expert GEMM (launch 2 of 3): persistent, warp-specialised
// tcgen05 kernel over the routed slots of ONE forward,
//
//   Y[slot rows, 128 weight rows] (fp32, TMEM) = sum_k  A_k (fp16, TMEM) * X_k^T (fp16, SMEM)
//
// per segment = (weight w, token tile, 128-row m-block).  A segment's steps are
//   nmain main steps: 128 K of packed b-bit codes + the fp16 scale slice,
//                     dequantized in registers (code * s', one HFMA2 per pair)
//                     and stored straight into TMEM (tcgen05.st);
//   n_ep ext pieces:  32 columns of the dense fp16 extension block
//                     [-zero * s' per group | U_p codes] against the extension
//                     rows [Sx | (X.A_q) * zscale] -- the zero-point correction
//                     and the rank-r tile correction (infer.cpp:158-174) in the
//                     SAME accumulator.
// Work split: every CTA derives the segment list from the per-expert slot counts
// and takes a contiguous range of the flattened step list (stream-K), so the
// per-segment pipeline cost is paid ~once per CTA; a segment cut by a CTA
// boundary is summed by its last-arriving CTA in fixed CTA order
// (deterministic, no float atomics).
//
// Warp roles (736 threads):
//   0..15   dequant: 2 groups of 8 warps; group g takes the CTA's steps j = g mod 2;
//           warps q and q+4 of a group share TMEM lane quarter q and split the
//           step's columns
//   16..19  epilogue: tcgen05.ld -> scale -> expert rows (or split partials)
//   20      producer (+ TMEM allocator): bulk copies of codes / ext pieces and the
//           activation tiles
//   21, 22  MMA issuers: issuer i takes steps j = i mod 2, own accumulator
//           columns (a single issuing thread sustains one M128 K16 MMA per ~56
//           cycles for N <= 64 -- tools/micro/mma_tput.cu -- so one stream
//           cannot keep up with HBM)
//
// Ring protocol, correct by construction: every ring (code stages S, activation
// stages SX, A stages KAS in TMEM, accumulator buffers) is consumed in CTA step
// order and S, SX, KAS are multiples of the number of consumer streams (2), so
// a consumer of ring slot x always consumed x's previous phase itself: no parity
// wait can run ahead by two phases, whatever the relative speed of the groups
// and issuers.
#include <cstdint>
#include <cstdio>

#include "tq_internal.h"
#include "tq_ptx.cuh"

namespace tqb {

namespace {

constexpr int kNG = 2;                 // dequant groups
constexpr int kNI = 2;                 // MMA issue streams
constexpr int kEpi0 = 16;              // first epilogue warp (lane quarter = warp % 4)
constexpr int kProd = 20;
constexpr int kMma0 = 21;
constexpr int kThreads = 23 * 32;
constexpr int kMaxCS = 32, kMaxXS = 16;
constexpr int kPieceCols = 32;                          // ext piece width (K)
constexpr int kPieceBytes = kBM * kPieceCols * 2;       // 8 KB
constexpr int kSmemBudget = 227 * 1024;
constexpr int kHdrBytes = 4096;

__host__ __device__ constexpr int dec_kas(int dn) { return dn <= 32 ? 6 : 4; }   // TMEM: kas * 64 + 2 * kNI * dn <= 512

struct Hdr {
    uint64_t c_full[kMaxCS], c_empty[kMaxCS];
    uint64_t x_full[kMaxXS], x_empty[kMaxXS];
    uint64_t a_full[8], a_empty[8];
    uint64_t d_full[2], d_empty[2];
    uint32_t tmem_base;
    int last_flag;
    int n_wt;                          // weight tiles (segments per m-block)
    int wt_first[kDecMaxW + 1];        // first weight-tile index of weight w
    int n_rows[kDecMaxW];              // rows (slots) of weight w
};
static_assert(sizeof(Hdr) <= kHdrBytes, "decode header");

struct Seg {
    int s, w, mb, row0, n_tok, n_pad;
};

template <int DN>
__device__ __forceinline__ Seg seg_info(const Hdr* h, const DecParams& p, int s) {
    Seg g;
    g.s = s;
    const int wt = s / p.mb_count;
    g.mb = s - wt * p.mb_count;
    int w = 0;
    while (h->wt_first[w + 1] <= wt) ++w;
    g.w = w;
    const int tile = wt - h->wt_first[w];
    g.n_tok = min(DN, h->n_rows[w] - tile * DN);
    g.row0 = w * p.cap8 + tile * DN;
    g.n_pad = (g.n_tok + 15) & ~15;
    return g;
}

__device__ __forceinline__ int64_t cta_start(int c, int64_t total, int grid) {
    return static_cast<int64_t>(c) * total / grid;
}
__device__ __forceinline__ int cta_of(int64_t x, int64_t total, int grid) {
    return static_cast<int>(((x + 1) * grid - 1) / total);
}

// the elected lane arms `bar` with `bytes` and issues up to 3 bulk copies into it
__device__ __forceinline__ void copy_group(uint64_t* bar, uint32_t bytes, void* d0, const void* s0, uint32_t n0,
                                           void* d1, const void* s1, uint32_t n1, void* d2, const void* s2,
                                           uint32_t n2) {
    if (elect_one()) {
        mbar_arrive_expect_tx(bar, bytes);
        if (n0) bulk_copy_g2s(d0, s0, n0, bar);
        if (n1) bulk_copy_g2s(d1, s1, n1, bar);
        if (n2) bulk_copy_g2s(d2, s2, n2, bar);
    }
    __syncwarp();
}

}  // namespace

template <int BITS, int DN>
__global__ void __launch_bounds__(kThreads, 1) dec_gemm_kernel(const __grid_constant__ DecParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    constexpr int KAS = dec_kas(DN);
    constexpr int kBlk = code_block_bytes(BITS);          // 128 x 64 codes
    constexpr int kWords = BITS;                          // u32 words per 32-code super-word
    constexpr int kHalf = kWords * kBM;                   // words per half block
    constexpr int kAccCol0 = KAS * 64;
    static_assert(kAccCol0 + 2 * kNI * DN <= 512, "TMEM budget");
    constexpr int kXStage = 2 * DN * 128;                  // two 64-column atoms of DN rows

    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t pad = (1024u - (raw & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    const uint32_t s_base = raw + pad;
    const int S = p.code_stages, SX = p.x_stages, SC = p.code_stage_bytes;
    const uint32_t x_off = static_cast<uint32_t>(S * SC);
    Hdr* h = reinterpret_cast<Hdr*>(smem + x_off + SX * kXStage);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&h->c_full[i], 1);
            mbar_init(&h->c_empty[i], 8);      // the 8 warps of the consuming dequant group
        }
        for (int i = 0; i < SX; ++i) {
            mbar_init(&h->x_full[i], 1);
            mbar_init(&h->x_empty[i], 1);      // tcgen05.commit of the issuer
        }
        for (int i = 0; i < KAS; ++i) {
            mbar_init(&h->a_full[i], 8);
            mbar_init(&h->a_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&h->d_full[i], kNI);
            mbar_init(&h->d_empty[i], 4);
        }
        fence_barrier_init();
    } else if (threadIdx.x == 32) {
        // segment table from the slot counts of this forward: weights w < K are the
        // routed experts (cnt[w] slots), then the shared experts (batch rows each)
        const int W = p.num_experts + p.num_shared;
        int acc = 0;
        for (int w = 0; w < W; ++w) {
            const int n = w < p.num_experts ? p.cnt[w] : p.batch;
            h->n_rows[w] = n;
            h->wt_first[w] = acc;
            acc += (n + DN - 1) / DN;
        }
        h->wt_first[W] = acc;
        for (int w = W + 1; w <= kDecMaxW; ++w) h->wt_first[w] = 0x7fffffff;
        h->n_wt = acc;
    }
    if (wid == kProd) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&h->tmem_base)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = h->tmem_base;

    const int steps_per_seg = p.nmain + p.n_ep;
    const int64_t total = static_cast<int64_t>(h->n_wt) * p.mb_count * steps_per_seg;
    const int G = gridDim.x;
    const int64_t g_begin = cta_start(blockIdx.x, total, G);
    const int64_t g_end = cta_start(blockIdx.x + 1, total, G);
    const int n_steps = static_cast<int>(g_end - g_begin);
    const int gshift = p.group_shift;

    if (n_steps > 0) {
        if (wid < 16) {
            // ===================== dequant groups =====================
            const int grp = wid >> 3;
            const int hw = (wid >> 2) & 1;                 // which half of the step's columns
            const int q = wid & 3;                         // TMEM lane quarter
            const int rloc = q * 32 + lane;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            int cs = grp, as = grp;
            uint32_t cph = 0, aph = 0;
            int64_t x = g_begin + grp;
            int s = static_cast<int>(x / steps_per_seg), k = static_cast<int>(x % steps_per_seg);
            for (int j = grp; j < n_steps; j += kNG) {
                mbar_wait(&h->c_full[cs], cph);
                const uint8_t* st = smem + cs * SC;
                if (k < p.nmain) {
                    // main step: 128 K = two 64-column code blocks; this warp dequantizes block hw
                    const int kb0 = 2 * k;
                    const int nat = min(2, p.kc64 - kb0);
                    uint32_t words[2][kWords];
                    uint16_t sbits[2];
                    if (hw < nat) {
                        const uint32_t* wst = reinterpret_cast<const uint32_t*>(st + hw * kBlk) + rloc;
                        const int e0 = kb0 * 64;                        // first K of the step
                        const int ein = gshift >= 0 ? (e0 & ((1 << gshift) - 1)) : e0 % p.group_size;
                        const uint16_t* sc = reinterpret_cast<const uint16_t*>(st + 2 * kBlk) + rloc;
#pragma unroll
                        for (int ss = 0; ss < 2; ++ss) {
#pragma unroll
                            for (int w = 0; w < kWords; ++w) words[ss][w] = wst[ss * kHalf + w * kBM];
                            const int off = ein + 64 * hw + 32 * ss;
                            const int gi = gshift >= 0 ? off >> gshift : off / p.group_size;
                            sbits[ss] = sc[gi * kBM];
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&h->c_empty[cs]);
                    mbar_wait(&h->a_empty[as], aph ^ 1u);
                    tc_fence_after();
                    if (hw < nat) {
#pragma unroll
                        for (int ss = 0; ss < 2; ++ss) {
                            uint32_t v[16];
                            const DqConst dq = make_dq(__ushort_as_half(sbits[ss]));
                            dequant32<BITS>(words[ss], dq, v);
                            tc_st_32x32b_x16(tmem + lane_base + as * 64 + (2 * hw + ss) * 16, v);
                        }
                        tc_wait_st();
                    }
                } else {
                    // ext piece: 32 dense fp16 columns = 16 u32 words per row; this warp moves 8
                    const uint32_t* eb = reinterpret_cast<const uint32_t*>(st) + rloc;
                    uint32_t v[8];
#pragma unroll
                    for (int w = 0; w < 8; ++w) v[w] = eb[(hw * 8 + w) * kBM];
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&h->c_empty[cs]);
                    mbar_wait(&h->a_empty[as], aph ^ 1u);
                    tc_fence_after();
                    tc_st_32x32b_x8(tmem + lane_base + as * 64 + hw * 8, v);
                    tc_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&h->a_full[as]);
                // next own step
                cs += kNG;
                if (cs >= S) { cs -= S; cph ^= 1u; }
                as += kNG;
                if (as >= KAS) { as -= KAS; aph ^= 1u; }
                k += kNG;
                while (k >= steps_per_seg) { k -= steps_per_seg; ++s; }
            }
        } else if (wid == kProd) {
            // ===================== producer =====================
            int cs = 0, xs = 0;
            uint32_t cph = 0, xph = 0;
            int s = static_cast<int>(g_begin / steps_per_seg), k = static_cast<int>(g_begin % steps_per_seg);
            Seg sg = seg_info<DN>(h, p, s);
            for (int j = 0; j < n_steps; ++j) {
                if (sg.s != s) sg = seg_info<DN>(h, p, s);
                const int64_t wm = static_cast<int64_t>(sg.w) * p.mb_count + sg.mb;
                uint8_t* cdst = smem + cs * SC;
                uint8_t* xdst = smem + x_off + xs * kXStage;
                mbar_wait(&h->c_empty[cs], cph ^ 1u);
                if (k < p.nmain) {
                    const int kb0 = 2 * k;
                    const int nat = min(2, p.kc64 - kb0);
                    const uint8_t* csrc = p.codes + (wm * p.kc64 + kb0) * kBlk;   // [w][mb][kb64] blocks
                    const int e0 = kb0 * 64;
                    int g0, g1;
                    if (gshift >= 0) {
                        g0 = e0 >> gshift;
                        g1 = (e0 + nat * 64 - 1) >> gshift;
                    } else {
                        g0 = e0 / p.group_size;
                        g1 = (e0 + nat * 64 - 1) / p.group_size;
                    }
                    g1 = min(p.groups - 1, g1);
                    const uint32_t cb = static_cast<uint32_t>(nat * kBlk);
                    const uint32_t sb = static_cast<uint32_t>(g1 - g0 + 1) * kBM * 2;
                    copy_group(&h->c_full[cs], cb + sb, cdst, csrc, cb, cdst + 2 * kBlk,
                               p.scales + (wm * p.groups + g0) * kBM, sb, nullptr, nullptr, 0);
                    mbar_wait(&h->x_empty[xs], xph ^ 1u);
                    const uint32_t xb = static_cast<uint32_t>(sg.n_pad) * 128u;
                    const __half* xa = p.xperm + (static_cast<int64_t>(kb0) * p.atom_rows + sg.row0) * 64;
                    copy_group(&h->x_full[xs], nat * xb, xdst, xa, xb, xdst + DN * 128, xa + p.atom_rows * 64,
                               nat > 1 ? xb : 0u, nullptr, nullptr, 0);
                } else {
                    const int piece = k - p.nmain;
                    const uint8_t* esrc = p.ext_blocks + wm * static_cast<int64_t>(p.n_ext64) * (2 * kPieceBytes) +
                                          static_cast<int64_t>(piece) * kPieceBytes;
                    copy_group(&h->c_full[cs], kPieceBytes, cdst, esrc, kPieceBytes, nullptr, nullptr, 0, nullptr,
                               nullptr, 0);
                    mbar_wait(&h->x_empty[xs], xph ^ 1u);
                    const uint32_t xb = static_cast<uint32_t>(sg.n_pad) * 128u;
                    const __half* ea = p.extperm + (static_cast<int64_t>(piece >> 1) * p.atom_rows + sg.row0) * 64;
                    copy_group(&h->x_full[xs], xb, xdst, ea, xb, nullptr, nullptr, 0, nullptr, nullptr, 0);
                }
                if (++cs == S) { cs = 0; cph ^= 1u; }
                if (++xs == SX) { xs = 0; xph ^= 1u; }
                if (++k == steps_per_seg) { k = 0; ++s; }
            }
        } else if (wid == kMma0 || wid == kMma0 + 1) {
            // ===================== MMA issuers =====================
            const int ii = wid - kMma0;
            int as = ii, xs = ii;
            uint32_t aph = 0, xph = 0;
            int64_t x = g_begin;                            // global step of the current part's start
            int m = 0;                                      // part ordinal (accumulator buffer m & 1)
            while (x < g_end) {
                const int s = static_cast<int>(x / steps_per_seg);
                const int64_t seg_end = static_cast<int64_t>(s + 1) * steps_per_seg;
                const int64_t pe = seg_end < g_end ? seg_end : g_end;
                const Seg sg = seg_info<DN>(h, p, s);
                const int buf = m & 1;
                mbar_wait(&h->d_empty[buf], ((m >> 1) & 1) ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem + kAccCol0 + (buf * kNI + ii) * DN;
                const uint32_t idesc = idesc_f16(static_cast<uint32_t>(sg.n_pad));
                // own steps of this part: local index j = x - g_begin, j = ii (mod 2)
                int64_t y = x + ((ii - (x - g_begin)) % kNI + kNI) % kNI;
                bool first = true;
                for (; y < pe; y += kNI) {
                    const int k = static_cast<int>(y - static_cast<int64_t>(s) * steps_per_seg);
                    mbar_wait(&h->a_full[as], aph);
                    mbar_wait(&h->x_full[xs], xph);
                    tc_fence_after();
                    const uint32_t xaddr = s_base + x_off + xs * kXStage;
                    const uint32_t a_tm = tmem + as * 64;
                    if (k < p.nmain) {
                        const int nat = min(2, p.kc64 - 2 * k);
                        tc_mma_ts_x4_elect(d_tmem, a_tm, sw128_desc(xaddr), idesc, first ? 0u : 1u);
                        if (nat > 1)
                            tc_mma_ts_x4_elect(d_tmem, a_tm + 32, sw128_desc(xaddr + DN * 128), idesc, 1u);
                    } else {
                        const int piece = k - p.nmain;
                        // 32-column slice (piece & 1) of the ext atom: start +64 B = +4 descriptor units
                        tc_mma_ts_x2_elect(d_tmem, a_tm, sw128_desc(xaddr) + static_cast<uint64_t>((piece & 1) * 4),
                                           idesc, first ? 0u : 1u);
                    }
                    tc_commit_elect(&h->a_empty[as]);
                    tc_commit_elect(&h->x_empty[xs]);
                    first = false;
                    as += kNI;
                    if (as >= KAS) { as -= KAS; aph ^= 1u; }
                    xs += kNI;
                    if (xs >= SX) { xs -= SX; xph ^= 1u; }
                }
                if (!first) tc_commit_elect(&h->d_full[buf]);
                else if (lane == 0) mbar_arrive(&h->d_full[buf]);
                __syncwarp();
                x = pe;
                ++m;
            }
        } else if (wid >= kEpi0 && wid < kEpi0 + 4) {
            // ===================== epilogue =====================
            const int q = wid & 3;
            int64_t x = g_begin;
            int m = 0;
            const int first_seg = static_cast<int>(g_begin / steps_per_seg);
            while (x < g_end) {
                const int s = static_cast<int>(x / steps_per_seg);
                const int64_t seg_begin = static_cast<int64_t>(s) * steps_per_seg;
                const int64_t seg_end = seg_begin + steps_per_seg;
                const int64_t pe = seg_end < g_end ? seg_end : g_end;
                const Seg sg = seg_info<DN>(h, p, s);
                const int buf = m & 1;
                const int npart = static_cast<int>(pe - x);
                const int j0 = static_cast<int>(x - g_begin);
                bool part[kNI];
#pragma unroll
                for (int ii = 0; ii < kNI; ++ii) part[ii] = npart >= kNI || ((ii - j0 % kNI + kNI) % kNI) < npart;
                const bool whole = x == seg_begin && pe == seg_end;
                const float oscale = p.w_outscale[sg.w];
                const int row = sg.mb * kBM + q * 32 + lane;
                const bool valid = row < p.o_valid;
                const int slot = s == first_seg ? 0 : 1;
                float* dst;
                int64_t ld;
                if (whole) {
                    dst = p.yslot + static_cast<int64_t>(sg.row0) * p.ldy + row;
                    ld = p.ldy;
                } else {
                    dst = p.scratch + (static_cast<int64_t>(blockIdx.x) * 2 + slot) * DN * kBM + q * 32 + lane;
                    ld = kBM;
                }
                mbar_wait_sleep(&h->d_full[buf], (m >> 1) & 1);
                tc_fence_after();
                const uint32_t dbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + kAccCol0 + buf * kNI * DN;
                for (int t0 = 0; t0 < sg.n_tok; t0 += 16) {
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = 0.0f;
#pragma unroll
                    for (int ii = 0; ii < kNI; ++ii) {   // fixed order: deterministic sum of the streams
                        if (!part[ii]) continue;
                        uint32_t w[16];
                        tc_ld_32x32b_x16(dbase + ii * DN + t0, w);
                        tc_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] += __uint_as_float(w[i]);
                    }
                    if (valid || !whole) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (t0 + i < sg.n_tok) dst[static_cast<int64_t>(t0 + i) * ld] = v[i] * oscale;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&h->d_empty[buf]);
                if (!whole) {
                    // split segment: the last CTA to finish its part sums all parts in CTA order
                    // (CTAs with an empty step range -- fewer steps than CTAs -- own no part)
                    const int c_a = cta_of(seg_begin, total, G), c_b = cta_of(seg_end - 1, total, G);
                    __threadfence();
                    named_bar_sync(1, 128);
                    if (q == 0 && lane == 0) {
                        int parts = 0;
                        for (int c = c_a; c <= c_b; ++c) parts += cta_start(c, total, G) < cta_start(c + 1, total, G);
                        const int old = atomicAdd(&p.seg_cnt[s], 1);
                        h->last_flag = old == parts - 1;
                        if (h->last_flag) p.seg_cnt[s] = 0;   // ready for the next launch
                    }
                    named_bar_sync(1, 128);
                    if (h->last_flag) {
                        __threadfence();
                        for (int t = 0; t < sg.n_tok; ++t) {
                            float acc = 0.0f;
                            for (int c = c_a; c <= c_b; ++c) {
                                if (cta_start(c, total, G) == cta_start(c + 1, total, G)) continue;
                                const int cslot = static_cast<int>(cta_start(c, total, G) / steps_per_seg) == s ? 0 : 1;
                                acc += __ldcg(p.scratch + ((static_cast<int64_t>(c) * 2 + cslot) * DN + t) * kBM + q * 32 + lane);
                            }
                            if (valid) p.yslot[static_cast<int64_t>(sg.row0 + t) * p.ldy + row] = acc;
                        }
                    }
                }
                x = pe;
                ++m;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (wid == kProd) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

// -----------------------------------------------------------------------------

int dec_code_stage_bytes(int bits) {
    const int main_bytes = 2 * code_block_bytes(bits) + (128 / 32 + 1) * kBM * 2;
    const int b = main_bytes > kPieceBytes ? main_bytes : kPieceBytes;
    return (b + 1023) / 1024 * 1024;
}

cudaError_t launch_decode(const DecParams& p0, int dn, int grid, cudaStream_t stream) {
    DecParams p = p0;
    if (dn != 32 && dn != 64) return cudaErrorInvalidValue;
    if (p.num_experts + p.num_shared > kDecMaxW) return cudaErrorInvalidValue;
    const int sc = dec_code_stage_bytes(p.bits);
    const int xst = 2 * dn * 128;
    // as many stages as fit: code stages (HBM latency) first, both counts even
    int xs = dn == 32 ? 8 : 6;
    int cs = (kSmemBudget - 1024 - kHdrBytes - xs * xst) / sc;
    cs = cs < kMaxCS ? cs : kMaxCS;
    cs &= ~1;
    if (cs < 4) return cudaErrorInvalidValue;
    p.code_stages = cs;
    p.x_stages = xs;
    p.code_stage_bytes = sc;
    p.group_shift = -1;
    for (int s = 0; s < 16; ++s)
        if ((1 << s) == p.group_size) p.group_shift = s;
    const int smem = 1024 + cs * sc + xs * xst + kHdrBytes;
    cudaError_t err = cudaSuccess;
    auto go = [&](auto kern) {
        static const void* done[16];
        static int n_done = 0;
        bool seen = false;
        for (int t = 0; t < n_done; ++t) seen |= done[t] == reinterpret_cast<const void*>(kern);
        if (!seen) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
            if (err != cudaSuccess) return;
            if (n_done < 16) done[n_done++] = reinterpret_cast<const void*>(kern);
        }
        err = launch_maybe_pdl(kern, dim3(grid), dim3(kThreads), smem, stream, p);
    };
#define TQ_DEC_CASES(DNV)                                           \
    switch (p.bits) {                                               \
        case 2: go(dec_gemm_kernel<2, DNV>); break;                 \
        case 3: go(dec_gemm_kernel<3, DNV>); break;                 \
        case 4: go(dec_gemm_kernel<4, DNV>); break;                 \
        case 8: go(dec_gemm_kernel<8, DNV>); break;                 \
        default: return cudaErrorInvalidValue;                      \
    }
    if (dn == 32) {
        TQ_DEC_CASES(32)
    } else {
        TQ_DEC_CASES(64)
    }
#undef TQ_DEC_CASES
    return err;
}

}  // namespace tqb
