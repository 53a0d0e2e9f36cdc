// Decode-path fused expert GEMM (launch 2 of 3): persistent, warp-specialised
// tcgen05 kernel over the routed slots of ONE forward,
//
//   Y[slot rows, 128 weight rows] (fp32, TMEM) = sum_k  A_k (fp16, TMEM) * X_k^T (fp16, SMEM)
//
// per segment = (weight w, token tile, 128-row m-block).  A segment's steps are
//   nmain main steps: 256 K (four 64-column atoms) of packed b-bit codes + the fp16
//                     scale slice, dequantized in registers (code * s', one HFMA2
//                     per pair) and stored straight into TMEM (tcgen05.st);
//   one ext step:     the dense fp16 extension block [-zero * s' per group | U_p
//                     codes] against the extension rows [Sx | (X.A_q) * zscale] --
//                     the zero-point correction and the rank-r tile correction
//                     (infer.cpp:158-174) in the SAME accumulators.
// Work split: every CTA derives the segment list from the per-expert slot counts
// and takes a contiguous range of the flattened step list (stream-K); a segment
// cut by a CTA boundary is summed by its last-arriving CTA in fixed CTA order
// (deterministic, no float atomics).
//
// Warp roles (896 threads) and why (tools/micro/*.cu, measured on B200):
//   0..3    MMA issuers (4 for 32-token tiles, 2 for 64): issuer i issues the K=16
//           MMAs of its atoms of every step into its own accumulator -- one issuing
//           warp sustains one M128 MMA per ~56 cycles whatever N <= 64
//           (mma_tput.cu, mma_acc.cu)
//   4, 5    code producers (steps j = p mod 2) -- one thread completes only ~1
//           bulk-copy stage per ~530 cycles (stream2.cu), so two issue in parallel
//   6, 7    activation producers (steps j = p mod 2), same reason
//   8..11   epilogue: tcgen05.ld of the accumulators -> expert rows / split partials
//   12..27  dequant: 2 groups of 8 warps; group g takes the CTA's steps j = g mod 2;
//           warps (h, q) cover TMEM lane quarter q and atoms 2h, 2h+1 of the step
//
// Ring protocol, correct by construction:
//   * every mbarrier ring is waited on by in-order waiters that consumed the
//     slot's previous phase themselves (the producers and dequant groups split the
//     steps by parity and the copy rings are even; each MMA issuer consumes every
//     step), or -- the A stages' "MMA done" -- whose phases complete in step order
//     (each issuer issues and commits in step order) and whose waiter observed an
//     earlier step's phase, so no parity wait can run two phases ahead;
//   * the accumulator hand-back (epilogue -> issuer) is a monotonic sequence
//     counter in shared memory (release / acquire), which cannot alias.
#include <cstdint>
#include <cstdio>

#include "tq_internal.h"
#include "tq_ptx.cuh"

// TQ_DEC_ABL (experiment builds only): 1 no activation copies, 2 no MMA, 4 no dequant
// arithmetic, 8 no code copies -- the ablations that locate the pipeline's limiter
#ifndef TQ_DEC_ABL
#define TQ_DEC_ABL 0
#endif

namespace tqb {

namespace {

// warp roles: the latency-critical single-thread roles at the LOWEST warp ids
// (the schedulers favour older warps: placed above the 16 dequant warps, the MMA
// issuers' loop took ~1000 cycles of waiting for issue slots per step)
constexpr int kMma0 = 0;                 // issuers 0.. (NI of them)
constexpr int kCProd = 4;                // code producers 4, 5
constexpr int kXProd = 6;                // activation producers 6, 7
constexpr int kEpi0 = 8;                 // epilogue 8..11 (lane quarter = warp % 4)
constexpr int kDq0 = 12;                 // dequant 12..27
constexpr int kMaxNI = 4;
constexpr int kThreads = 28 * 32;
constexpr int kAtomsPerStep = 4;         // 256 K per step
constexpr int kAS = 3;                   // A stages in TMEM (128 columns each)
#ifndef TQ_DEC_NI32
#define TQ_DEC_NI32 4
#endif
// MMA issuers per tile height: TMEM = kAS * 128 + NI * DN columns <= 512
__host__ __device__ constexpr int dec_ni(int dn) { return dn <= 32 ? TQ_DEC_NI32 : 2; }
constexpr int kMaxCS = 16, kMaxXS = 16;
constexpr int kSmemBudget = 227 * 1024;
constexpr int kHdrBytes = 4096;
constexpr int kExtAtomBytes = kBM * 64 * 2;   // dense fp16 128 x 64 block

struct Hdr {
    uint64_t c_full[kMaxCS], c_empty[kMaxCS];
    uint64_t x_full[kMaxXS], x_empty[kMaxXS];
    uint64_t a_full[kAS], a_empty[kAS];
    uint64_t d_full[kMaxNI];
    uint32_t epi_seq[kMaxNI];            // parts drained from issuer i's accumulator
    uint32_t tmem_base;
    int last_flag;
    int n_wt;                            // weight tiles (segments per m-block)
    int wt_first[kDecMaxW + 1];          // first weight-tile index of weight w
    int n_rows[kDecMaxW];                // rows (slots) of weight w
};
static_assert(sizeof(Hdr) <= kHdrBytes, "decode header");

struct Seg {
    int s, w, mb, row0, n_tok;
};

// TQ_DEC_CHECK builds: bounds checks that report and trap (compute-sanitizer is
// unavailable on the GPU pool)
#ifdef TQ_DEC_CHECK
#define DEC_CHECK(cond, ...)                                                            \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            printf("DEC_CHECK %s:%d cta %d thr %d: " #cond "\n", __FILE__, __LINE__,   \
                   blockIdx.x, threadIdx.x);                                            \
            printf(__VA_ARGS__);                                                        \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define DEC_CHECK(cond, ...) \
    do {                     \
    } while (0)
#endif

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
    DEC_CHECK(w < p.num_experts + p.num_shared && g.n_tok > 0 && g.row0 + g.n_tok <= (w + 1) * p.cap8 + 0 &&
                  g.mb < p.mb_count,
              "seg %d: w %d tile %d n_tok %d row0 %d mb %d cap8 %d n_rows %d\n", s, w, tile, g.n_tok, g.row0, g.mb,
              p.cap8, h->n_rows[w]);
    return g;
}

__device__ __forceinline__ int64_t cta_start(int c, int64_t total, int grid) {
    return static_cast<int64_t>(c) * total / grid;
}
__device__ __forceinline__ int cta_of(int64_t x, int64_t total, int grid) {
    return static_cast<int>(((x + 1) * grid - 1) / total);
}

__device__ __forceinline__ void seq_store_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t seq_load_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
// spin until *p >= target (monotonic counters: a waiter can never alias a later use)
// (backs off between polls: a spinning warp would take issue slots from the dequant warps)
__device__ __forceinline__ void seq_wait(const uint32_t* p, uint32_t target) {
    while (static_cast<int32_t>(seq_load_acquire(p) - target) < 0) __nanosleep(64);
}

// atoms of step k of a segment: main steps carry up to 4 code atoms, the ext step E64
__device__ __forceinline__ int step_atoms(const DecParams& p, int k) {
    return k < p.nmain ? min(kAtomsPerStep, p.kc64 - kAtomsPerStep * k) : p.n_ext64;
}

// TQ_DEC_TRACE builds: clock64 of pipeline events of CTA p.trace_cta into p.trace
// ([slot][1024] u64): 0 code issue, 1 x issue, 2 dequant data ready, 3 dequant done,
// 4 issuer A ready, 5 issuer X ready, 6 issuer committed, 7 epilogue part,
// 8 dequant A stage free, 9 issuer 3 committed
// per-CTA timeline (globaltimer ns): p.trace[8192 + cta * 4 + k], k = 0 entry, 1 prologue done,
// 2 roles done (before teardown), 3 exit
__device__ __forceinline__ void ctrace(const DecParams& p, int k) {
#ifdef TQ_DEC_TRACE
    if (threadIdx.x == 0 && p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[12288 + blockIdx.x * 4 + k] = t;
    }
#else
    (void)p;
    (void)k;
#endif
}
__device__ __forceinline__ void dtrace(const DecParams& p, int slot, int idx) {
#ifdef TQ_DEC_TRACE
    if (static_cast<int>(blockIdx.x) == p.trace_cta && idx < 1024 && slot < 10 && p.trace) p.trace[slot * 1024 + idx] = clock64();
#else
    (void)p;
    (void)slot;
    (void)idx;
#endif
}

}  // namespace

template <int BITS, int DN>
__global__ void __launch_bounds__(kThreads, 1) dec_gemm_kernel(const __grid_constant__ DecParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    ctrace(p, 0);
    constexpr int kBlk = code_block_bytes(BITS);          // 128 x 64 codes
    constexpr int kWords = BITS;                          // u32 words per 32-code super-word
    constexpr int kHalf = kWords * kBM;                   // words per half block
    constexpr int kNIss = dec_ni(DN);                     // MMA issuers
    constexpr int kAPI = kAtomsPerStep / kNIss;           // atoms per issuer per step
    constexpr int kAcc0 = kAS * 128;                      // TMEM: [A stages | accumulators]
    static_assert(kAcc0 + kNIss * DN <= 512, "TMEM budget");
    constexpr int kXStage = kAtomsPerStep * DN * 128;     // four 64-column atoms of DN rows

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
            mbar_init(&h->x_empty[i], kNIss);  // one tcgen05.commit per issuer
        }
        for (int i = 0; i < kAS; ++i) {
            mbar_init(&h->a_full[i], 8);       // the 8 warps of the group that wrote the stage
            mbar_init(&h->a_empty[i], kNIss);
        }
        for (int i = 0; i < kNIss; ++i) {
            mbar_init(&h->d_full[i], 1);
            h->epi_seq[i] = 0;
        }
        fence_barrier_init();
    } else if (threadIdx.x == 32) {
        // segment table from the slot counts of this forward: weights w < K are the
        // routed experts (cnt[w] slots), then the shared experts (batch rows each)
        const int W = p.num_experts + p.num_shared;
        int acc = 0;
        for (int w = 0; w < W; ++w) {
            int n = w < p.num_experts ? p.cnt[w] : p.batch;
            DEC_CHECK(n >= 0 && n <= p.cap8, "weight %d: %d slots, cap8 %d\n", w, n, p.cap8);
            n = n < 0 ? 0 : (n > p.cap8 ? p.cap8 : n);   // the router never hands out more (it flags instead)
            h->n_rows[w] = n;
            h->wt_first[w] = acc;
            acc += (n + DN - 1) / DN;
        }
        h->wt_first[W] = acc;
        for (int w = W + 1; w <= kDecMaxW; ++w) h->wt_first[w] = 0x7fffffff;
        h->n_wt = acc;
#ifdef TQ_DEC_CHECK
        {
            int slots = 0;
            for (int w = 0; w < p.num_experts; ++w) slots += p.cnt[w];
            DEC_CHECK(p.check_slots <= 0 || slots == p.check_slots, "routed slots %d, expected %d (batch %d)\n", slots,
                      p.check_slots, p.batch);
        }
#endif
    }
    if (wid == kCProd) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&h->tmem_base)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    ctrace(p, 1);
    const uint32_t tmem = h->tmem_base;

    const int sps = p.nmain + (p.n_ext64 > 0 ? 1 : 0);    // steps per segment
    const int64_t total = static_cast<int64_t>(h->n_wt) * p.mb_count * sps;
    const int G = gridDim.x;
    const int64_t g_begin = cta_start(blockIdx.x, total, G);
    const int64_t g_end = cta_start(blockIdx.x + 1, total, G);
    const int n_steps = static_cast<int>(g_end - g_begin);
    const int gshift = p.group_shift;

    if (n_steps > 0) {
        if (wid >= kDq0) {
            // ===================== dequant groups =====================
            const int dw = wid - kDq0;
            const int grp = dw >> 3;
            const int hw = (dw >> 2) & 1;                  // atoms 2hw, 2hw+1 of the step
            const int q = wid & 3;                         // TMEM lane quarter (warp id % 4)
            const int rloc = q * 32 + lane;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            int cs = grp, as = grp;
            uint32_t cph = 0, aph = 0;
            int k = static_cast<int>((g_begin + grp) % sps);
            for (int j = grp; j < n_steps; j += 2) {
                const int nat = step_atoms(p, k);
                mbar_wait(&h->c_full[cs], cph);
                if (lane == 0 && q == 0 && hw == 0) dtrace(p, 2, j);
                const uint8_t* st = smem + cs * SC;
                if (k < p.nmain) {
                    // main step: atoms 2hw, 2hw+1 (if present), two 32-code super-words each;
                    // one super-word live in registers at a time (896 threads: <= 72 registers)
                    const int e0 = k * kAtomsPerStep * 64;        // first K of the step
                    const int ein = gshift >= 0 ? (e0 & ((1 << gshift) - 1)) : e0 % p.group_size;
                    const int glast = p.groups - 1 - (gshift >= 0 ? e0 >> gshift : e0 / p.group_size);
                    const uint16_t* sc = reinterpret_cast<const uint16_t*>(st + kAtomsPerStep * kBlk) + rloc;
                    // groups of >= 128 columns: this warp's 128 columns (atoms 2hw, 2hw+1, the
                    // step being 256-aligned) share one scale -- one scale load and one bias
                    // table for all four super-words
                    const bool one_group = gshift >= 7;
                    DqConst dq1;
                    if (one_group)
                        dq1 = make_dq(__ushort_as_half(sc[min((ein + 128 * hw) >> gshift, glast) * kBM]));
                    mbar_wait(&h->a_empty[as], aph ^ 1u);
                    if (lane == 0 && q == 0 && hw == 0) dtrace(p, 8, j);
                    tc_fence_after();
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int at = 2 * hw + t;
                        if (at < nat) {
                            const uint32_t* wst = reinterpret_cast<const uint32_t*>(st + at * kBlk) + rloc;
                            uint32_t words[2][kWords];
                            uint16_t sbits[2] = {0, 0};
#pragma unroll
                            for (int ss = 0; ss < 2; ++ss) {
#pragma unroll
                                for (int w = 0; w < kWords; ++w) words[ss][w] = wst[ss * kHalf + w * kBM];
                                if (!one_group) {
                                    const int off = ein + 64 * at + 32 * ss;
                                    // a super-word past in_dim (zero codes) may lie past the last group
                                    const int gi = min(gshift >= 0 ? off >> gshift : off / p.group_size, glast);
                                    sbits[ss] = sc[gi * kBM];
                                }
                            }
#pragma unroll
                            for (int ss = 0; ss < 2; ++ss) {
                                uint32_t v[16];
#if (TQ_DEC_ABL & 4)
#pragma unroll
                                for (int w = 0; w < 16; ++w) v[w] = words[ss][w % kWords] + sbits[ss];
#else
                                if (one_group) {
                                    dequant32<BITS>(words[ss], dq1, v);
                                } else {
                                    const DqConst dq = make_dq(__ushort_as_half(sbits[ss]));
                                    dequant32<BITS>(words[ss], dq, v);
                                }
#endif
                                tc_st_32x32b_x16(tmem + lane_base + as * 128 + at * 32 + ss * 16, v);
                            }
                        }
                    }
                    tc_wait_st();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&h->c_empty[cs]);
                } else {
                    // ext step: dense fp16 atoms (32 u32 words per row each); this warp moves atoms 2hw, 2hw+1
                    mbar_wait(&h->a_empty[as], aph ^ 1u);
                    tc_fence_after();
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int at = 2 * hw + t;
                        if (at < nat) {
                            const uint32_t* eb = reinterpret_cast<const uint32_t*>(st + at * kExtAtomBytes) + rloc;
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh) {
                                uint32_t v[16];
#pragma unroll
                                for (int w = 0; w < 16; ++w) v[w] = eb[(hh * 16 + w) * kBM];
                                tc_st_32x32b_x16(tmem + lane_base + as * 128 + at * 32 + hh * 16, v);
                            }
                        }
                    }
                    tc_wait_st();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&h->c_empty[cs]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&h->a_full[as]);
                if (lane == 0 && q == 0 && hw == 0) dtrace(p, 3, j);
                // next own step (stage indices advance by 2 = the group count)
                cs += 2;
                if (cs >= S) { cs -= S; cph ^= 1u; }
                as += 2;
                if (as >= kAS) { as -= kAS; aph ^= 1u; }
                k += 2;
                while (k >= sps) k -= sps;
            }
        } else if (wid == kCProd || wid == kCProd + 1) {
            // ===================== code producers =====================
            const int pp = wid - kCProd;
            int cs = pp;
            uint32_t cph = 0;
            int s = static_cast<int>((g_begin + pp) / sps), k = static_cast<int>((g_begin + pp) % sps);
            Seg sg = seg_info<DN>(h, p, s);
            for (int j = pp; j < n_steps; j += 2) {
                if (sg.s != s) sg = seg_info<DN>(h, p, s);
                const int64_t wm = static_cast<int64_t>(sg.w) * p.mb_count + sg.mb;
                uint8_t* cdst = smem + cs * SC;
                const int nat = step_atoms(p, k);
                mbar_wait(&h->c_empty[cs], cph ^ 1u);
                if (lane == 0) dtrace(p, 0, j);
                if (k < p.nmain) {
                    const int kb0 = k * kAtomsPerStep;
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
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&h->c_full[cs], cb + sb);
#if !(TQ_DEC_ABL & 8)
                        bulk_copy_g2s(cdst, csrc, cb, &h->c_full[cs]);
                        bulk_copy_g2s(cdst + kAtomsPerStep * kBlk, p.scales + (wm * p.groups + g0) * kBM, sb,
                                      &h->c_full[cs]);
#else
                        (void)csrc;
                        asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&h->c_full[cs])),
                                     "r"(cb + sb)
                                     : "memory");
#endif
                    }
                } else {
                    const uint32_t eb = static_cast<uint32_t>(p.n_ext64 * kExtAtomBytes);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&h->c_full[cs], eb);
                        bulk_copy_g2s(cdst, p.ext_blocks + wm * eb, eb, &h->c_full[cs]);
                    }
                }
                __syncwarp();
                cs += 2;
                if (cs >= S) { cs -= S; cph ^= 1u; }
                k += 2;
                while (k >= sps) { k -= sps; ++s; }
            }
        } else if (wid == kXProd || wid == kXProd + 1) {
            // ===================== activation producers =====================
            const int pp = wid - kXProd;
            int xs = pp;
            uint32_t xph = 0;
            int s = static_cast<int>((g_begin + pp) / sps), k = static_cast<int>((g_begin + pp) % sps);
            Seg sg = seg_info<DN>(h, p, s);
            for (int j = pp; j < n_steps; j += 2) {
                if (sg.s != s) sg = seg_info<DN>(h, p, s);
                uint8_t* xdst = smem + x_off + xs * kXStage;
                const int nat = step_atoms(p, k);
                const uint32_t xb = static_cast<uint32_t>((sg.n_tok + 7) & ~7) * 128u;   // 8-row granules
                mbar_wait(&h->x_empty[xs], xph ^ 1u);
                if (lane == 0) dtrace(p, 1, j);
                const __half* src;
                if (k < p.nmain) src = p.xperm + (static_cast<int64_t>(k * kAtomsPerStep) * p.atom_rows + sg.row0) * 64;
                else src = p.extperm + static_cast<int64_t>(sg.row0) * 64;
                if (elect_one()) {
                    mbar_arrive_expect_tx(&h->x_full[xs], nat * xb);
#if !(TQ_DEC_ABL & 1)
                    for (int at = 0; at < nat; ++at)
                        bulk_copy_g2s(xdst + at * DN * 128, src + at * p.atom_rows * 64, xb, &h->x_full[xs]);
#else
                    (void)src;
                    asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&h->x_full[xs])),
                                 "r"(nat * xb)
                                 : "memory");
#endif
                }
                __syncwarp();
                xs += 2;
                if (xs >= SX) { xs -= SX; xph ^= 1u; }
                k += 2;
                while (k >= sps) { k -= sps; ++s; }
            }
        } else if (wid >= kMma0 && wid < kMma0 + kNIss) {
            // ===================== MMA issuers: atoms [ii * kAPI, +kAPI) of every step =====================
            const int ii = wid - kMma0;
            int as = 0, xs = 0;
            uint32_t xph = 0, aph = 0;
            int64_t x = g_begin;
            uint32_t m = 0;                                 // part ordinal
            while (x < g_end) {
                const int s = static_cast<int>(x / sps);
                const int64_t seg_end = static_cast<int64_t>(s + 1) * sps;
                const int64_t pe = seg_end < g_end ? seg_end : g_end;
                const Seg sg = seg_info<DN>(h, p, s);
                const uint32_t idesc = idesc_f16(static_cast<uint32_t>((sg.n_tok + 15) & ~15));
                const uint32_t d_tmem = tmem + kAcc0 + ii * DN;
                seq_wait(&h->epi_seq[ii], m);               // the epilogue drained part m - 1
                tc_fence_after();
                bool first = true;
                for (; x < pe; ++x) {
                    const int k = static_cast<int>(x - static_cast<int64_t>(s) * sps);
                    const int nat = step_atoms(p, k);
                    mbar_wait(&h->a_full[as], aph);             // every issuer waits every step, in order
                    if (lane == 0) dtrace(p, 4, static_cast<int>(x - g_begin));
                    mbar_wait(&h->x_full[xs], xph);
                    if (lane == 0) dtrace(p, 5, static_cast<int>(x - g_begin));
                    tc_fence_after();
#if !(TQ_DEC_ABL & 2)
#pragma unroll
                    for (int a2 = 0; a2 < kAPI; ++a2) {
                        const int at = ii * kAPI + a2;
                        if (at < nat) {
                            const uint32_t xaddr = s_base + x_off + xs * kXStage + at * DN * 128;
                            tc_mma_ts_x4_elect(d_tmem, tmem + as * 128 + at * 32, sw128_desc(xaddr), idesc,
                                               first ? 0u : 1u);
                            first = false;
                        }
                    }
#else
                    (void)idesc;
                    (void)d_tmem;
#endif
                    tc_commit_elect(&h->a_empty[as]);
                    tc_commit_elect(&h->x_empty[xs]);
                    if (lane == 0) dtrace(p, ii == 0 ? 6 : (ii == kNIss - 1 ? 9 : 15), static_cast<int>(x - g_begin));
                    if (++as == kAS) { as = 0; aph ^= 1u; }
                    if (++xs == SX) { xs = 0; xph ^= 1u; }
                }
                if (!first) tc_commit_elect(&h->d_full[ii]);
                else if (lane == 0) mbar_arrive(&h->d_full[ii]);
                __syncwarp();
                ++m;
            }
        } else if (wid >= kEpi0 && wid < kEpi0 + 4) {
            // ===================== epilogue =====================
            const int q = wid & 3;
            int64_t x = g_begin;
            uint32_t m = 0;
            const int first_seg = static_cast<int>(g_begin / sps);
            while (x < g_end) {
                const int s = static_cast<int>(x / sps);
                const int64_t seg_begin = static_cast<int64_t>(s) * sps;
                const int64_t seg_end = seg_begin + sps;
                const int64_t pe = seg_end < g_end ? seg_end : g_end;
                const Seg sg = seg_info<DN>(h, p, s);
                // issuer ii took part iff some step of the part has more than ii atoms
                int max_at = 0;
                for (int64_t y = x; y < pe; ++y) max_at = max(max_at, step_atoms(p, static_cast<int>(y - seg_begin)));
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
                for (int ii = 0; ii < kNIss; ++ii) mbar_wait_sleep(&h->d_full[ii], m & 1u);
                if (lane == 0 && q == 0) dtrace(p, 7, static_cast<int>(m));
                tc_fence_after();
                const uint32_t dbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + kAcc0;
                for (int t0 = 0; t0 < sg.n_tok; t0 += 16) {
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = 0.0f;
#pragma unroll
                    for (int ii = 0; ii < kNIss; ++ii) {   // fixed order: deterministic sum of the atom streams
                        if (ii * kAPI >= max_at) continue;
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
                named_bar_sync(1, 128);   // all four quarters have read the accumulators
                if (q == 0 && lane < kNIss) seq_store_release(&h->epi_seq[lane], m + 1u);
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
                                const int cslot = static_cast<int>(cta_start(c, total, G) / sps) == s ? 0 : 1;
                                acc += __ldcg(p.scratch + ((static_cast<int64_t>(c) * 2 + cslot) * DN + t) * kBM + q * 32 +
                                              lane);
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
    ctrace(p, 2);
    if (wid == kCProd) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

// -----------------------------------------------------------------------------

static int dec_code_stage_bytes(int bits, int n_ext64) {
    const int main_bytes = kAtomsPerStep * code_block_bytes(bits) + (256 / 32 + 1) * kBM * 2;
    const int ext_bytes = n_ext64 * kExtAtomBytes;
    const int b = main_bytes > ext_bytes ? main_bytes : ext_bytes;
    return (b + 1023) / 1024 * 1024;
}

cudaError_t launch_decode(const DecParams& p0, int dn, int grid, cudaStream_t stream) {
    DecParams p = p0;
    if (dn != 32 && dn != 64) return cudaErrorInvalidValue;
    if (p.num_experts + p.num_shared > kDecMaxW || p.n_ext64 > kAtomsPerStep) return cudaErrorInvalidValue;
    const int sc = dec_code_stage_bytes(p.bits, p.n_ext64);
    const int xst = kAtomsPerStep * dn * 128;
    const int avail = kSmemBudget - 1024 - kHdrBytes;
    // both rings even (two producers / two dequant groups split them by step parity);
    // 8 code stages when they fit with >= 4 activation stages, the rest to activations
    int cs = 8;
    int xs = ((avail - cs * sc) / xst) & ~1;
    while (xs < 4 && cs > 4) {
        cs -= 2;
        xs = ((avail - cs * sc) / xst) & ~1;
    }
    if (xs > kMaxXS) xs = kMaxXS;
    if (xs < 2 || cs < 4) return cudaErrorInvalidValue;
    cs = ((avail - xs * xst) / sc) & ~1;
    if (cs > kMaxCS) cs = kMaxCS;
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
