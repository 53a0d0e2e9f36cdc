// THE fused kernel: a persistent, warp-specialised tcgen05 grouped GEMM whose
// A operand (the quantized expert weights) is dequantized in registers and
// stored straight into tensor memory, never touching shared memory as fp16.
//
//   D[128 weight rows x N tokens] (fp32, TMEM)  +=  A[128 x K] (fp16, TMEM)  *  X[N x K]^T (fp16, SMEM)
//
// per work unit (weight matrix, 128-row m-block, token tile, K range).  After
// the main K chunks, extension chunks append, in the SAME accumulator,
//   [-zero*s per scale group | U_p codes]  x  [group sums of x | (X.A_q) * su]
// i.e. the zero-point correction of the affine residual codes and the
// rank-r tile correction (X.A).B_p of the shared low-rank factors.
//
// Warp roles:
//   0  code producer: cp.async.bulk of packed code blocks + fp16 scale slices
//      (+ per-unit extension blocks) into a deep smem ring
//   1  MMA issuer: one thread, tcgen05.mma.cta_group::1.kind::f16, A in TMEM
//   2  TMEM allocator
//   3  activation producer: TMA 2D tiles (large token tiles) or cp.async
//      16-byte rows with the 128B swizzle applied in software (small tiles)
//   4 .. 4+4*NG-1  dequant: NG independent groups of 4 warps; warp q of a
//      group owns TMEM lanes (weight rows) 32q..32q+31; the groups take whole
//      K chunks round-robin so NG chunks are in flight at once (each chunk's
//      barrier/TMEM latency chain overlaps the others)
//   last 4  epilogue: tcgen05.ld -> scale -> coalesced fp32 stores
//
// Configurations (KC = K elements per chunk, DN = TMEM accumulator columns):
//   decode  KC=128 NG=3 DN=64    mid  KC=128 NG=3 DN=128    prefill  KC=64 NG=2 DN=192
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "tq_internal.h"
#include "tq_ptx.cuh"

namespace tqb {

constexpr int kTmemCols = 512;
constexpr int kMaxXStages = 64;   // activation ring stages, or resident slots (one per chunk of a unit)
constexpr int kMaxCStages = 24;
constexpr int kMaxAStages = 8;
constexpr int kSmemBudget = 225 * 1024;

// TMEM: [A stages: kc/2 columns each][accumulators: 2 buffers x ni issuers x dn]
__host__ __device__ constexpr int a_stages(int kc, int dn, int ni) {
    return ((kTmemCols - 2 * ni * dn) / (kc / 2)) < kMaxAStages ? ((kTmemCols - 2 * ni * dn) / (kc / 2)) : kMaxAStages;
}
__host__ __device__ constexpr int gemm_threads(int ng) { return (8 + 4 * ng) * 32; }
__host__ __device__ constexpr int scale_trailer(int bits, int kc) {
    return bits == kDenseBits ? 0 : (kc / 32) * kBM * 2;
}
__host__ __device__ constexpr int code_stage_bytes(int bits, int kc) {
    return (kc / kKC) * code_block_bytes(bits) + scale_trailer(bits, kc);
}
// extension blocks of one (weight, m-block): n_ext64 dense fp16 128 x 64 blocks
__host__ __device__ inline int ext_slot_bytes(int n_ext64) { return n_ext64 * code_block_bytes(kDenseBits); }

#ifndef TQ_DECODE_NI
#define TQ_DECODE_NI 2   // MMA issue streams of the decode configuration (experiments: 3)
#endif
constexpr int kHdrBytes = 2048;   // barrier header region
constexpr int kUnitCache = 64;    // work units staged in shared memory per CTA
struct SharedHdr {
    // one ring for the MMA operands: stage s = A columns in TMEM + an activation
    // tile in smem; full = 4 dequant warps + the activation producer (with its
    // TMA bytes), empty = one tcgen05.commit after the stage's MMAs
    uint64_t full[kMaxAStages], empty[kMaxAStages];
    // activation ring, deeper than the A ring: its TMA loads queue behind the
    // packed-code bulk copies in the SM's copy engine, so they are issued early
    uint64_t x_full[kMaxXStages], x_empty[kMaxXStages];
    uint64_t c_full[kMaxCStages], c_empty[kMaxCStages];
    uint64_t d_full[2], d_empty[2];
    uint64_t e_full[2], e_empty[2];
    uint32_t tmem_base;
    // extension blocks fully consumed so far, counted in dequant-warp arrivals:
    // a consumer of ext block n waits for blocks < n - e_slots + 1 first, so its
    // parity wait on the (1-2 slot) ext ring is never more than one phase ahead
    // -- the warps of the dequant groups drift up to the A-stage ring depth apart,
    // which spans several ext blocks when units carry few main chunks
    int ext_arrivals;
};

static_assert(sizeof(SharedHdr) <= kHdrBytes, "barrier header");

// TQ_TRACE_ID builds: record identities instead of times (debugging the chunk accounting)
__device__ __forceinline__ void trace_id(const GemmParams& p, int slot, int idx, unsigned long long v) {
#ifdef TQ_TRACE_ID
    if ((p.debug & 8) && static_cast<int>(blockIdx.x) == (p.debug >> 16) && idx < 4096) p.trace[slot * 4096 + idx] = v;
#endif
}

__device__ __forceinline__ void trace_ev(const GemmParams& p, int slot, int idx) {
#if defined(TQ_TRACE) && !defined(TQ_TRACE_ID)
    if ((p.debug & 8) && static_cast<int>(blockIdx.x) == (p.debug >> 16) && idx < 4096) p.trace[slot * 4096 + idx] = clock64();
#endif
}

// TQ_PROFILE builds: every warp accumulates the cycles it spends in selected
// waits / phases (4 slots) and writes them, with its total, at exit.
#ifdef TQ_PROFILE
#define TQ_TIMED(slot, stmt)                   \
    do {                                       \
        const long long t0_ = clock64();       \
        stmt;                                  \
        prof[slot] += clock64() - t0_;         \
    } while (0)
#else
#define TQ_TIMED(slot, stmt) stmt
#endif

// NI MMA issuers (logical warps 1 and 2): a single issuing thread sustains
// one M=128 K=16 MMA per ~56 cycles for N <= 64 whatever N is, so small-N
// decode tiles need several issue streams; issuer j takes the chunks whose
// CTA-wide index is j mod NI and accumulates into its own TMEM columns; the
// epilogue adds the NI partial accumulators in a fixed order.
template <int BITS, int KC, int NG, int DN, int NI>
__global__ void __launch_bounds__(gemm_threads(NG), 1) gemm_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
#ifdef TQ_PROFILE
    unsigned long long g_entry;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
    const long long c_entry = clock64();
#endif
    constexpr int kAS = a_stages(KC, DN, NI);
    static_assert(NI >= 1 && NI <= 3, "issuers");
    // decode configuration: the activation tile of a RUN of units (same expert,
    // token tile and K range; consecutive m-blocks) stays resident in shared
    // memory -- loaded once, chunk by chunk, by the code producer -- instead of
    // being re-fetched for every 128-row m-block
    constexpr bool kXR = DN == 32;
    constexpr bool kGX = false;
    constexpr int kAtoms = KC / kKC;                  // 128-byte swizzle atoms per activation row
    constexpr int kACols = KC / 2;                    // TMEM columns per A stage
    constexpr int kDCol0 = kAS * kACols;
    constexpr int kBlk = code_block_bytes(BITS);      // one 128 x 64 code block
    constexpr int kCBytes = kAtoms * kBlk;            // codes per chunk
    constexpr int kCStage = code_stage_bytes(BITS, KC);
    constexpr int kSW = KC / 32;                      // 32-code super-words per dequant thread per chunk
    constexpr int kWords = BITS;                      // u32 words per super-word (dense fp16: 16)
    constexpr int kDqWarps = 4 * NG;
    constexpr int kEpi0 = 4 + kDqWarps;               // first epilogue warp
    static_assert(kDCol0 + 2 * NI * DN <= kTmemCols, "TMEM budget");

    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t pad = (1024u - (raw & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    const uint32_t s_base = raw + pad;
    const int ext_bytes = ext_slot_bytes(p.n_ext64);
    const int x_rows = p.x_stage_rows;
    const int x_atom_bytes = x_rows * 128;
    const int x_stage_bytes = kAtoms * x_atom_bytes;
    const int x_stages = p.x_stages;
    const int c_stages = p.c_stages;
    const uint32_t x_off = 0;
    const uint32_t c_off = x_off + x_stages * x_stage_bytes;
    const uint32_t e_off = c_off + c_stages * kCStage;
    SharedHdr* hdr = reinterpret_cast<SharedHdr*>(smem + e_off + p.e_slots * ext_bytes);
#ifdef TQ_WAIT_TRAP_LAYOUT
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("TQ_WAIT_TRAP layout: hdr 0x%x (full +0, empty +%d, x_full +%d, x_empty +%d, c_full +%d, c_empty +%d, "
               "d_full +%d, d_empty +%d, e_full +%d, e_empty +%d) kAS %d xs %d cs %d\n",
               smem_u32(hdr), (int)offsetof(SharedHdr, empty), (int)offsetof(SharedHdr, x_full),
               (int)offsetof(SharedHdr, x_empty), (int)offsetof(SharedHdr, c_full), (int)offsetof(SharedHdr, c_empty),
               (int)offsetof(SharedHdr, d_full), (int)offsetof(SharedHdr, d_empty), (int)offsetof(SharedHdr, e_full),
               (int)offsetof(SharedHdr, e_empty), kAS, x_stages, c_stages);
#endif

    // Role layout: the scheduler arbitrates highest-warp-id first, so the
    // latency-critical single-thread roles sit at the top:
    //   [0, 4NG) dequant | [4NG, 4NG+4) epilogue | +4 TMEM alloc | +5 code producer
    //   | +6 activation producer | +7 MMA issuer
    const int wid = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    constexpr int kRoleBase = 4 * NG + 4;
    const int warp = wid < 4 * NG ? wid + 4                       // dequant -> logical 4..
                   : wid < kRoleBase ? wid - 4 * NG + kEpi0        // epilogue -> logical kEpi0..
                   : (wid == kRoleBase ? 2 : wid == kRoleBase + 1 ? 0 : wid == kRoleBase + 2 ? 3 : 1);
#ifdef TQ_EXPERIMENT
    const int kDbg = p.debug;   // experiment builds: runtime skip flags (TQ_DEBUG)
#elif defined(TQ_DBG_CONST)
    constexpr int kDbg = TQ_DBG_CONST;   // compile-time skip flags (ablation builds)
#else
    constexpr int kDbg = 0;     // production: every debug branch folds away
#endif

    if (threadIdx.x == 0) {
        prefetch_tmap(&p.tmap_x64);
        prefetch_tmap(&p.tmap_e64);
        prefetch_tmap(&p.tmap_x16);
        prefetch_tmap(&p.tmap_e16);
        for (int s = 0; s < kAS; ++s) {
            mbar_init(&hdr->full[s], 4);
            mbar_init(&hdr->empty[s], 1);
        }
        for (int s = 0; s < x_stages; ++s) {
            mbar_init(&hdr->x_full[s], 1);
            mbar_init(&hdr->x_empty[s], kXR ? NI : 1);   // kXR: one commit per issuer at the run's end
        }
        for (int s = 0; s < c_stages; ++s) {
            mbar_init(&hdr->c_full[s], 1);
            mbar_init(&hdr->c_empty[s], 4);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&hdr->d_full[s], NI);
            mbar_init(&hdr->d_empty[s], 4);
            mbar_init(&hdr->e_full[s], 1);
            mbar_init(&hdr->e_empty[s], 4 * (p.n_ext_chunks > 0 ? p.n_ext_chunks : 1));   // p.e_slots used
        }
        hdr->ext_arrivals = 0;
        fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&hdr->tmem_base)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // programmatic dependent launch: the prologue above overlapped the previous
    // kernel; everything below reads its outputs
    pdl_wait();
    pdl_launch_dependents();
    const int n_all = (kDbg & 256) ? 0 : *p.n_units;   // 256: prologue/epilogue only (fixed cost)
    // unit range of this CTA: contiguous (runs of units share their activation
    // tile) or strided over the persistent grid
    const int n_units = p.contig ? static_cast<int>((static_cast<int64_t>(blockIdx.x) + 1) * n_all / gridDim.x) : n_all;
    const uint32_t tmem = hdr->tmem_base;
#ifdef TQ_PROFILE
    long long prof[4] = {0, 0, 0, 0};
    const long long prof_t0 = clock64();
    const long long prologue_cycles = prof_t0 - c_entry;
#endif
    const int first = p.contig ? static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_all / gridDim.x) : blockIdx.x;
    const int stride = p.contig ? 1 : gridDim.x;
    // this CTA's work units, staged in shared memory once: every role walks the
    // same list (a dependent global load per unit per role otherwise)
    Unit* s_units = reinterpret_cast<Unit*>(reinterpret_cast<uint8_t*>(hdr) + kHdrBytes);
    {
        const int n_mine = first < n_units ? (n_units - first + stride - 1) / stride : 0;
        const int n_cache = n_mine < kUnitCache ? n_mine : kUnitCache;
        for (int i = threadIdx.x; i < 2 * n_cache; i += blockDim.x)
            reinterpret_cast<int4*>(s_units)[i] =
                reinterpret_cast<const int4*>(p.units + first + static_cast<int64_t>(i >> 1) * stride)[i & 1];
        __syncthreads();
    }
    auto unit_at = [&](int u) -> Unit {
        const int k = stride == 1 ? u - first : (u - first) / stride;
        return k < kUnitCache ? s_units[k] : p.units[u];
    };
    // resident activation slots (kXR): slot c holds chunk c of the current run
    const int xr_slot_bytes = kAtoms * x_atom_bytes;
    auto same_run = [](const Unit& a, const Unit& b) {
        return a.weight == b.weight && a.x_row == b.x_row && a.n_tok == b.n_tok && a.kc_begin == b.kc_begin &&
               a.kc_end == b.kc_end && a.n_ext == b.n_ext;
    };
    const int gshift = p.group_shift;

    if (warp == 0) {
        // ===================== code producer (converged warp, one elected lane issues) =====
        {
            int cs = 0, es = 0, tcnt = 0;
            uint32_t cph = 0, eph = 0;
            uint64_t xm = 0;   // kXR: per-slot count (mod 2) of runs that have used the slot
            Unit prev{};
            Unit nxt = first < n_units ? unit_at(first) : Unit{};
            for (int u = first; u < n_units; u += stride) {
                const Unit un = nxt;
                if (u + stride < n_units) nxt = unit_at(u + stride);
                const bool run_start = u == first || !same_run(prev, un);
#ifndef TQ_TRACE_UNIT
                if (kXR && lane == 0) trace_ev(p, 1, u - first);
#endif
                prev = un;
                const int nmain = un.kc_end - un.kc_begin;
                const int64_t wm = static_cast<int64_t>(un.weight) * (p.o_pad / kBM) + un.mb;  // (w, mb) slab
                const uint8_t* wbase = p.codes + static_cast<int64_t>(un.weight) * p.weight_stride +
                                       static_cast<int64_t>(un.mb) * p.kc_total * kCBytes;
                // kXR: the run's activation tile for chunk c, queued just ahead of chunk c's codes
                auto load_x = [&](int c) {
                    const bool ext = c >= nmain;
                    const int col0 = ext ? (c - nmain) * KC : (un.kc_begin + c) * KC;
                    const int natoms = ext ? min(kAtoms, p.n_ext64 - (c - nmain) * kAtoms) : kAtoms;
                    const __half* src = ext ? p.e_ptr : p.x_ptr;
                    TQ_TIMED(1, mbar_wait_sleep(&hdr->x_empty[c], static_cast<uint32_t>((xm >> c) & 1u) ^ 1u));
                    xm ^= 1ull << c;
                    if (elect_one()) {
                        const uint32_t nrow = static_cast<uint32_t>((un.n_tok + 15) & ~15);
                        mbar_arrive_expect_tx(&hdr->x_full[c], natoms * nrow * 128u);
                        uint8_t* xst = smem + x_off + c * xr_slot_bytes;
                        for (int at = 0; at < natoms; ++at)
                            bulk_copy_g2s(xst + at * x_atom_bytes,
                                          src + ((static_cast<int64_t>(col0 / kKC + at) * p.x_atom_rows) + un.x_row) * kKC,
                                          nrow * 128u, &hdr->x_full[c]);
                    }
                    __syncwarp();
                };
                // per-chunk issue path kept short: pointers advance incrementally, the
                // activation loads of a run's first unit take a separate loop
                const uint8_t* csrc = wbase + static_cast<int64_t>(un.kc_begin) * kCBytes;
                uint8_t* cdst = smem + c_off + cs * kCStage;
                const __half* sbase = p.scales + wm * p.groups * kBM;
                int e0 = un.kc_begin * KC;
                auto issue_codes = [&]() {
#ifdef TQ_TRACE_PROD
                    if (lane == 0) trace_ev(p, 5, tcnt);
#endif
                    TQ_TIMED(0, mbar_wait_sleep(&hdr->c_empty[cs], cph ^ 1u));
#ifdef TQ_TRACE_PROD
                    if (lane == 0) trace_ev(p, 6, tcnt);
#endif
                    if (kDbg & 128) {
                        if (lane == 0) mbar_arrive(&hdr->c_full[cs]);
                    } else if constexpr (BITS == kDenseBits) {
                        bulk_copy2_elect(&hdr->c_full[cs], cdst, csrc, kCBytes, cdst, csrc, 0u);
                    } else {
                        int g0, glast;
                        if (gshift >= 0) {
                            g0 = e0 >> gshift;
                            glast = (e0 + KC - 1) >> gshift;
                        } else {
                            g0 = e0 / p.group_size;
                            glast = (e0 + KC - 1) / p.group_size;
                        }
                        const int g1 = min(p.groups - 1, glast);
                        bulk_copy2_elect(&hdr->c_full[cs], cdst, csrc, kCBytes, cdst + kCBytes, sbase + g0 * kBM,
                                         static_cast<uint32_t>(g1 - g0 + 1) * kBM * 2);
                    }
                    if (lane == 0) trace_ev(p, 0, tcnt);
                    ++tcnt;
                    csrc += kCBytes;
                    e0 += KC;
                    cdst += kCStage;
                    if (++cs == c_stages) {
                        cs = 0;
                        cph ^= 1u;
                        cdst = smem + c_off;
                    }
                };
                if (kXR && run_start) {
                    for (int c = 0; c < nmain; ++c) {
                        load_x(c);
                        issue_codes();
                    }
                } else {
                    for (int c = 0; c < nmain; ++c) issue_codes();
                }
#ifndef TQ_TRACE_UNIT
                if (kXR && lane == 0) trace_ev(p, 3, u - first);
#endif
                if (kXR && run_start)
                    for (int c = nmain; c < nmain + un.n_ext; ++c) load_x(c);
                if (un.n_ext > 0 && p.n_ext64 > 0) {
                    TQ_TIMED(1, mbar_wait_sleep(&hdr->e_empty[es], eph ^ 1u));
                    uint8_t* dst = smem + e_off + es * ext_bytes;
                    bulk_copy2_elect(&hdr->e_full[es], dst, p.ext_blocks + wm * ext_bytes, ext_bytes, dst, dst, 0u);
                    if (lane == 0) trace_id(p, 1, u - first, (static_cast<unsigned long long>(es) << 8) | eph | (static_cast<unsigned long long>(un.n_ext) << 16) | (static_cast<unsigned long long>(nmain) << 24));
                    if (++es == p.e_slots) { es = 0; eph ^= 1u; }
                }
            }
        }
    } else if (warp == 3 && NI < 3) {
        // ===================== activation producer (all 32 lanes) ==========
        if (kXR) {
        } else {
        // small token tiles (decode): cp.async 16-byte pieces through the LSU with
        // the 128B swizzle applied in software -- TMA loads would queue behind
        // the packed-code bulk copies in the SM's copy engine; large tiles: TMA
        int xs = 0, tcnt = 0;
        uint32_t xph = 0;
        Unit nxt = first < n_units ? unit_at(first) : Unit{};
        for (int u = first; u < n_units; u += stride) {
            const Unit un = nxt;
            if (u + stride < n_units) nxt = unit_at(u + stride);
            const int nmain = un.kc_end - un.kc_begin;
            const int nch = nmain + un.n_ext;
            const bool small = un.n_tok <= 8;   // a few rows: LSU; 16-row granules and up: TMA
            const int box = un.n_tok > 48 ? 64 : 16;
            const int nbox = (un.n_tok + box - 1) / box;
            for (int c = 0; c < nch; ++c) {
                const bool ext = c >= nmain;
                TQ_TIMED(0, mbar_wait(&hdr->x_empty[xs], xph ^ 1u));
                const int col0 = ext ? (c - nmain) * KC : (un.kc_begin + c) * KC;
                const int natoms = ext ? min(kAtoms, p.n_ext64 - (c - nmain) * kAtoms) : kAtoms;
                if (kDbg & 32) {
                    if (lane == 0) mbar_arrive(&hdr->x_full[xs]);
                } else if (p.x_atom_rows > 0) {
                    if (lane == 0) {
                        const __half* src = ext ? p.e_ptr : p.x_ptr;
                        const uint32_t nrow = static_cast<uint32_t>((un.n_tok + 15) & ~15);
                        mbar_arrive_expect_tx(&hdr->x_full[xs], natoms * nrow * 128u);
                        uint8_t* xst = smem + x_off + xs * x_stage_bytes;
                        for (int at = 0; at < natoms; ++at)
                            bulk_copy_g2s(xst + at * x_atom_bytes,
                                          src + ((static_cast<int64_t>(col0 / kKC + at) * p.x_atom_rows) + un.x_row) * kKC,
                                          nrow * 128u, &hdr->x_full[xs]);
                    }
                    __syncwarp();
                } else if (small) {
                    const __half* src = ext ? p.e_ptr : p.x_ptr;
                    const int64_t ld = ext ? p.e_ld : p.x_ld;
                    const uint32_t sx = s_base + x_off + xs * x_stage_bytes;
                    // lanes per row = natoms * 8 pieces (a power of two <= 32)
                    const int lshift = 3 + (natoms >= 4 ? 2 : natoms >= 2 ? 1 : 0);
                    const int rows_per_it = 32 >> lshift;
                    const int piece = lane & ((1 << lshift) - 1);
                    const int at = piece >> 3, ch = piece & 7;
                    const __half* g = src + static_cast<int64_t>(un.x_row) * ld + col0 + at * kKC + ch * 8;
                    for (int row = lane >> lshift; row < un.n_tok; row += rows_per_it)
                        cp_async_16(sx + at * x_atom_bytes + row * 128 + ((ch ^ (row & 7)) << 4), g + row * ld);
                    cp_async_mbar_arrive_inc(&hdr->x_full[xs]);   // pending += 1, -1 when this lane's copies land
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&hdr->x_full[xs]);
                } else {
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&hdr->x_full[xs], static_cast<uint32_t>(natoms * nbox * box * 128));
                        const CUtensorMap* map = ext ? (box == 64 ? &p.tmap_e64 : &p.tmap_e16)
                                                     : (box == 64 ? &p.tmap_x64 : &p.tmap_x16);
                        uint8_t* xst = smem + x_off + xs * x_stage_bytes;
                        for (int at = 0; at < natoms; ++at)
                            for (int bx = 0; bx < nbox; ++bx)
                                tma_load_2d(xst + at * x_atom_bytes + bx * box * 128, map, col0 + at * kKC,
                                            un.x_row + bx * box, &hdr->x_full[xs]);
                    }
                    __syncwarp();
                }
                if (lane == 0) trace_ev(p, 1, tcnt);
                ++tcnt;
                if (++xs == x_stages) { xs = 0; xph ^= 1u; }
            }
        }
        }
    } else if (warp == 1 || (NI >= 2 && warp == 2) || (NI >= 3 && warp == 3)) {
        // ===================== MMA issuers (converged warp, one elected lane issues) ==========
        const int j = warp == 1 ? 0 : warp == 2 ? 1 : 2;   // logical 3 = the idle activation producer (kXR)
        int as = j, lu = 0, tcnt = 0;   // issuer j's chunks: CTA-wide index j, j+NI, ...
        uint32_t aph = 0;
        int xs = j;
        uint32_t xph = 0;
        int c_next = j;
        uint64_t xm = 0;   // kXR: per-slot count (mod 2) of completed runs that used the slot
        Unit nxt = first < n_units ? unit_at(first) : Unit{};
        for (int u = first; u < n_units; u += stride, ++lu) {
            const Unit un = nxt;
            if (u + stride < n_units) nxt = unit_at(u + stride);
            const bool run_end = u + stride >= n_units || !same_run(un, nxt);
            const int nmain = un.kc_end - un.kc_begin;
            const int nch = nmain + un.n_ext;
            const int ds = lu & 1;
            const uint32_t dph = (lu >> 1) & 1;
            const uint32_t n = static_cast<uint32_t>((un.n_tok + 15) & ~15);
            const uint32_t idesc = idesc_f16(n);
            const uint32_t d_tmem = tmem + kDCol0 + (ds * NI + j) * DN;
            int c = c_next;
            // every issuer (even one without a chunk in this unit) waits for the
            // epilogue to release this accumulator buffer before it arrives on
            // d_full[ds], so its arrival cannot fall into an older phase
            TQ_TIMED(1, mbar_wait(&hdr->d_empty[ds], dph ^ 1u));
#ifdef TQ_TRACE_UNIT
            if (lane == 0) trace_ev(p, j == 0 ? 1 : 7, lu);
#endif
            tc_fence_after();
            const int c_first = c;
            for (; c < nch; c += NI) {
                TQ_TIMED(0, mbar_wait(&hdr->full[as], aph));
                if (lane == 0) trace_ev(p, 2, tcnt);
                if (kXR) {
                    TQ_TIMED(3, mbar_wait(&hdr->x_full[c], static_cast<uint32_t>((xm >> c) & 1u)));
                } else {
                    TQ_TIMED(3, mbar_wait(&hdr->x_full[xs], xph));
                    if (un.n_tok <= 8) fence_proxy_async_smem();   // cp.async (generic proxy) tiles -> MMA reads
                }
                ++tcnt;
                tc_fence_after();
                const uint32_t xaddr = s_base + x_off + (kXR ? c * xr_slot_bytes : xs * x_stage_bytes);
                const uint64_t bdesc = sw128_desc(xaddr);
                const uint32_t a_tm = tmem + as * kACols;
                // atoms of 64 K: 4 MMAs each, one elected lane, descriptors advanced in PTX
                const int natoms = c < nmain ? kAtoms : min(kAtoms, p.n_ext64 - (c - nmain) * kAtoms);
                if (!(kDbg & 2)) {
#pragma unroll
                    for (int at = 0; at < kAtoms; ++at)
                        if (at < natoms)
                            tc_mma_ts_x4_elect(d_tmem, a_tm + at * 32,
                                               bdesc + static_cast<uint64_t>((at * x_atom_bytes) >> 4), idesc,
                                               (c > c_first || at > 0) ? 1u : 0u);
                }
                tc_commit_elect(&hdr->empty[as]);
                if (!kXR) tc_commit_elect(&hdr->x_empty[xs]);

#ifdef TQ_PROFILE
                prof[2] += 1;   // chunks
#endif
                as += NI;
                if (as >= kAS) { as -= kAS; aph ^= 1u; }
                xs += NI;
                if (xs >= x_stages) { xs -= x_stages; xph ^= 1u; }
            }
            // this issuer's part of unit u is accumulated (or it had no chunk in it)
            if (c_first < nch) tc_commit_elect(&hdr->d_full[ds]);
            else if (lane == 0) mbar_arrive(&hdr->d_full[ds]);
#ifdef TQ_TRACE_UNIT
            if (lane == 0 && j == 0) trace_ev(p, 3, lu);
#endif
            c_next = c - nch;
            if (kXR && run_end) {
                // every issuer releases every slot of the run: a commit covers only the
                // committing thread's MMAs, and with an odd chunk count per unit both
                // issuers have read each slot
                for (int cc = 0; cc < nch; ++cc) tc_commit_elect(&hdr->x_empty[cc]);
                xm ^= (nch >= 64 ? ~0ull : ((1ull << nch) - 1ull));
            }
        }
    } else if (warp >= 4 && warp < kEpi0) {
        // ===================== dequant groups =====================
        const int q = wid & 3;  // TMEM lane quarter = physical warp id % 4
        const int grp = wid >> 2;
        const int rloc = q * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        // the CTA's chunk stream (main + extension chunks of its units, in order)
        // is dealt round-robin to the NG groups: group grp takes global chunk
        // indices grp, grp+NG, ...; ring positions advance incrementally
        int cs = 0, as = grp, es = 0;                  // as: chunk index grp mod kAS (NG <= kAS)
        int eo = 0;                                    // ext blocks before this unit (ordinal)
        volatile int* ext_arrivals = &hdr->ext_arrivals;
        const int ext_per_block = 4 * (p.n_ext_chunks > 0 ? p.n_ext_chunks : 1);
        uint32_t cph = 0, aph = 0, eph = 0;
        int m_cur = 0;                                 // main-chunk index that (cs, cph) denotes
        int q_base = 0, m_base = 0;                    // chunks / main chunks before this unit
        int c_next = grp;                              // next own chunk, relative to q_base
        int tcnt = 0;
        const bool tr = (lane == 0 && q == 0);
        // GX (small token tiles): the group loads the activation tile of its NEXT
        // own chunk with cp.async while it dequantizes the current one -- 128
        // threads keep the LSU busy; no copy-engine queue in the way
        const int gt = threadIdx.x & 127;              // thread within the group (wid & 3 -> q)
        int xs_n = grp, xph_n = 0;                     // X ring slot of the next load (chunk grp, grp+NG, ...)
        auto issue_x = [&](const Unit& xu, int xc) {
            const int xnmain = xu.kc_end - xu.kc_begin;
            const bool ext = xc >= xnmain;
            const int col0 = ext ? (xc - xnmain) * KC : (xu.kc_begin + xc) * KC;
            const int natoms = ext ? min(kAtoms, p.n_ext64 - (xc - xnmain) * kAtoms) : kAtoms;
            mbar_wait(&hdr->x_empty[xs_n], static_cast<uint32_t>(xph_n) ^ 1u);
            const __half* src = ext ? p.e_ptr : p.x_ptr;
            if (p.x_atom_rows > 0) {
                // pre-swizzled atom-major rows: one bulk copy per 64-column atom (async proxy)
                if (gt == 0) {
                    const uint32_t nrow = static_cast<uint32_t>((xu.n_tok + 15) & ~15);
                    mbar_arrive_expect_tx(&hdr->x_full[xs_n], natoms * nrow * 128u);
                    uint8_t* xst = smem + x_off + xs_n * x_stage_bytes;
                    for (int at = 0; at < natoms; ++at)
                        bulk_copy_g2s(xst + at * x_atom_bytes,
                                      src + ((static_cast<int64_t>(col0 / kKC + at) * p.x_atom_rows) + xu.x_row) * kKC,
                                      nrow * 128u, &hdr->x_full[xs_n]);
                }
                return;
            }
            const int64_t ld = ext ? p.e_ld : p.x_ld;
            const uint32_t sx = s_base + x_off + xs_n * x_stage_bytes;
            const int lshift = 3 + (natoms >= 4 ? 2 : natoms >= 2 ? 1 : 0);   // lanes per row = natoms * 8
            const int piece = gt & ((1 << lshift) - 1);
            const int at = piece >> 3, ch = piece & 7;
            if (at < natoms) {
                const __half* g = src + static_cast<int64_t>(xu.x_row) * ld + col0 + at * kKC + ch * 8;
                for (int row = gt >> lshift; row < xu.n_tok; row += (128 >> lshift))
                    cp_async_16(sx + at * x_atom_bytes + row * 128 + ((ch ^ (row & 7)) << 4), g + row * ld);
            }
            cp_async_commit();
        };
        auto advance_x = [&]() {
            xs_n += NG;
            if (xs_n >= x_stages) { xs_n -= x_stages; xph_n ^= 1; }
        };
        Unit nxt = first < n_units ? unit_at(first) : Unit{};
        if (kGX && first < n_units) {
            const int nch0 = (nxt.kc_end - nxt.kc_begin) + nxt.n_ext;
            if (grp < nch0) issue_x(nxt, grp);
            else cp_async_commit();
            advance_x();
        }
        for (int u = first; u < n_units; u += stride) {
            const Unit un = nxt;
            if (u + stride < n_units) nxt = unit_at(u + stride);
            const bool has_nxt = u + stride < n_units;
            const int nmain = un.kc_end - un.kc_begin;
            const int nch = nmain + un.n_ext;
            int c = c_next;
            for (; c < nch; c += NG) {
                // the group's four warps enter each chunk together: unsynchronised they
                // can drift several chunks apart, and a fast warp's parity wait on a
                // ring stage (A stages: kAS = 6 for 4 groups) could then alias a phase
                // two back (named barrier 1 + grp, 128 threads)
                asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(128) : "memory");
                const bool main_chunk = c < nmain;
                if (kGX) {   // prefetch the activation tile of the next own chunk
                    const int cn = c + NG;
                    const int nch_n = has_nxt ? (nxt.kc_end - nxt.kc_begin) + nxt.n_ext : 0;
                    if (cn < nch) TQ_TIMED(0, issue_x(un, cn));
                    else if (cn - nch < nch_n) TQ_TIMED(0, issue_x(nxt, cn - nch));
                    else cp_async_commit();
                    advance_x();
                }
                if (main_chunk) {
                    // move the code-ring position to main chunk m_base + c (at most one wrap:
                    // consecutive own chunks are <= NG <= c_stages main chunks apart)
                    cs += (m_base + c) - m_cur;
                    m_cur = m_base + c;
                    if (cs >= c_stages) { cs -= c_stages; cph ^= 1u; }
                }
                {
                    // registers: the packed words of the chunk (kSW x BITS) plus ONE
                    // super-word of fp16 pairs at a time -- dequantize, tcgen05.st, reuse
                    if (main_chunk) {
                        const int kc = un.kc_begin + c;
#ifdef TQ_PROFILE
                        const long long tcf0 = clock64();
#endif
                        mbar_wait(&hdr->c_full[cs], cph);
                        if (tr) trace_ev(p, 4, grp * 1024 + tcnt);
                        const uint8_t* st = smem + c_off + cs * kCStage;
                        const uint32_t* wst = reinterpret_cast<const uint32_t*>(st) + rloc;
                        constexpr int kHalf = kWords * kBM;
                        if constexpr (BITS == kDenseBits) {
                            // dense fp16 operand (projection pass): stream each super-word smem -> TMEM
                            TQ_TIMED(1, mbar_wait(&hdr->empty[as], aph ^ 1u));
                            tc_fence_after();
#pragma unroll
                            for (int s = 0; s < kSW; ++s) {
                                uint32_t v[16];
#pragma unroll
                                for (int w = 0; w < 16; ++w)
                                    v[w] = wst[(s >> 1) * (kBlk / 4) + (s & 1) * kHalf + w * kBM];
                                tc_st_32x32b_x16(tmem + lane_base + as * kACols + s * 16, v);
                            }
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&hdr->c_empty[cs]);
                        } else {
                            // all packed words of the chunk in registers, stage released, then
                            // one super-word of fp16 pairs at a time: dequantize, tcgen05.st
                            uint32_t words[kSW][kWords];
                            uint16_t sbits[kSW];
                            const int e0 = kc * KC;
                            const int ein = gshift >= 0 ? (e0 & ((1 << gshift) - 1)) : e0 % p.group_size;
                            const uint16_t* sc = reinterpret_cast<const uint16_t*>(st + kCBytes) + rloc;
#pragma unroll
                            for (int s = 0; s < kSW; ++s) {   // super-word s: 64-column block s/2, half s%2
#pragma unroll
                                for (int w = 0; w < kWords; ++w)
                                    words[s][w] = wst[(s >> 1) * (kBlk / 4) + (s & 1) * kHalf + w * kBM];
                                const int off = ein + 32 * s;
                                // a super-word past in_dim (zero codes) may lie past the last group
                                const int gi = min(gshift >= 0 ? off >> gshift : off / p.group_size,
                                                   p.groups - 1 - (gshift >= 0 ? e0 >> gshift : e0 / p.group_size));
                                sbits[s] = sc[gi * kBM];
                            }
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&hdr->c_empty[cs]);
#ifdef TQ_PROFILE
                            prof[1] += clock64() - tcf0;
#endif
                            TQ_TIMED(3, mbar_wait(&hdr->empty[as], aph ^ 1u));
#if !defined(TQ_TRACE_PROD) && !defined(TQ_TRACE_UNIT)
                            if (tr) trace_ev(p, 5, grp * 1024 + tcnt);
#endif
                            tc_fence_after();
#ifdef TQ_PROFILE
                            const long long tdq0 = clock64();
#endif
#pragma unroll
                            for (int s = 0; s < kSW; ++s) {
                                uint32_t v[16];
                                if (kDbg & 1) {
#pragma unroll
                                    for (int w = 0; w < 16; ++w) v[w] = words[s][w % kWords];
                                } else {
                                    const DqConst dq = make_dq(__ushort_as_half(sbits[s]));
                                    dequant32<BITS>(words[s], dq, v);
                                }
                                if (!(kDbg & 64)) tc_st_32x32b_x16(tmem + lane_base + as * kACols + s * 16, v);
                                else {
#pragma unroll
                                    for (int w = 0; w < 16; ++w) asm volatile("" ::"r"(v[w]));
                                }
                            }
#ifdef TQ_PROFILE
                            prof[2] += clock64() - tdq0;
#endif
                        }
                    } else {
                        // extension chunk: precomputed fp16 columns [-zero*s per group | U_p codes | 0]
                        {
                            const int need = (eo - p.e_slots + 1) * ext_per_block;
                            while (*ext_arrivals < need) __nanosleep(20);
                        }
                        TQ_TIMED(0, mbar_wait(&hdr->e_full[es], eph));
                        const uint32_t* eb = reinterpret_cast<const uint32_t*>(smem + e_off + es * ext_bytes) + rloc;
                        TQ_TIMED(1, mbar_wait(&hdr->empty[as], aph ^ 1u));
#if !defined(TQ_TRACE_PROD) && !defined(TQ_TRACE_UNIT)
                        if (tr) trace_ev(p, 5, grp * 1024 + tcnt);
#endif
                        tc_fence_after();
#pragma unroll
                        for (int s = 0; s < kSW; ++s) {
                            const int colbase = (c - nmain) * KC + 32 * s;
                            const int blk = colbase >> 6, hh = (colbase >> 5) & 1;
                            uint32_t v[16];
                            if (blk < p.n_ext64) {   // blocks past the last real one are never read by the MMA
#pragma unroll
                                for (int w = 0; w < 16; ++w)
                                    v[w] = eb[blk * (code_block_bytes(kDenseBits) / 4) + (hh * 16 + w) * kBM];
                                tc_st_32x32b_x16(tmem + lane_base + as * kACols + s * 16, v);
                            }
                        }
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(&hdr->e_empty[es]);
                            atomicAdd(const_cast<int*>(ext_arrivals), 1);
                        }
                    }
                    if (!(kDbg & 64)) tc_wait_st();
                    if (kGX && p.x_atom_rows == 0) {
                        cp_async_wait_group1();          // this chunk's tile landed (the next may be in flight)
                        fence_proxy_async_smem();        // generic-proxy cp.async writes -> MMA operand reads
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&hdr->full[as]);
                    if (lane == 0 && q == 0)
                        trace_id(p, 4 + (grp & 3), tcnt,
                                 (static_cast<unsigned long long>(u - first) << 40) | (static_cast<unsigned long long>(c) << 24) |
                                     (static_cast<unsigned long long>(nmain) << 8) | (main_chunk ? 1ull : 0ull) |
                                     (static_cast<unsigned long long>(as) << 16) | (static_cast<unsigned long long>(es) << 4));
#if !defined(TQ_TRACE_PROD) && !defined(TQ_TRACE_UNIT)
                    if (tr) trace_ev(p, 6, grp * 1024 + tcnt);
#endif
#ifndef TQ_TRACE_UNIT
                    if (lane == 0 && grp == 0) trace_ev(p, 7, q * 1024 + tcnt);   // per-warp skew of group 0
#endif
                    ++tcnt;
                }
                as += NG;
                if (as >= kAS) { as -= kAS; aph ^= 1u; }
            }
            c_next = c - nch;
            q_base += nch;
            m_base += nmain;
            if (un.n_ext > 0 && p.n_ext64 > 0) {
                ++eo;
                if (++es == p.e_slots) { es = 0; eph ^= 1u; }
            }
        }
    } else if (warp >= kEpi0) {
        // ===================== epilogue =====================
        const int q = wid & 3;  // TMEM lane quarter = physical warp id % 4
        int lu = 0;
        int q_base_e = 0;       // CTA-wide chunk index of the unit's first chunk
        Unit nxt = first < n_units ? unit_at(first) : Unit{};
        float nscale = first < n_units ? p.w_outscale[nxt.weight] : 1.0f;
        for (int u = first; u < n_units; u += stride, ++lu) {
            const Unit un = nxt;
            const float oscale = nscale;
            if (u + stride < n_units) {
                nxt = unit_at(u + stride);
                nscale = p.w_outscale[nxt.weight];
            }
            const int ds = lu & 1;
            const uint32_t dph = (lu >> 1) & 1;
            const int row = un.mb * kBM + q * 32 + lane;
            const bool valid = row < p.o_valid;
            float* out = p.y + static_cast<int64_t>(un.split) * p.y_split_stride +
                         static_cast<int64_t>(un.y_row) * p.ldy + row;
            TQ_TIMED(0, mbar_wait_sleep(&hdr->d_full[ds], dph));
#ifdef TQ_TRACE_UNIT
            if (lane == 0 && q == 0) trace_ev(p, 5, lu);
#endif
            tc_fence_after();
            const uint32_t dbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + kDCol0 + ds * NI * DN;
            const int nch = (un.kc_end - un.kc_begin) + un.n_ext;
            // issuer j took part iff the unit holds a chunk whose CTA-wide index is j mod NI
            bool part[NI];
#pragma unroll
            for (int jj = 0; jj < NI; ++jj) part[jj] = nch >= NI || ((jj - q_base_e % NI + NI) % NI) < nch;
            q_base_e += nch;
            for (int t0 = 0; t0 < un.n_tok; t0 += 16) {
                uint32_t v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = 0u;
#pragma unroll
                for (int jj = 0; jj < NI; ++jj) {   // fixed order: deterministic sum of the partials
                    if (!part[jj]) continue;
                    uint32_t w[16];
                    tc_ld_32x32b_x16(dbase + jj * DN + t0, w);
                    tc_wait_ld();
#pragma unroll
                    for (int k = 0; k < 16; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) + __uint_as_float(w[k]));
                }
                if (valid && !(kDbg & 4)) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (t0 + j < un.n_tok) out[static_cast<int64_t>(t0 + j) * p.ldy] = __uint_as_float(v[j]) * oscale;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->d_empty[ds]);
#ifdef TQ_TRACE_UNIT
            if (lane == 0 && q == 0) trace_ev(p, 6, lu);
#endif
        }
    }

#ifdef TQ_PROFILE
    if (lane == 0 && p.trace) {
        unsigned long long* o = p.trace + (static_cast<size_t>(blockIdx.x) * 32 + wid) * 8;
        o[0] = clock64() - prof_t0;
        o[1] = warp;
        for (int k = 0; k < 4; ++k) o[2 + k] = prof[k];
        o[6] = prologue_cycles;
        o[7] = g_entry;   // globaltimer (ns) at kernel entry of this warp
    }
#endif
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
#ifdef TQ_PROFILE
    if (threadIdx.x == 0 && p.trace) {
        // row 31: per-CTA summary (word 0 stays 0 so per-warp views skip it)
        unsigned long long* o = p.trace + (static_cast<size_t>(blockIdx.x) * 32 + 31) * 8;
        unsigned long long g_exit;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
        o[0] = 0;
        o[1] = static_cast<unsigned long long>(first < n_units ? (n_units - first + stride - 1) / stride : 0);
        o[7] = g_exit;
    }
#endif
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                     : "memory");
    }
}

// -----------------------------------------------------------------------------

cudaError_t launch_gemm(const GemmParams& p0, int grid, cudaStream_t stream) {
    GemmParams p = p0;
    const int kc = p.kc_width;
    const int dn = p.dn;
    const bool cfg_ok = (kc == 128 && (dn == 32 || dn == 64 || dn == 128)) || (kc == 64 && dn == 192);
    if (!cfg_ok) return cudaErrorInvalidValue;
    if (p.bn_max > dn) return cudaErrorInvalidValue;
    // activation ring: stage rows = token tile rounded to the box (64) or the MMA N granularity (16)
    const int rows = p.bn_max > 48 ? ((p.bn_max + 63) / 64) * 64 : ((p.bn_max + 15) / 16) * 16;  // cp.async tiles: 16-row granules
    p.x_stage_rows = rows;
    const int x_stage = (kc / kKC) * rows * 128;
    const int c_stage = code_stage_bytes(p.bits, kc);
    if (p.e_slots != 1) p.e_slots = 2;
    const int fixed = kHdrBytes + kUnitCache * static_cast<int>(sizeof(Unit)) + p.e_slots * ext_slot_bytes(p.n_ext64);
    const int ni = (kc == 128 && dn <= 64) ? (dn == 32 ? TQ_DECODE_NI : 2) : 1;
    const int as_n = a_stages(kc, dn, ni);
    int cs, xs;
    if (dn == 32) {
        // resident activation slots, one per chunk of a unit; codes get the rest
        if (p.xr_slots < 1 || p.xr_slots > kMaxXStages || p.x_atom_rows <= 0) return cudaErrorInvalidValue;
        xs = p.xr_slots;
        cs = (kSmemBudget - fixed - xs * x_stage) / c_stage;
        cs = cs < kMaxCStages ? cs : kMaxCStages;
        if (cs < 4) return cudaErrorInvalidValue;
    } else {
        // >= 80 KB of packed-code stages in flight (HBM latency), the activation
        // ring as deep as the rest allows (<= 16), leftovers to codes
        cs = (80 * 1024 + c_stage - 1) / c_stage;
        xs = (kSmemBudget - fixed - cs * c_stage) / x_stage;
        xs = xs < 16 ? xs : 16;
        if (xs < as_n) xs = as_n;
        cs = (kSmemBudget - fixed - xs * x_stage) / c_stage;
        cs = cs < kMaxCStages ? cs : kMaxCStages;
        if (cs < 2 || xs < 2) return cudaErrorInvalidValue;
    }
    p.x_stages = xs;
    p.c_stages = cs;
    p.group_shift = -1;
    for (int s = 0; s < 16; ++s)
        if ((1 << s) == p.group_size) p.group_shift = s;
    const int smem = 1024 + xs * x_stage + cs * c_stage + p.e_slots * ext_slot_bytes(p.n_ext64) + kHdrBytes +
                     kUnitCache * static_cast<int>(sizeof(Unit));
    static const int dbg = getenv("TQ_DEBUG") ? atoi(getenv("TQ_DEBUG")) : 0;
    p.debug = dbg;
    static unsigned long long* trace_buf = nullptr;
    constexpr size_t kTraceWords = 160 * 32 * 8;   // >= 8 x 4096 event slots, and 8 words per warp of 160 CTAs
    if ((dbg & 8) && !trace_buf) {
        cudaMalloc(&trace_buf, kTraceWords * sizeof(unsigned long long));
        cudaMemset(trace_buf, 0, kTraceWords * sizeof(unsigned long long));
    }
    p.trace = trace_buf;
    cudaError_t err = cudaSuccess;
    auto go = [&](auto kern, int threads) {
        // the attribute is raised once per kernel (launches may be captured into graphs);
        // all instantiations share one function-pointer type, so key by address
        static const void* cfg_fn[64];
        static int cfg_smem[64];
        static int cfg_n = 0;
        int slot = -1;
        for (int t = 0; t < cfg_n; ++t)
            if (cfg_fn[t] == reinterpret_cast<const void*>(kern)) slot = t;
        if (slot < 0 && cfg_n < 64) {
            slot = cfg_n++;
            cfg_fn[slot] = reinterpret_cast<const void*>(kern);
            cfg_smem[slot] = 0;
        }
        if (slot < 0 || smem > cfg_smem[slot]) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (err != cudaSuccess) return;
            if (slot >= 0) cfg_smem[slot] = smem;
        }
        err = launch_maybe_pdl(kern, dim3(grid), dim3(threads), smem, stream, p);
    };
#define TQ_GEMM_CASES(KCV, NGV, DNV, NIV)                                                                 \
    switch (p.bits) {                                                                              \
        case 2: go(gemm_kernel<2, KCV, NGV, DNV, NIV>, gemm_threads(NGV)); break;                  \
        case 3: go(gemm_kernel<3, KCV, NGV, DNV, NIV>, gemm_threads(NGV)); break;                  \
        case 4: go(gemm_kernel<4, KCV, NGV, DNV, NIV>, gemm_threads(NGV)); break;                  \
        case 8: go(gemm_kernel<8, KCV, NGV, DNV, NIV>, gemm_threads(NGV)); break;                  \
        case kDenseBits: go(gemm_kernel<kDenseBits, KCV, NGV, DNV, NIV>, gemm_threads(NGV)); break; \
        default: return cudaErrorInvalidValue;                                                     \
    }
    if (kc == 128 && dn == 32) {
        TQ_GEMM_CASES(128, 4, 32, TQ_DECODE_NI)
    } else if (kc == 128 && dn == 64) {
        TQ_GEMM_CASES(128, 4, 64, 2)
    } else if (kc == 128) {
        TQ_GEMM_CASES(128, 3, 128, 1)
    } else {
        TQ_GEMM_CASES(64, 2, 192, 1)
    }
#undef TQ_GEMM_CASES
    if (err == cudaSuccess && (dbg & 8) && getenv("TQ_TRACE_FILE")) {
        // debug only: dump CTA 0's event trace of this launch (8 slots x 4096 u64)
        static unsigned long long host[kTraceWords];
        cudaStreamSynchronize(stream);
        cudaMemcpy(host, trace_buf, sizeof(host), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(getenv("TQ_TRACE_FILE"), "wb")) {
            fwrite(host, 1, sizeof(host), f);
            fclose(f);
        }
        cudaMemset(trace_buf, 0, sizeof(host));
    }
    return err;
}

}  // namespace tqb
