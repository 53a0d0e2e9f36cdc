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
#include <cuda_fp16.h>

#include "tq_internal.h"

namespace tqb {

// =============================================================================
// PTX helpers
// =============================================================================

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TQ_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TQ_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16, fp32 accumulate, cta_group::1.
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tc_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, rows of
// 128 B, 8-row core-matrix groups 1024 B apart (SBO), sm_100 version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;                 // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;         // SBO
    d |= static_cast<uint64_t>(1u) << 46;                 // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2u) << 61;                 // SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::f16, A=B=F16, D=F32, both K-major, M=128.
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n) {
    return (1u << 4) | ((n >> 3) << 17) | ((uint32_t(kBM) >> 4) << 24);
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t orv) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(orv));  // (a & b) | c
    return r;
}

__device__ __forceinline__ uint32_t hfma2_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// =============================================================================
// in-register dequant: 32 consecutive codes of one row -> 16 half2 = code * s
// =============================================================================
//
// Super-word encodings (written by the loader, tq_runtime.cpp pack_superword):
// pair p holds codes (c_{2p}, c_{2p+1}) in the low / high 16-bit half of a
// word at bit offset `pos` inside the half.  A field at pos (pos + b <= 10)
// is turned into fp16 by OR-ing the exponent 25-pos: value = 2^(10-pos) +
// code exactly; one HFMA2 with s and bias = -2^(10-pos)*s yields code*s with
// a single rounding.  Fields above bit 9 are shifted down first.

__device__ __forceinline__ uint32_t magic_for(int pos) {
    const uint32_t e = static_cast<uint32_t>(25 - pos) << 10;
    return e | (e << 16);
}

struct DqConst {
    uint32_t s2;         // half2 (s, s)
    uint32_t bias[10];   // bias for field position pos (index pos): -2^(10-pos) * s
};

__device__ __forceinline__ DqConst make_dq(__half s) {
    DqConst c;
    const __half2 s2 = __half2half2(s);
    c.s2 = *reinterpret_cast<const uint32_t*>(&s2);
#pragma unroll
    for (int pos = 0; pos < 10; ++pos) {
        uint32_t m = 0x8000u | (static_cast<uint32_t>(25 - pos) << 10);  // -2^(10-pos) in fp16
        m |= m << 16;
        c.bias[pos] = hmul2_u32(c.s2, m);
    }
    return c;
}

__device__ __forceinline__ uint32_t dq_field(uint32_t w, int pos, int bits, const DqConst& c) {
    const uint32_t fmask = ((1u << bits) - 1u) << pos;
    return hfma2_u32(lop3_and_or(w, fmask | (fmask << 16), magic_for(pos)), c.s2, c.bias[pos]);
}

template <int BITS>
__device__ __forceinline__ void dequant32(const uint32_t* w, const DqConst& c, uint32_t (&out)[16]);

template <>
__device__ __forceinline__ void dequant32<2>(const uint32_t* w, const DqConst& c, uint32_t (&out)[16]) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const uint32_t v = w[j];
        const uint32_t u = v >> 10;
        out[8 * j + 0] = dq_field(v, 0, 2, c);
        out[8 * j + 1] = dq_field(v, 2, 2, c);
        out[8 * j + 2] = dq_field(v, 4, 2, c);
        out[8 * j + 3] = dq_field(v, 6, 2, c);
        out[8 * j + 4] = dq_field(v, 8, 2, c);
        out[8 * j + 5] = dq_field(u, 0, 2, c);
        out[8 * j + 6] = dq_field(u, 2, 2, c);
        out[8 * j + 7] = dq_field(u, 4, 2, c);
    }
}

template <>
__device__ __forceinline__ void dequant32<3>(const uint32_t* w, const DqConst& c, uint32_t (&out)[16]) {
    uint32_t u[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const uint32_t v = w[j];
        u[j] = v >> 9;
        out[5 * j + 0] = dq_field(v, 0, 3, c);
        out[5 * j + 1] = dq_field(v, 3, 3, c);
        out[5 * j + 2] = dq_field(v, 6, 3, c);
        out[5 * j + 3] = dq_field(u[j], 0, 3, c);
        out[5 * j + 4] = dq_field(u[j], 3, 3, c);
    }
    // pair 15: bit k of (c30, c31) sits at bits (15, 31) of word k -> (6, 22) of u[k]
    uint32_t t = lop3_and_or(u[0], 0x00400040u, magic_for(6));
    t = lop3_and_or(u[1] << 1, 0x00800080u, t);
    t = lop3_and_or(u[2] << 2, 0x01000100u, t);
    out[15] = hfma2_u32(t, c.s2, c.bias[6]);
}

template <>
__device__ __forceinline__ void dequant32<4>(const uint32_t* w, const DqConst& c, uint32_t (&out)[16]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t v = w[j];
        const uint32_t u = v >> 8;
        out[4 * j + 0] = dq_field(v, 0, 4, c);
        out[4 * j + 1] = dq_field(v, 4, 4, c);
        out[4 * j + 2] = dq_field(u, 0, 4, c);
        out[4 * j + 3] = dq_field(u, 4, 4, c);
    }
}

template <>
__device__ __forceinline__ void dequant32<8>(const uint32_t* w, const DqConst& c, uint32_t (&out)[16]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t v = w[j];
        out[2 * j + 0] = dq_field(v, 0, 8, c);
        out[2 * j + 1] = dq_field(v >> 8, 0, 8, c);
    }
}

// =============================================================================
// the fused grouped GEMM
// =============================================================================

constexpr int kThreads = 512;          // 16 warps
constexpr int kXStages = 4;
constexpr int kXStageBytes = kBNMax * 128;   // 24 KB
constexpr int kAStages = 4;
constexpr int kACols = kKC / 2;        // 32 TMEM columns per A stage (128 x 64 fp16)
constexpr int kDCol0 = kAStages * kACols;  // 128
constexpr int kTmemCols = 512;
constexpr int kCodeRingBytes = 48 * 1024;
constexpr int kScaleTrailer = 2 * kBM * 2;  // two 128-row fp16 scale slices (one per 32-column half)
constexpr int kMaxCStages = 16;

__host__ __device__ constexpr int code_stage_bytes(int bits) {
    return code_block_bytes(bits) + (bits == kDenseBits ? 0 : kScaleTrailer);
}
__host__ __device__ constexpr int code_stages(int bits) {
    return (kCodeRingBytes / code_stage_bytes(bits)) < kMaxCStages ? (kCodeRingBytes / code_stage_bytes(bits))
                                                                   : kMaxCStages;
}
// extension tables of one (weight, m-block): scales [G][128] fp16, zeros [G][128] u8, U [128][r] int8
__host__ __device__ inline int ext_slot_bytes(int groups, int rank) {
    return (groups * kBM * 3 + kBM * rank + 1023) & ~1023;
}

struct SharedHdr {
    uint64_t x_full[kXStages], x_empty[kXStages];
    uint64_t a_full[kAStages], a_empty[kAStages];
    uint64_t c_full[kMaxCStages], c_empty[kMaxCStages];
    uint64_t d_full[2], d_empty[2];
    uint64_t e_full[2], e_empty[2];
    uint32_t tmem_base;
};

__host__ int gemm_smem_bytes(int groups, int rank) {
    return 1024 + kXStages * kXStageBytes + kCodeRingBytes + 2 * ext_slot_bytes(groups, rank) + 1024;
}

template <int BITS>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kCBytes = code_block_bytes(BITS);
    constexpr int kCStage = code_stage_bytes(BITS);
    constexpr int kCStages = code_stages(BITS);
    constexpr int kWords = BITS;  // u32 words per 32 codes of one row (dense fp16: 16)
    const int ext_bytes = ext_slot_bytes(p.groups, p.rank);
    uint8_t* x_smem = smem;
    uint8_t* c_smem = smem + kXStages * kXStageBytes;
    uint8_t* e_smem = c_smem + kCodeRingBytes;
    SharedHdr* hdr = reinterpret_cast<SharedHdr*>(e_smem + 2 * ext_bytes);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int n_units = *p.n_units;

    if (threadIdx.x == 0) {
        prefetch_tmap(&p.tmap_x16);
        prefetch_tmap(&p.tmap_x64);
        prefetch_tmap(&p.tmap_e16);
        prefetch_tmap(&p.tmap_e64);
        for (int s = 0; s < kXStages; ++s) {
            mbar_init(&hdr->x_full[s], 1);
            mbar_init(&hdr->x_empty[s], 1);
        }
        for (int s = 0; s < kAStages; ++s) {
            mbar_init(&hdr->a_full[s], 8);
            mbar_init(&hdr->a_empty[s], 1);
        }
        for (int s = 0; s < kCStages; ++s) {
            mbar_init(&hdr->c_full[s], 1);
            mbar_init(&hdr->c_empty[s], 8);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&hdr->d_full[s], 1);
            mbar_init(&hdr->d_empty[s], 4);
            mbar_init(&hdr->e_full[s], 1);
            mbar_init(&hdr->e_empty[s], 8);
        }
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
    const uint32_t tmem = hdr->tmem_base;
    const int64_t slab_groups = static_cast<int64_t>(p.groups) * kBM;  // scale/zero entries per (w, mb)

    if (warp == 0) {
        // ===================== producer: TMA activations + bulk weight blocks =====================
        if (lane == 0) {
            int xs = 0, cs = 0, es = 0;
            uint32_t xph = 0, cph = 0, eph = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const Unit un = p.units[u];
                const int nmain = un.kc_end - un.kc_begin;
                const int nch = nmain + un.n_ext;
                const bool big = un.n_tok > 32;
                const int box_rows = big ? 64 : 16;
                const int nbox = (un.n_tok + box_rows - 1) / box_rows;
                const int64_t wm = static_cast<int64_t>(un.weight) * (p.o_pad / kBM) + un.mb;  // (w, mb) slab
                const uint8_t* wbase = p.codes + static_cast<int64_t>(un.weight) * p.weight_stride +
                                       static_cast<int64_t>(un.mb) * p.kc_total * kCBytes;
                for (int c = 0; c < nch; ++c) {
                    const bool ext = c >= nmain;
                    if (!ext) {
                        const int kc = un.kc_begin + c;
                        mbar_wait(&hdr->c_empty[cs], cph ^ 1u);
                        uint8_t* st = c_smem + cs * kCStage;
                        if constexpr (BITS == kDenseBits) {
                            mbar_arrive_expect_tx(&hdr->c_full[cs], kCBytes);
                            bulk_copy_g2s(st, wbase + static_cast<int64_t>(kc) * kCBytes, kCBytes, &hdr->c_full[cs]);
                        } else {
                            mbar_arrive_expect_tx(&hdr->c_full[cs], kCBytes + kScaleTrailer);
                            bulk_copy_g2s(st, wbase + static_cast<int64_t>(kc) * kCBytes, kCBytes, &hdr->c_full[cs]);
                            for (int h = 0; h < 2; ++h) {
                                const int g = (kc * kKC + 32 * h) / p.group_size;
                                bulk_copy_g2s(st + kCBytes + h * kBM * 2, p.scales + (wm * p.groups + g) * kBM,
                                              kBM * 2, &hdr->c_full[cs]);
                            }
                        }
                        if (++cs == kCStages) { cs = 0; cph ^= 1u; }
                    } else if (c == nmain) {
                        const int ub = p.w_ublock[un.weight];
                        mbar_wait(&hdr->e_empty[es], eph ^ 1u);
                        uint8_t* eb = e_smem + es * ext_bytes;
                        const uint32_t zb = static_cast<uint32_t>(slab_groups);
                        const uint32_t ubytes = (ub >= 0) ? static_cast<uint32_t>(kBM * p.rank) : 0u;
                        mbar_arrive_expect_tx(&hdr->e_full[es], zb * 2 + zb + ubytes);
                        bulk_copy_g2s(eb, p.scales + wm * slab_groups, zb * 2, &hdr->e_full[es]);
                        bulk_copy_g2s(eb + zb * 2, p.zeros + wm * slab_groups, zb, &hdr->e_full[es]);
                        if (ub >= 0)
                            bulk_copy_g2s(eb + zb * 3,
                                          p.ucodes + (static_cast<int64_t>(ub) * p.o_pad + un.mb * kBM) * p.rank,
                                          ubytes, &hdr->e_full[es]);
                        if (++es == 2) { es = 0; eph ^= 1u; }
                    }
                    mbar_wait(&hdr->x_empty[xs], xph ^ 1u);
                    mbar_arrive_expect_tx(&hdr->x_full[xs], nbox * box_rows * 128);
                    const CUtensorMap* map =
                        ext ? (big ? &p.tmap_e64 : &p.tmap_e16) : (big ? &p.tmap_x64 : &p.tmap_x16);
                    const int col = ext ? (c - nmain) * kKC : (un.kc_begin + c) * kKC;
                    for (int bx = 0; bx < nbox; ++bx)
                        tma_load_2d(x_smem + xs * kXStageBytes + bx * box_rows * 128, map, col,
                                    un.x_row + bx * box_rows, &hdr->x_full[xs]);
                    if (++xs == kXStages) { xs = 0; xph ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (single thread) =====================
        if (lane == 0) {
            int xs = 0, as = 0, lu = 0;
            uint32_t xph = 0, aph = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
                const Unit un = p.units[u];
                const int nch = (un.kc_end - un.kc_begin) + un.n_ext;
                const int ds = lu & 1;
                const uint32_t dph = (lu >> 1) & 1;
                const uint32_t n = static_cast<uint32_t>((un.n_tok + 15) & ~15);
                const uint32_t idesc = idesc_f16(n);
                const uint32_t d_tmem = tmem + kDCol0 + ds * kBNMax;
                mbar_wait(&hdr->d_empty[ds], dph ^ 1u);
                tc_fence_after();
                for (int c = 0; c < nch; ++c) {
                    mbar_wait(&hdr->a_full[as], aph);
                    mbar_wait(&hdr->x_full[xs], xph);
                    tc_fence_after();
                    const uint32_t xaddr = smem_u32(x_smem + xs * kXStageBytes);
#pragma unroll
                    for (int k = 0; k < kKC / 16; ++k) {
                        tc_mma_ts(d_tmem, tmem + as * kACols + k * 8, sw128_desc(xaddr + k * 32), idesc,
                                  (c > 0 || k > 0) ? 1u : 0u);
                    }
                    tc_commit(&hdr->a_empty[as]);
                    tc_commit(&hdr->x_empty[xs]);
                    if (++as == kAStages) { as = 0; aph ^= 1u; }
                    if (++xs == kXStages) { xs = 0; xph ^= 1u; }
                }
                tc_commit(&hdr->d_full[ds]);
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ===================== dequant warps: codes -> fp16 -> TMEM (A operand) =====================
        const int q = warp & 3;
        const int h = (warp - 4) >> 2;
        const int rloc = q * 32 + lane;
        int cs = 0, as = 0, es = 0;
        uint32_t cph = 0, aph = 0, eph = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const Unit un = p.units[u];
            const int nmain = un.kc_end - un.kc_begin;
            const int nch = nmain + un.n_ext;
            const int ub = p.w_ublock[un.weight];
            for (int c = 0; c < nch; ++c) {
                uint32_t v[16];
                if (c < nmain) {
                    mbar_wait(&hdr->c_full[cs], cph);
                    const uint8_t* st = c_smem + cs * kCStage;
                    const uint32_t* blk = reinterpret_cast<const uint32_t*>(st);
                    uint32_t words[kWords];
#pragma unroll
                    for (int j = 0; j < kWords; ++j) words[j] = blk[(h * kWords + j) * kBM + rloc];
                    if constexpr (BITS == kDenseBits) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&hdr->c_empty[cs]);
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = words[j];
                    } else {
                        const __half s = reinterpret_cast<const __half*>(st + kCBytes)[h * kBM + rloc];
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&hdr->c_empty[cs]);
                        const DqConst dq = make_dq(s);
                        dequant32<BITS>(words, dq, v);
                    }
                    if (++cs == kCStages) { cs = 0; cph ^= 1u; }
                } else {
                    // extension chunk: columns [-zero*s per group | U_p codes | 0]
                    if (c == nmain) mbar_wait(&hdr->e_full[es], eph);
                    const uint8_t* eb = e_smem + es * ext_bytes;
                    const __half* es_s = reinterpret_cast<const __half*>(eb);
                    const uint8_t* es_z = eb + slab_groups * 2;
                    const int8_t* es_u = reinterpret_cast<const int8_t*>(eb + slab_groups * 3);
                    const int colbase = (c - nmain) * kKC + 32 * h;
                    const int zcols = p.groups;  // extension layout is fixed: [groups | rank | pad]
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        __half hv[2];
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) {
                            const int col = colbase + 2 * j + e2;
                            __half val = __float2half_rn(0.0f);
                            if (col < zcols) {
                                if (!p.ext_zero) {
                                    hv[e2] = val;
                                    continue;
                                }
                                const __half s = es_s[col * kBM + rloc];
                                const __half z = __float2half_rn(static_cast<float>(es_z[col * kBM + rloc]));
                                val = __hneg(__hmul(z, s));
                            } else if (ub >= 0 && col - zcols < p.rank) {
                                val = __float2half_rn(static_cast<float>(es_u[rloc * p.rank + (col - zcols)]));
                            }
                            hv[e2] = val;
                        }
                        const __half2 h2 = __halves2half2(hv[0], hv[1]);
                        v[j] = *reinterpret_cast<const uint32_t*>(&h2);
                    }
                    if (c == nch - 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&hdr->e_empty[es]);
                        if (++es == 2) { es = 0; eph ^= 1u; }
                    }
                }
                mbar_wait(&hdr->a_empty[as], aph ^ 1u);
                tc_fence_after();
                tc_st_32x32b_x16(tmem + (static_cast<uint32_t>(q * 32) << 16) + as * kACols + h * 16, v);
                tc_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&hdr->a_full[as]);
                if (++as == kAStages) { as = 0; aph ^= 1u; }
            }
        }
    } else if (warp >= 12) {
        // ===================== epilogue: TMEM -> registers -> global =====================
        const int q = warp & 3;
        int lu = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
            const Unit un = p.units[u];
            const int ds = lu & 1;
            const uint32_t dph = (lu >> 1) & 1;
            const int row = un.mb * kBM + q * 32 + lane;
            const bool valid = row < p.o_valid;
            const float oscale = p.w_outscale[un.weight];
            float* out = p.y + static_cast<int64_t>(un.split) * p.y_split_stride +
                         static_cast<int64_t>(un.y_row) * p.ldy + row;
            mbar_wait(&hdr->d_full[ds], dph);
            tc_fence_after();
            const uint32_t dbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + kDCol0 + ds * kBNMax;
            for (int t0 = 0; t0 < un.n_tok; t0 += 16) {
                uint32_t v[16];
                tc_ld_32x32b_x16(dbase + t0, v);
                tc_wait_ld();
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (t0 + j < un.n_tok)
                            out[static_cast<int64_t>(t0 + j) * p.ldy] = __uint_as_float(v[j]) * oscale;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->d_empty[ds]);
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                     : "memory");
    }
}

// =============================================================================
// router: bit-exact route() (moe.cpp:43-89)
// =============================================================================

// Per token: scores[k] = float(sum_c double(x[c]) * double(G[k,c])) with the
// reference's sequential index-order f64 sum (matrix.cpp:25-36).  The warp
// computes a parallel f64 sum plus sum|p|; the reference result differs from
// ours by at most (gamma_{i-1} + gamma_{i/32+5}) * sum|p| (every product is
// exact in f64), so if both ends of that interval round to the same f32 the
// f32 score is certified identical; otherwise lane 0 replays the sequential
// loop.  Then f64 max-subtracted softmax, total summed k = 0..K-1, ordering
// by (prob desc, index asc), gates = float(prob / selected).
__global__ void __launch_bounds__(256) route_kernel(const float* __restrict__ x, int in_dim,
                                                   const float* __restrict__ gate, int num_experts, int top_k,
                                                   int group_size, int groups, int k_pad,
                                                   int32_t* __restrict__ ids, float* __restrict__ gates,
                                                   __half* __restrict__ x16, float* __restrict__ sx) {
    extern __shared__ __align__(16) float rs_smem[];
    float* xs = rs_smem;                 // in_dim
    float* scores = rs_smem + in_dim;    // num_experts
    const int b = blockIdx.x;
    const float* xb = x + static_cast<int64_t>(b) * in_dim;
    for (int c = threadIdx.x; c < in_dim; c += blockDim.x) xs[c] = xb[c];
    __syncthreads();
    // fp16 activations (zero-padded to k_pad) and per-group sums of them
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    if (x16) {
        __half* xo = x16 + static_cast<int64_t>(b) * k_pad;
        for (int c = threadIdx.x; c < k_pad; c += blockDim.x) xo[c] = __float2half_rn(c < in_dim ? xs[c] : 0.0f);
    }
    for (int g = warp; sx && g < groups; g += nwarps) {
        float acc = 0.0f;
        const int c0 = g * group_size, c1 = min(in_dim, c0 + group_size);
        for (int c = c0 + lane; c < c1; c += 32) acc += __half2float(__float2half_rn(xs[c]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
        if (lane == 0) sx[static_cast<int64_t>(b) * groups + g] = acc;
    }
    if (num_experts == 0) return;  // activations-only prep (tq_forward with given routing)
    // certified scores
    for (int k = warp; k < num_experts; k += nwarps) {
        const float* gk = gate + static_cast<int64_t>(k) * in_dim;
        double s = 0.0, a = 0.0;
        for (int c = lane; c < in_dim; c += 32) {
            const double prod = static_cast<double>(xs[c]) * static_cast<double>(gk[c]);
            s += prod;
            a += fabs(prod);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            s += __shfl_down_sync(0xffffffffu, s, off);
            a += __shfl_down_sync(0xffffffffu, a, off);
        }
        if (lane == 0) {
            const double u = 1.1102230246251565e-16;  // 2^-53
            const double nterms = static_cast<double>(in_dim) + static_cast<double>((in_dim + 31) / 32) + 8.0;
            const double err = __dmul_ru(__dmul_ru(nterms * u, 1.01), __dmul_ru(a, 1.0001));
            const float lo = __double2float_rn(__dsub_rd(s, err));
            const float hi = __double2float_rn(__dadd_ru(s, err));
            float score;
            if (lo == hi) {
                score = __double2float_rn(s);
            } else {
                double acc = 0.0;  // the reference's exact sequential loop
                for (int c = 0; c < in_dim; ++c) acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(xs[c]),
                                                                                static_cast<double>(gk[c])));
                score = __double2float_rn(acc);
            }
            scores[k] = score;
        }
    }
    __syncthreads();
    if (warp == 0) {
        double mx = -INFINITY;
        for (int k = lane; k < num_experts; k += 32) mx = fmax(mx, static_cast<double>(scores[k]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        // every lane computes the total in the reference order k = 0..K-1
        double total = 0.0;
        for (int k = 0; k < num_experts; ++k) total = __dadd_rn(total, exp(static_cast<double>(scores[k]) - mx));
        double selected = 0.0;
        int picked[64];
        double pprob[64];
        for (int t = 0; t < top_k; ++t) {
            double best_p = -1.0;
            int best_k = 0x7fffffff;
            for (int k = lane; k < num_experts; k += 32) {
                bool taken = false;
                for (int tt = 0; tt < t; ++tt) taken |= (picked[tt] == k);
                if (taken) continue;
                const double pk = __ddiv_rn(exp(static_cast<double>(scores[k]) - mx), total);
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
            picked[t] = best_k;
            pprob[t] = best_p;
            selected = __dadd_rn(selected, best_p);
        }
        if (lane == 0) {
            for (int t = 0; t < top_k; ++t) {
                ids[static_cast<int64_t>(b) * top_k + t] = picked[t];
                gates[static_cast<int64_t>(b) * top_k + t] = __double2float_rn(__ddiv_rn(pprob[t], selected));
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
    // units: routed experts (e, mb, tile, split), then shared (s, mb, tile, split)
    if (threadIdx.x == 0) {
        int nu = 0;
        const int n_slots = tot[K];
        const int ext = a.n_ext;
        for (int e = a.e_begin; e < a.e_end; ++e) {
            const int ne = tot[e + 1] - tot[e];
            const int tiles = (ne + kBNMax - 1) / kBNMax;
            for (int mb = 0; mb < a.mb_count; ++mb)
                for (int tl = 0; tl < tiles; ++tl)
                    for (int sp = 0; sp < a.nsplit; ++sp) {
                        Unit u;
                        u.weight = e - a.e_begin;
                        u.mb = mb;
                        u.x_row = tot[e] + tl * kBNMax;
                        u.n_tok = min(kBNMax, ne - tl * kBNMax);
                        u.y_row = u.x_row;
                        const int k0 = a.main_kc ? sp * a.kc_total / a.nsplit : 0;
                        const int k1 = a.main_kc ? (sp + 1) * a.kc_total / a.nsplit : 0;
                        u.kc_begin = static_cast<int16_t>(k0);
                        u.kc_end = static_cast<int16_t>(k1);
                        u.n_ext = static_cast<int16_t>(sp == a.nsplit - 1 ? ext : 0);
                        u.split = static_cast<int16_t>(sp);
                        u.pad = 0;
                        if (u.kc_end > u.kc_begin || u.n_ext > 0) a.units[nu++] = u;
                    }
        }
        for (int s = 0; s < a.num_shared; ++s) {
            const int tiles = (a.batch + kBNMax - 1) / kBNMax;
            for (int mb = 0; mb < a.mb_count; ++mb)
                for (int tl = 0; tl < tiles; ++tl)
                    for (int sp = 0; sp < a.nsplit; ++sp) {
                        Unit u;
                        u.weight = (a.e_end - a.e_begin) + s;
                        u.mb = mb;
                        u.x_row = n_slots + tl * kBNMax;
                        u.n_tok = min(kBNMax, a.batch - tl * kBNMax);
                        u.y_row = n_slots + s * a.batch + tl * kBNMax;
                        u.kc_begin = static_cast<int16_t>(sp * a.kc_total / a.nsplit);
                        u.kc_end = static_cast<int16_t>((sp + 1) * a.kc_total / a.nsplit);
                        u.n_ext = static_cast<int16_t>(sp == a.nsplit - 1 ? ext : 0);
                        u.split = static_cast<int16_t>(sp);
                        u.pad = 0;
                        a.units[nu++] = u;
                    }
        }
        *a.n_units = nu;
        // projection pass units: stacked projection weight (index 0) x all tokens
        int np = 0;
        if (a.proj_mb > 0) {
            const int tiles = (a.batch + kBNMax - 1) / kBNMax;
            for (int mb = 0; mb < a.proj_mb; ++mb)
                for (int tl = 0; tl < tiles; ++tl)
                    for (int sp = 0; sp < a.proj_nsplit; ++sp) {
                        Unit u;
                        u.weight = 0;
                        u.mb = mb;
                        u.x_row = tl * kBNMax;
                        u.n_tok = min(kBNMax, a.batch - tl * kBNMax);
                        u.y_row = tl * kBNMax;
                        u.kc_begin = static_cast<int16_t>(sp * a.proj_kc_total / a.proj_nsplit);
                        u.kc_end = static_cast<int16_t>((sp + 1) * a.proj_kc_total / a.proj_nsplit);
                        u.n_ext = 0;
                        u.split = static_cast<int16_t>(sp);
                        u.pad = 0;
                        a.proj_units[np++] = u;
                    }
        }
        if (a.n_proj_units) *a.n_proj_units = np;
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
    const int b = blockIdx.y;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.out_dim) return;
    const int n_slots = a.offsets ? a.offsets[a.num_experts] : 0;
    float acc = 0.0f;
    if (a.use_routed) {
        for (int t = 0; t < a.top_k; ++t) {
            const int f = b * a.top_k + t;
            const int pos = a.inv[f];
            if (pos < 0) continue;  // invalid expert id (reported through the error flag)
            float v = 0.0f;
            for (int sp = 0; sp < a.nsplit; ++sp)
                v += a.y[sp * a.split_stride + static_cast<int64_t>(pos) * a.out_dim + c];
            acc = fmaf(a.gates[f], v, acc);
        }
    }
    const int64_t sh0 = a.sh_from_offsets ? n_slots : 0;
    for (int s = 0; s < a.num_shared; ++s) {
        const int64_t r = sh0 + static_cast<int64_t>(s) * a.batch + b;
        float v = 0.0f;
        for (int sp = 0; sp < a.sh_nsplit; ++sp) v += a.ysh[sp * a.sh_split_stride + r * a.out_dim + c];
        acc += v;
    }
    a.out[static_cast<int64_t>(b) * a.out_dim + c] = acc;
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

cudaError_t launch_gemm(const GemmParams& p, int grid, cudaStream_t stream) {
    const int smem = gemm_smem_bytes(p.groups, p.rank);
    cudaError_t err = cudaSuccess;
    auto go = [&](auto kern) {
        err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err != cudaSuccess) return;
        kern<<<grid, kThreads, smem, stream>>>(p);
        err = cudaGetLastError();
    };
    switch (p.bits) {
        case 2: go(gemm_kernel<2>); break;
        case 3: go(gemm_kernel<3>); break;
        case 4: go(gemm_kernel<4>); break;
        case 8: go(gemm_kernel<8>); break;
        case kDenseBits: go(gemm_kernel<kDenseBits>); break;
        default: return cudaErrorInvalidValue;
    }
    return err;
}

cudaError_t launch_route(const float* x, int batch, int in_dim, const float* gate, int num_experts, int top_k,
                         int group_size, int groups, int k_pad, int32_t* ids, float* gates, __half* x16,
                         float* sx, cudaStream_t stream) {
    const size_t smem = sizeof(float) * (static_cast<size_t>(in_dim) + num_experts);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    route_kernel<<<batch, 256, smem, stream>>>(x, in_dim, gate, num_experts, top_k, group_size, groups, k_pad, ids,
                                               gates, x16, sx);
    return cudaGetLastError();
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
    dim3 grid((a.out_dim + 255) / 256, a.batch);
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
