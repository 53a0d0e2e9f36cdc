// PTX helpers and the in-register dequantizers shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#ifdef TQ_WAIT_TRAP
#include <cstdio>
#endif
#include <cuda_fp16.h>

#include "tq_internal.h"

namespace tqb {

// =============================================================================
// PTX helpers
// =============================================================================

static __device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

static __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

static __device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

static __device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef TQ_SPIN_WAIT
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TQ_SPIN_%=:\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TQ_SPIN_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
    return;
#endif
#ifdef TQ_WAIT_HINT
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TQ_WAITH_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra TQ_WAITH_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(static_cast<uint32_t>(TQ_WAIT_HINT))
        : "memory");
    return;
#endif
#ifdef TQ_WAIT_TRAP
    // diagnostics: a wait that has not completed after ~2 s reports the barrier
    // (shared-memory offset, parity, CTA, warp) and gives up
    {
        uint32_t ok = 0;
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;   // the common case costs what the production wait costs
        const long long t0 = clock64();
        while (true) {
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, P1;\n}"
                : "=r"(ok)
                : "r"(smem_u32(bar)), "r"(parity)
                : "memory");
            if (ok) return;
            if (clock64() - t0 > 4000000000ll) {
                if ((threadIdx.x & 31) == 0)
                    printf("TQ_WAIT_TRAP cta %d warp %d bar smem 0x%x parity %u\n", blockIdx.x, threadIdx.x >> 5,
                           smem_u32(bar), parity);
                return;   // give up: the kernel runs to completion (garbage) so the report is flushed
            }
        }
    }
#endif
#ifdef TQ_WAIT_BACKOFF
    uint32_t ok = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(TQ_WAIT_BACKOFF);
    }
#endif
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TQ_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TQ_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Same with a suspend-time hint: for roles that wait long (epilogue), so their
// polling does not steal issue slots from the dequant warps.
static __device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#if defined(TQ_WAIT_TRAP) || defined(TQ_NO_SLEEP)
    mbar_wait(bar, parity);
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TQ_WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra TQ_WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(20000u)
        : "memory");
}

static __device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

static __device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Warp-converged producer issue: every lane executes, one elected lane arms
// the barrier with the expected bytes and starts up to two bulk copies into
// it (the second is skipped when bytes2 == 0).
static __device__ __forceinline__ void bulk_copy2_elect(uint64_t* bar, void* dst1, const void* src1, uint32_t bytes1,
                                                        void* dst2, const void* src2, uint32_t bytes2) {
    asm volatile(
        "{\n\t.reg .pred e, two;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.and.b32 two, %6, 0, e;\n\t"
        "@e mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %7;\n\t"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%2], %3, [%0];\n\t"
        "@two cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5], %6, [%0];\n}" ::"r"(
            smem_u32(bar)),
        "r"(smem_u32(dst1)), "l"(src1), "r"(bytes1), "r"(smem_u32(dst2)), "l"(src2), "r"(bytes2),
        "r"(bytes1 + bytes2)
        : "memory");
}

static __device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// programmatic dependent launch (PDL)
static __device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifdef TQ_PDL_LATE
// variant: no early trigger -- a CTA's exit triggers its dependents, so a
// dependent grid only overlaps the primary's tail (launch latency, prologue)
static __device__ __forceinline__ void pdl_launch_dependents() {}
#else
static __device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

// true in exactly one lane of a converged warp
static __device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, e;\n}"
        : "=r"(pred));
    return pred != 0;
}

static __device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

static __device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
static __device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16, fp32 accumulate, cta_group::1.
static __device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Warp-converged variants: the whole warp executes, one elected lane issues.
// Keeps descriptors warp-uniform (uniform registers, no per-instruction
// register->uniform moves or waterfall loops) -- ~3x faster MMA issue.
static __device__ __forceinline__ void tc_mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                      uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Four K=16 MMAs over one 64-wide K atom (A: 4 x 8 TMEM columns, B: 4 x 32 bytes
// inside a 128B-swizzled atom -> descriptor start field +2 per step), issued by
// one elected lane of a converged warp.  acc = 0 overwrites D on the first.
static __device__ __forceinline__ void tc_mma_ts_x4_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                         uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 a1, a2, a3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 t, %4, %4;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

static __device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}

static __device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

static __device__ __forceinline__ void tc_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

static __device__ __forceinline__ void tc_st_32x32b_x8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// Two K=16 MMAs over a 32-column slice of a 128B-swizzled atom (descriptor start +2 per step).
static __device__ __forceinline__ void tc_mma_ts_x2_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                         uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b64 b1;\n\t.reg .b32 a1;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 t, %4, %4;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.u32 a1, %1, 8;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

static __device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

static __device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
static __device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

static __device__ __forceinline__ void tc_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}

static __device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

static __device__ __forceinline__ uint16_t ld_shared_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

// 16-byte async global->shared copy (L2 only) and its mbarrier completion hook
static __device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
static __device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
static __device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// async arrive that first raises the barrier's pending count (no .noinc): the
// arrival is extra to the count the barrier was initialised with
static __device__ __forceinline__ void cp_async_mbar_arrive_inc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
static __device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// make generic-proxy shared-memory writes visible to the async proxy (tcgen05.mma operand reads)
static __device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, rows of
// 128 B, 8-row core-matrix groups 1024 B apart (SBO), sm_100 version 1.
static __device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;                 // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;         // SBO
    d |= static_cast<uint64_t>(1u) << 46;                 // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2u) << 61;                 // SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::f16, A=B=F16, D=F32, both K-major, M=128.
static __device__ __forceinline__ uint32_t idesc_f16(uint32_t n) {
    return (1u << 4) | ((n >> 3) << 17) | ((uint32_t(kBM) >> 4) << 24);
}

static __device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t orv) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(orv));  // (a & b) | c
    return r;
}

static __device__ __forceinline__ uint32_t hfma2_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

static __device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b) {
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

static __device__ __forceinline__ uint32_t magic_for(int pos) {
    const uint32_t e = static_cast<uint32_t>(25 - pos) << 10;
    return e | (e << 16);
}

struct DqConst {
    uint32_t s2;         // half2 (s, s)
    uint32_t bias[10];   // bias for field position pos (index pos): -2^(10-pos) * s
};

static __device__ __forceinline__ DqConst make_dq(__half s) {
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

static __device__ __forceinline__ uint32_t dq_field(uint32_t w, int pos, int bits, const DqConst& c) {
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


}  // namespace tqb
