// PTX wrappers shared by the tcgen05 kernels (sm_100a): mbarriers, bulk
// copies, tcgen05 MMA / commit / TMEM loads and stores, smem descriptors.
#pragma once

#include "common.cuh"

namespace cq {

// ---------------------------------------------------------------------------
// PTX wrappers (tcgen05 / mbarrier / bulk copy)

__device__ __forceinline__ uint32_t u_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// x >> 16 on the FMA pipe (IMAD.HI) — the ALU pipe is the expanders' bottleneck.
__device__ __forceinline__ uint32_t hi16(uint32_t x) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, 65536;" : "=r"(r) : "r"(x));
    return r;
}

// a | b for halves with disjoint non-zero bytes (== a + b, no carries), as an
// integer multiply-add so it issues on the FMA pipe instead of the saturated ALU pipe.
__device__ __forceinline__ uint32_t u_merge(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

__device__ __forceinline__ uint32_t u_prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}

__device__ __forceinline__ void u_bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void u_bar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void u_bar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// UM_WAIT_NS > 0: try_wait with a suspend-time hint, so a waiting warp sleeps
// until the phase completes (up to the hint) instead of re-issuing the probe.
#ifndef UM_WAIT_NS
#define UM_WAIT_NS 0
#endif
__device__ __forceinline__ void u_bar_wait(uint32_t bar, uint32_t phase) {
#if UM_WAIT_NS > 0
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "UW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra UW_%=;\n}" ::"r"(bar),
        "r"(phase), "n"(UM_WAIT_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "UW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra UW_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
#endif
}
__device__ __forceinline__ void u_bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// Warp-converged variants: every lane calls, one elected lane acts (a divergent
// `if (lane == 0)` around async-proxy instructions costs ~200 cycles each).
__device__ __forceinline__ void u_bar_expect_elect(uint32_t bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(bar),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void u_bar_arrive_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void u_bulk_elect(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ uint32_t u_pin(uint32_t x) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(u_smem(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void u_prefetch_elect(const void *src, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e cp.async.bulk.prefetch.L2.global [%0], %1;\n\t}" ::"l"(src),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// D[tmem d] (+)= A[tmem a] x B[smem desc], kind::i8, 128 x N x 32.  Called by a
// whole converged warp; one elected lane issues.
__device__ __forceinline__ void tc_mma_i8(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u)
        : "memory");
}
// One chunk of the merged-digit GEMM: KS k-steps x P planes of
// tcgen05.mma kind::i8, issued by one elected lane from one asm block, so the
// operands become uniform registers once per chunk instead of once per MMA.
//   D plane p    : d0 + p * nt           (TMEM accumulator columns)
//   A (kk, p)    : a0 + kk * P * 8 + p * 8 (TMEM A stage columns)
//   B k-step kk  : bdesc0 with its start address advanced kk * 256 bytes
// The first k-step accumulates only when acc != 0.
#define CQ_MMA1(D, A, B, P_) "@e tcgen05.mma.cta_group::1.kind::i8 [" D "], [" A "], " B ", %4, " P_ ";\n\t"
template <int KS, int P>
__device__ __forceinline__ void tc_mma_chunk(uint32_t d0, uint32_t nt, uint32_t a0, uint64_t bdesc0, uint32_t idesc,
                                             uint32_t acc) {
    static_assert((KS == 4 || KS == 2) && (P == 3 || P == 2), "chunk shapes of the merged layouts");
    if constexpr (KS == 4 && P == 3) {
        asm volatile(
            "{\n\t.reg .pred e, f, on;\n\t.reg .b32 d1, d2, a1, a2, a3, a4, a5, a6, a7, a8, a9, a10, a11;\n\t"
            ".reg .b64 b1, b2, b3;\n\t"
            "setp.ne.b32 f, %5, 0;\n\tsetp.eq.b32 on, 0, 0;\n\t"
            "add.u32 d1, %0, %1;\n\tadd.u32 d2, d1, %1;\n\t"
            "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\tadd.u32 a4, %2, 32;\n\t"
            "add.u32 a5, %2, 40;\n\tadd.u32 a6, %2, 48;\n\tadd.u32 a7, %2, 56;\n\tadd.u32 a8, %2, 64;\n\t"
            "add.u32 a9, %2, 72;\n\tadd.u32 a10, %2, 80;\n\tadd.u32 a11, %2, 88;\n\t"
            "add.u64 b1, %3, 16;\n\tadd.u64 b2, %3, 32;\n\tadd.u64 b3, %3, 48;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            CQ_MMA1("%0", "%2", "%3", "f") CQ_MMA1("d1", "a1", "%3", "f") CQ_MMA1("d2", "a2", "%3", "f")
            CQ_MMA1("%0", "a3", "b1", "on") CQ_MMA1("d1", "a4", "b1", "on") CQ_MMA1("d2", "a5", "b1", "on")
            CQ_MMA1("%0", "a6", "b2", "on") CQ_MMA1("d1", "a7", "b2", "on") CQ_MMA1("d2", "a8", "b2", "on")
            CQ_MMA1("%0", "a9", "b3", "on") CQ_MMA1("d1", "a10", "b3", "on") CQ_MMA1("d2", "a11", "b3", "on")
            "}" ::"r"(d0), "r"(nt), "r"(a0), "l"(bdesc0), "r"(idesc), "r"(acc)
            : "memory");
    } else if constexpr (KS == 4 && P == 2) {
        asm volatile(
            "{\n\t.reg .pred e, f, on;\n\t.reg .b32 d1, a1, a2, a3, a4, a5, a6, a7;\n\t"
            ".reg .b64 b1, b2, b3;\n\t"
            "setp.ne.b32 f, %5, 0;\n\tsetp.eq.b32 on, 0, 0;\n\t"
            "add.u32 d1, %0, %1;\n\t"
            "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\tadd.u32 a4, %2, 32;\n\t"
            "add.u32 a5, %2, 40;\n\tadd.u32 a6, %2, 48;\n\tadd.u32 a7, %2, 56;\n\t"
            "add.u64 b1, %3, 16;\n\tadd.u64 b2, %3, 32;\n\tadd.u64 b3, %3, 48;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            CQ_MMA1("%0", "%2", "%3", "f") CQ_MMA1("d1", "a1", "%3", "f")
            CQ_MMA1("%0", "a2", "b1", "on") CQ_MMA1("d1", "a3", "b1", "on")
            CQ_MMA1("%0", "a4", "b2", "on") CQ_MMA1("d1", "a5", "b2", "on")
            CQ_MMA1("%0", "a6", "b3", "on") CQ_MMA1("d1", "a7", "b3", "on")
            "}" ::"r"(d0), "r"(nt), "r"(a0), "l"(bdesc0), "r"(idesc), "r"(acc)
            : "memory");
    } else if constexpr (KS == 2 && P == 3) {
        asm volatile(
            "{\n\t.reg .pred e, f, on;\n\t.reg .b32 d1, d2, a1, a2, a3, a4, a5;\n\t.reg .b64 b1;\n\t"
            "setp.ne.b32 f, %5, 0;\n\tsetp.eq.b32 on, 0, 0;\n\t"
            "add.u32 d1, %0, %1;\n\tadd.u32 d2, d1, %1;\n\t"
            "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\tadd.u32 a4, %2, 32;\n\t"
            "add.u32 a5, %2, 40;\n\tadd.u64 b1, %3, 16;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            CQ_MMA1("%0", "%2", "%3", "f") CQ_MMA1("d1", "a1", "%3", "f") CQ_MMA1("d2", "a2", "%3", "f")
            CQ_MMA1("%0", "a3", "b1", "on") CQ_MMA1("d1", "a4", "b1", "on") CQ_MMA1("d2", "a5", "b1", "on")
            "}" ::"r"(d0), "r"(nt), "r"(a0), "l"(bdesc0), "r"(idesc), "r"(acc)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, f, on;\n\t.reg .b32 d1, a1, a2, a3;\n\t.reg .b64 b1;\n\t"
            "setp.ne.b32 f, %5, 0;\n\tsetp.eq.b32 on, 0, 0;\n\t"
            "add.u32 d1, %0, %1;\n\t"
            "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\tadd.u64 b1, %3, 16;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            CQ_MMA1("%0", "%2", "%3", "f") CQ_MMA1("d1", "a1", "%3", "f")
            CQ_MMA1("%0", "a2", "b1", "on") CQ_MMA1("d1", "a3", "b1", "on")
            "}" ::"r"(d0), "r"(nt), "r"(a0), "l"(bdesc0), "r"(idesc), "r"(acc)
            : "memory");
    }
}
#undef CQ_MMA1


// One digit plane of a merged-layout chunk: KS MMAs into the plane's accumulator d, A k-step kk at
// a0 + kk * astride, B k-step kk at bdesc0 advanced kk * 256 bytes (per-plane MMA warps).
template <int KS>
__device__ __forceinline__ void tc_mma_plane(uint32_t d, uint32_t a0, uint32_t astride, uint64_t bdesc0, uint32_t idesc,
                                             uint32_t acc) {
    static_assert(KS == 4 || KS == 2, "chunk shapes of the merged layouts");
    if constexpr (KS == 4) {
        asm volatile(
            "{\n\t.reg .pred e, f, on;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
            "setp.ne.b32 f, %5, 0;\n\tsetp.eq.b32 on, 0, 0;\n\t"
            "add.u32 a1, %1, %2;\n\tadd.u32 a2, a1, %2;\n\tadd.u32 a3, a2, %2;\n\t"
            "add.u64 b1, %3, 16;\n\tadd.u64 b2, %3, 32;\n\tadd.u64 b3, %3, 48;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %3, %4, f;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, on;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a2], b2, %4, on;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a3], b3, %4, on;\n\t}" ::"r"(d),
            "r"(a0), "r"(astride), "l"(bdesc0), "r"(idesc), "r"(acc)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, f, on;\n\t.reg .b32 a1;\n\t.reg .b64 b1;\n\t"
            "setp.ne.b32 f, %5, 0;\n\tsetp.eq.b32 on, 0, 0;\n\t"
            "add.u32 a1, %1, %2;\n\tadd.u64 b1, %3, 16;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %3, %4, f;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, on;\n\t}" ::"r"(d),
            "r"(a0), "r"(astride), "l"(bdesc0), "r"(idesc), "r"(acc)
            : "memory");
    }
}

// Arrive `count` times on an mbarrier from one elected lane of a converged warp.
__device__ __forceinline__ void u_bar_arrive_cnt_elect(uint32_t bar, uint32_t count) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(bar),
        "r"(count)
        : "memory");
}

__device__ __forceinline__ void tc_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

// 8 consecutive 32-bit TMEM columns of this thread's lane.
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major, no-swizzle smem descriptor: core matrices of 8 rows x 16 bytes,
// LBO = byte distance between the two 16-byte K halves, SBO = between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    return d;                // base offset 0, layout SWIZZLE_NONE
}

// K-major operand with 128-byte rows in SWIZZLE_128B (8-row atoms of 1 KB, atom-aligned base): the
// layout a TMA tile load with that swizzle writes.  A k-slice inside the row is addressed by
// advancing the start address (the swizzle applies to the final address).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;            // LBO: unused for swizzled K-major
    d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8-row atoms
    d |= (uint64_t)1 << 46;            // descriptor version (Blackwell)
    d |= (uint64_t)2 << 61;            // SWIZZLE_128B
    return d;
}

// kind::i8 instruction descriptor: s32 accumulate, A and B signed, both K-major.
__device__ __forceinline__ uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

}  // namespace cq
