// ptx_sm100.cuh -- thin inline-PTX wrappers for the sm_100a features the
// FPx kernels use: mbarrier, bulk/tensor TMA copies, tcgen05 (TMEM alloc,
// st/ld, UMMA issue/commit) and fp16x2 RNE multiply.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda.h>

#define FPX_DEV __device__ __forceinline__

namespace fpxk {

FPX_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

FPX_DEV uint32_t lane_id() { return threadIdx.x & 31u; }

FPX_DEV uint32_t warp_id_uniform() {
    return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
}

FPX_DEV bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
FPX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

FPX_DEV void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

FPX_DEV void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

FPX_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

FPX_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// FPX_TRYWAIT_HINT (ns): suspend-time hint of every try_wait; the waiting
// thread sleeps in hardware until the phase completes or the hint expires,
// instead of re-polling the barrier unit.  0 = no hint (system default).
#ifndef FPX_TRYWAIT_HINT
#define FPX_TRYWAIT_HINT 0
#endif
FPX_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
#if FPX_TRYWAIT_HINT
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "n"(FPX_TRYWAIT_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
#endif
    return ok != 0;
}

// FPX_WATCHDOG builds (debug variant only): a wait that has not completed
// after ~2^28 polls prints the barrier's shared address, parity and the
// caller's block/thread, then traps -- a diagnosable crash instead of a hang.
#ifndef FPX_WATCHDOG
#define FPX_WATCHDOG 0
#endif
FPX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
#if FPX_WATCHDOG
    uint32_t n = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++n == (1u << 22)) {
            printf("watchdog: block %d thread %d stuck on mbarrier smem+0x%x parity %u\n", blockIdx.x, threadIdx.x,
                   smem_u32(bar), parity);
            __trap();
        }
    }
#else
    while (!mbar_try_wait(bar, parity)) {
    }
#endif
}

// Polling with back-off, for waiters off the critical path: every
// try_wait occupies the SM's barrier unit, so idle spinners slow down the
// latency-critical waiters (MMA issuer, producer) sharing it.
FPX_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
#if FPX_WATCHDOG
    uint32_t n = 0;
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(ns);
        if (++n == (1u << 22)) {
            printf("watchdog: block %d thread %d stuck (sleeping) on mbarrier smem+0x%x parity %u\n", blockIdx.x,
                   threadIdx.x, smem_u32(bar), parity);
            __trap();
        }
    }
#else
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(ns);
    }
#endif
}

// Programmatic dependent launch (PDL).  launch_dependents lets the next
// kernel in the stream be scheduled (its CTAs still need this grid's SM
// resources to free up); wait blocks until the preceding grid has completed
// and its memory is visible.  Both are no-ops without the PDL launch attribute.
FPX_DEV void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
FPX_DEV void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Named CTA barrier over `threads` threads (multiple of 32); id 0 is
// __syncthreads.
FPX_DEV void named_bar_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---------------------------------------------------------------- TMA
FPX_DEV uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

FPX_DEV uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 16-byte global store / L2 load with an L2 cache-eviction policy.
FPX_DEV void st_global_v4_hint(void* ptr, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(a), "r"(b), "r"(c),
                 "r"(d), "l"(policy)
                 : "memory");
}

FPX_DEV float4 ld_global_cg_v4_hint(const void* ptr, uint64_t policy) {
    float4 v;
    asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(ptr), "l"(policy)
                 : "memory");
    return v;
}

// 1-D bulk copy global -> shared, completion on an mbarrier (bytes % 16 == 0).
FPX_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 2-D tiled tensor copy global -> shared.
FPX_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar,
                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 3-D tiled tensor copy global -> shared.
FPX_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, int32_t z, uint64_t* bar,
                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

FPX_DEV void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------- tcgen05
template <uint32_t kCols>
FPX_DEV void tmem_alloc(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
FPX_DEV void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

FPX_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FPX_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem desc]; kind::f16, cta_group::1.
FPX_DEV void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[smem desc] * B[smem desc].
FPX_DEV void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Warp-wide variants for warp-uniform issue loops: the whole warp executes
// the asm, one elected lane issues.  Keeps the loop's bookkeeping in uniform
// registers without the per-instruction elect/branch loop nvcc generates for
// an `if (lane == 0)` around each tcgen05 instruction.
FPX_DEV void umma_f16_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// kind::f8f6f4 (A = FP6/FP8 codes in 8-bit containers from TMEM, B = FP8
// from shared memory, K = 32 per instruction), warp-wide with one elected
// issuer like umma_f16_ts_warp.
FPX_DEV void umma_f8f6f4_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

FPX_DEV void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

// Arrive on `bar` once every previously issued tcgen05.mma of this thread
// has completed (implies tcgen05.fence::before_thread_sync).
FPX_DEV void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 16 lanes x 32 columns (32-bit): 16x128b repeated 8 times. Register 2i
// goes to (lane base + t/4, col 4i + t%4), register 2i+1 to lane base + 8 + t/4.
FPX_DEV void tmem_st_16x128b_x8(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

// 16 lanes x 16 columns: 16x128b repeated 4 times (register 2i -> lane base
// + t/4, col 4i + t%4; register 2i+1 -> lane base + 8 + t/4).
FPX_DEV void tmem_st_16x128b_x4(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

FPX_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes (thread t -> lane base + t) x 16 consecutive 32-bit columns.
FPX_DEV void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

FPX_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major operand with 128-byte swizzle:
// rows of 128 B, 8-row (1024 B) swizzle atoms stacked at SBO = 1024 B.
FPX_DEV uint64_t umma_desc_sw128_kmajor(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3fffu);  // start address
    d |= static_cast<uint64_t>(1u) << 16;                      // LBO (unused for SW128 K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;              // SBO
    d |= static_cast<uint64_t>(1u) << 46;                      // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2u) << 61;                      // SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::f16: A=B=f16, D=f32, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_f16(uint32_t m, uint32_t n) {
    return (1u << 4)            // D format f32
           | (0u << 7)          // A f16
           | (0u << 10)         // B f16
           | ((n >> 3) << 17)   // N / 8
           | ((m >> 4) << 24);  // M / 16
}

// Instruction descriptor, kind::f8f6f4: D=f32, A/B formats (MXF8F6F4:
// e4m3 0, e5m2 1, e2m3 3, e3m2 4, e2m1 5), both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_f8f6f4(uint32_t m, uint32_t n, uint32_t a_fmt, uint32_t b_fmt) {
    return (1u << 4) | (a_fmt << 7) | (b_fmt << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// ---------------------------------------------------------------- fp16
// Correctly rounded (RN, subnormals kept) fp16x2 multiply; `.rn` also
// forbids contraction, so this is exactly the reference's half_mul per lane.
FPX_DEV uint32_t hmul2_rn(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

FPX_DEV uint32_t lds32(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}

}  // namespace fpxk
