// fpx_linear_x8.cu -- the fused FPx linear for N <= 32 on tcgen05.mma
// kind::f8f6f4.  Drop-in for the reference's gemm_packed (gemm.cpp:170-219)
// like the kind::f16 decode kernel of fpx_linear.cu, with two changes that
// follow from B200's tensor core:
//  * A is the packed FP6 codes themselves, 8-bit containers straight from
//    the stitched words (codes8_slice_half: 4 LOP3 + 5 shifts + 4 PRMT per 16
//    weights, no conversion) -- FP5 e2m2 as e2m3 codes;
//  * B is the fp16 activations split exactly into three e4m3 parts with one
//    power-of-two scale per (K chunk, column) (act_split_kernel), N = 3 NPAD.
// One kind::f8f6f4 MMA covers M=128 x K=32 in the tensor-pipe time one
// kind::f16 MMA needs for K=16 (tools/micro/mma_f8f6f4_bench.cu: 56 cycles
// either way for N <= 96, distinct operands), and an A stage is half the
// TMEM: 13 A slots at NPAD 16 against 7.  Products are exact either way, so
// the result is the same sum of products as kind::f16, grouped into three
// fp32 partial sums (one per part) that the epilogue combines smallest first.
//
// Units whose 128 row scales all lie in the f8 range (tile_scales_f8_ok:
// s in [2^-14, 2^11], every valid packed weight in practice) run kind::f8f6f4
// and apply the row scale to the fp32 accumulator; others (hand-made tiny or
// huge scales) run kind::f16 with the decode kernel's per-quarter scale
// placement, in the same launch.  The A ring is counted in A-steps of 32
// TMEM columns: an f8 stage (two k-tiles of codes) takes one, an f16 stage
// (two k-tiles of fp16) two.
//
// Warps: 0 .. 4G-1 de-quantisers (group w/4, TMEM lane quarter w%4), 4G ..
// 4G+3 epilogue, 4G+4 MMA issuer, 4G+5 weight producer (also allocates
// TMEM), 4G+6 activation producer.
#include <algorithm>
#include <type_traits>

#include "fpx_linear_common.cuh"

namespace fpxk {

#ifndef FPX_X8_SB16
#define FPX_X8_SB16 10  // activation-ring depth at NPAD 16 (6 KB stages)
#endif
#ifndef FPX_X8_SB32
#define FPX_X8_SB32 6  // at NPAD 32 (12 KB stages)
#endif
#ifndef FPX_X8_SMEM_KB
#define FPX_X8_SMEM_KB 216
#endif
#ifndef FPX_X8_BS
#define FPX_X8_BS 3
#endif

template <int F, int NPAD, int G_>
struct X8Cfg {
    static constexpr int kKS = 2;  // k-tiles per stage: one 128-byte e4m3 row of every part-column
    static constexpr int kG = G_;
    static constexpr int kEpiWarp0 = 4 * kG;
    static constexpr int kMmaWarp = kEpiWarp0 + 4;
    static constexpr int kProdWarp = kMmaWarp + 1;
    static constexpr int kActWarp = kProdWarp + 1;
    static constexpr int kWarps = kActWarp + 1;
    static constexpr int kThreads = 32 * kWarps;
    static constexpr int kHiBytes = 512 * FmtTraits<F>::kBitsHi;  // per 64x64 tile
    static constexpr int kLoBytes = 512 * FmtTraits<F>::kBitsLo;
    // weight stage: [hi r0 x KS][hi r1 x KS][lo r0 x KS][lo r1 x KS]
    static constexpr int kLoOff = 2 * kKS * kHiBytes;
    static constexpr int kWStageBytes = (2 * kKS * (kHiBytes + kLoBytes) + 1023) / 1024 * 1024;
    static constexpr int kBBytes = NPAD * 128;       // fp16 activation k-tile (kind::f16 units)
    static constexpr int kB8Bytes = 3 * NPAD * 128;  // e4m3 parts of both k-tiles (kind::f8f6f4 units)
    static constexpr int kBStageBytes = (std::max(kKS * kBBytes, kB8Bytes) + 1023) / 1024 * 1024;
    static constexpr int kAccCols = 3 * NPAD;  // per accumulator: one NPAD block per part
    static constexpr int kAccCol0 = int(kTmemCols) - 2 * kAccCols;
    static constexpr int kASlots = std::min(kAccCol0 / 32, 16);  // A-steps of 32 TMEM columns
    static constexpr int kBS = FPX_X8_BS;                        // A-steps per commit batch
    static constexpr int kBStages = NPAD <= 16 ? FPX_X8_SB16 : FPX_X8_SB32;
    static constexpr int kNB = 16;  // batch barriers: waiters are never more than a few batches behind
    static constexpr int kBarBytes = 8 * (2 * 24 + kBStages + kNB + kASlots + 5) + 16 + 4 * 16;
    // weight ring: a multiple of G, so stage si - SW was read by the same
    // group, whose wait proved that phase complete (no parity aliasing)
    static constexpr int kWStages =
        std::min(24, (FPX_X8_SMEM_KB * 1024 - kBarBytes - 1024 - kBStages * kBStageBytes) / kWStageBytes) / kG * kG;
    static constexpr int kSmemBytes = kWStages * kWStageBytes + kBStages * kBStageBytes + kBarBytes + 1024;
    static constexpr uint32_t kWTx = 2 * kKS * (kHiBytes + kLoBytes);
    static constexpr uint32_t kBTx = kKS * kBBytes;
    static constexpr uint32_t kB8Tx = kB8Bytes;
    static_assert(NPAD == 16 || NPAD == 32, "N = 3 NPAD <= 96 keeps the MMA at its flat cost");
    // A slot reuse: the group storing A-step a waits for the batch of a - R,
    // which ends at or before A-step a - R + BS - 1.  R >= G + BS keeps that
    // batch clear of the group's own previous kind::f8f6f4 stage (one A-step
    // per stage), so groups never wait on their own MMAs; kind::f16 fallback
    // stages (two A-steps) may, which only slows those rare units.  R > BS
    // suffices for progress: a batch never needs a later stage's A-step.
    static_assert(kASlots >= kG + kBS, "A ring must cover the groups plus a commit batch");
    static_assert(kBStages >= kBS + 1, "activation ring must outlast a commit batch");
    static_assert(kWStages >= 2 * kG && kWStages % kG == 0, "weight ring");
    static_assert(kSmemBytes <= 227 * 1024, "shared memory");
};

template <int F, int NPAD, int G_>
__global__ void __launch_bounds__(X8Cfg<F, NPAD, G_>::kThreads, 1)
    fpx_linear_x8_kernel(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap hi_map,
                         const __grid_constant__ CUtensorMap lo_map, const __grid_constant__ CUtensorMap b8_map,
                         const KParams p) {
    using C = X8Cfg<F, NPAD, G_>;
    constexpr int KS = C::kKS, G = C::kG, SW = C::kWStages, SB = C::kBStages, R = C::kASlots, BS = C::kBS,
                  NB = C::kNB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bring = smem;                         // [SB] activation stages (SW128 K-major)
    uint8_t* wring = smem + SB * C::kBStageBytes;  // [SW] packed weight stages
    uint64_t* bars = reinterpret_cast<uint64_t*>(wring + SW * C::kWStageBytes);
    uint64_t* wfull = bars;            // [SW] weights landed                       (tx bytes)
    uint64_t* wempty = wfull + SW;     // [SW] group's 4 warps read the stage       (arrivals)
    uint64_t* bfull = wempty + SW;     // [SB] activations landed                   (tx bytes)
    uint64_t* done = bfull + SB;       // [NB] MMAs of a batch of BS A-steps complete (commit)
    uint64_t* aready = done + NB;      // [R]  group's 4 warps stored an A-step      (arrivals)
    uint64_t* accfull = aready + R;    // [2]  unit's MMAs complete                 (commit)
    uint64_t* accempty = accfull + 2;  // [2]  epilogue drained the accumulator
    uint64_t* f8ready = accempty + 2;  // [1]  epilogue warps published f8mask
    uint32_t* b_alast = reinterpret_cast<uint32_t*>(f8ready + 1);  // [SB] last A-step of the stage in B slot
    uint32_t* tmem_slot = b_alast + 16;
    __shared__ uint32_t red_tq[4 * kMaxDefer];
    __shared__ uint32_t red_n[4];
    __shared__ unsigned long long f8mask;  // bit i: unit u_begin + i runs kind::f8f6f4 (i < 64)

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();
    const uint32_t u_begin = static_cast<uint32_t>((uint64_t)blockIdx.x * p.units / gridDim.x);
    const uint32_t u_end = static_cast<uint32_t>((uint64_t)(blockIdx.x + 1) * p.units / gridDim.x);
    if (threadIdx.x == 0) trace_cta(p, 15);  // kernel entry, before the prologue

    if (warp == C::kEpiWarp0 && lane == 0) {
        for (int i = 0; i < SW; ++i) mbar_init(&wfull[i], 1), mbar_init(&wempty[i], 4);
        for (int i = 0; i < SB; ++i) mbar_init(&bfull[i], 1);
        for (int i = 0; i < NB; ++i) mbar_init(&done[i], 1);
        for (int i = 0; i < R; ++i) mbar_init(&aready[i], 4);
        for (int i = 0; i < 2; ++i) mbar_init(&accfull[i], 1), mbar_init(&accempty[i], 4);
        mbar_init(f8ready, 4);
        for (int i = 0; i < 4; ++i) red_n[i] = 0;
        f8mask = 0ull;
        fence_mbar_init();
    }
    if (warp == C::kProdWarp) {
        if (lane == 0) prefetch_tmap(&act_map), prefetch_tmap(&hi_map), prefetch_tmap(&lo_map), prefetch_tmap(&b8_map);
        tmem_alloc<kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) trace_cta(p, 0);
    if (p.pdl) grid_dep_launch();
    // MMA kind of unit u (tile mt): f8mask once the epilogue warps published
    // it (the CTA's first 64 units), else voted on the spot.  Warp-collective.
    bool f8_waited = false;
    auto unit_is_f8 = [&](uint32_t u, uint32_t mt) -> bool {
        const uint32_t i = u - u_begin;
        if (i >= 64u) return tile_scales_f8_ok(p, mt);
        if (!f8_waited) mbar_wait(f8ready, 0), f8_waited = true;
        return (f8mask >> i) & 1ull;
    };

    if (p.dbg & 256u) {
        // FPX_LINEAR_DBG=256: launch + prologue + teardown only (bring-up)
    } else if (warp == C::kProdWarp) {
        // ------------------------------------------------ weight producer
        // The weight ring -- where the bytes are -- recycles as soon as a
        // group holds the words in registers.  PDL mode 2: the packed weights
        // are immutable while linears run, so they stream before the
        // preceding kernel has finished.
        if (p.pdl != 2u) grid_dep_wait();
        const bool leader = lane == 0;
        const uint64_t pol_w = policy_evict_first();
        const uint32_t wtx = (p.dbg & 4u) ? 0u : C::kWTx;
        uint32_t si = 0, ws = 0, wph = 0;
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, s0, ns;
            unit_stages<KS>(p, u, mt, ch, s0, ns);
            const int32_t tr0 = static_cast<int32_t>(2 * mt);
            for (uint32_t ls = 0; ls < ns; ++ls, ++si) {
                const int32_t k = static_cast<int32_t>((s0 + ls) * KS);
                if (si >= static_cast<uint32_t>(SW)) wait_rec(p, &wempty[ws], wph ^ 1u, 1, si);
                if (leader) {
                    trace_mark(p, kTrProdIssue, si);
                    mbar_arrive_expect_tx(&wfull[ws], wtx);
                    if (!(p.dbg & 4u)) {
                        uint8_t* wb = wring + ws * C::kWStageBytes;
                        tma_load_3d(wb, &hi_map, 0, k, tr0, &wfull[ws], pol_w);
                        tma_load_3d(wb + C::kLoOff, &lo_map, 0, k, tr0, &wfull[ws], pol_w);
                    }
                }
                __syncwarp();
                if (++ws == static_cast<uint32_t>(SW)) ws = 0, wph ^= 1u;
            }
        }
    } else if (warp == C::kActWarp) {
        // ------------------------------------------------ activation producer
        // kind::f8f6f4 units: one [3 NPAD x 128 B] box of the e4m3 parts per
        // stage; kind::f16 units: the fp16 activations.  A B slot is reused
        // once the MMA batch holding the last A-step of its previous stage
        // completed (b_alast).
        grid_dep_wait();
        const bool leader = lane == 0;
        const uint64_t pol_b = policy_evict_last();
        uint32_t si = 0, bs = 0, abase = 0;
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, s0, ns;
            unit_stages<KS>(p, u, mt, ch, s0, ns);
            const bool f8 = unit_is_f8(u, mt);
            const uint32_t w = f8 ? 1u : 2u;
            const uint32_t btx = (p.dbg & 8u) ? 0u : (f8 ? C::kB8Tx : C::kBTx);
            for (uint32_t ls = 0; ls < ns; ++ls, ++si) {
                const int32_t k = static_cast<int32_t>((s0 + ls) * KS);
                if (si >= static_cast<uint32_t>(SB)) {
                    const uint32_t b = b_alast[bs] / BS;
                    wait_rec(p, &done[b % NB], (b / NB) & 1u, 7, si);
                }
                if (leader) {
                    b_alast[bs] = abase + ls * w + w - 1;
                    mbar_arrive_expect_tx(&bfull[bs], btx);
                    if (!(p.dbg & 8u)) {
                        if (f8)
                            tma_load_2d(bring + bs * C::kBStageBytes, &b8_map, k * 64, 0, &bfull[bs], pol_b);
                        else
                            tma_load_3d(bring + bs * C::kBStageBytes, &act_map, 0, 0, k, &bfull[bs], pol_b);
                    }
                }
                __syncwarp();
                if (++bs == static_cast<uint32_t>(SB)) bs = 0;
            }
            abase += ns * w;
        }
    } else if (warp == C::kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc16 = umma_idesc_f16(kTileM, NPAD);
        constexpr uint32_t idesc8 = umma_idesc_f8f6f4(kTileM, 3 * NPAD, f8_a_format<F>(), 0u /* e4m3 */);
        const bool leader = lane == 0;
        uint32_t si = 0, lu = 0, bsl = 0, bph = 0;
        uint32_t a = 0, as = 0, aph = 0;   // A-step, its slot and phase parity
        uint32_t nb = 0, nbatch = 0;       // A-steps in the open batch, batches committed
        auto astep_done = [&]() {
            if (++nb == static_cast<uint32_t>(BS)) {
                umma_commit_warp(&done[nbatch % NB]);
                ++nbatch;
                nb = 0;
            }
            ++a;
            if (++as == static_cast<uint32_t>(R)) as = 0, aph ^= 1u;
        };
        for (uint32_t u = u_begin; u < u_end; ++u, ++lu) {
            uint32_t mt, ch, s0, ns;
            unit_stages<KS>(p, u, mt, ch, s0, ns);
            const bool f8 = unit_is_f8(u, mt);
            const uint32_t ab = lu & 1u;
            wait_rec(p, &accempty[ab], ((lu >> 1) & 1u) ^ 1u, 5, lu);  // epilogue done with unit lu-2
            tc_fence_after();
            const uint32_t d_tmem = tmem + C::kAccCol0 + ab * C::kAccCols;
            for (uint32_t ls = 0; ls < ns; ++ls, ++si) {
                if (leader) trace_mark(p, kTrMmaWait, si);
                wait_rec(p, &bfull[bsl], bph, 8, si);
                const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bring + bsl * C::kBStageBytes));
                if (f8) {
                    wait_rec(p, &aready[as], aph, 4, si);
                    tc_fence_after();
                    if (leader) trace_mark(p, kTrMmaGo, si);
                    if (!(p.dbg & 2u)) {
                        const uint32_t a_tmem = tmem + as * 32;
#pragma unroll
                        for (int kk = 0; kk < KS; ++kk)
#pragma unroll
                            for (uint32_t ks = 0; ks < 2; ++ks)
                                umma_f8f6f4_ts_warp(d_tmem, a_tmem + kk * 16 + ks * 8,
                                                    bdesc + static_cast<uint64_t>((kk * 64 + ks * 32) >> 4), idesc8,
                                                    (ls > 0 || kk > 0 || ks > 0) ? 1u : 0u);
                    }
                    astep_done();
                } else {
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk) {
                        wait_rec(p, &aready[as], aph, 4, si);
                        tc_fence_after();
                        if (!(p.dbg & 2u)) {
                            const uint32_t a_tmem = tmem + as * 32;
#pragma unroll
                            for (uint32_t ks = 0; ks < 4; ++ks)
                                umma_f16_ts_warp(d_tmem, a_tmem + ks * 8,
                                                 bdesc + static_cast<uint64_t>((kk * C::kBBytes + ks * 32) >> 4),
                                                 idesc16, (ls > 0 || kk > 0 || ks > 0) ? 1u : 0u);
                        }
                        astep_done();
                    }
                }
                if (leader) trace_mark(p, kTrMmaIssued, si);
                if (++bsl == static_cast<uint32_t>(SB)) bsl = 0, bph ^= 1u;
            }
            umma_commit_warp(&accfull[ab]);
        }
        if (nb != 0) umma_commit_warp(&done[nbatch % NB]), ++nbatch;  // final partial batch
        // no tcgen05.commit arrival may outlive the CTA (it would land in the
        // barriers of the next CTA on this SM): wait for the newest
        if (nbatch != 0) {
            const uint32_t b = nbatch - 1;
            mbar_wait(&done[b % NB], (b / NB) & 1u);
        }
    } else if (warp >= C::kEpiWarp0) {
        // ------------------------------------------------ epilogue
        const uint32_t q = warp & 3u;
        const uint32_t row_l = 32 * q + lane;
        {
            // publish the MMA kind of the CTA's first 64 units: warp q votes
            // units q, q + 4, ...  Scales are immutable like the weights under
            // PDL mode 2, else they wait for the preceding kernel.
            if (p.pdl != 2u) grid_dep_wait();
            unsigned long long bits = 0ull;
            const uint32_t nu = min(u_end - u_begin, 64u);
            for (uint32_t i = q; i < nu; i += 4)
                if (tile_scales_f8_ok(p, (u_begin + i) / p.split)) bits |= 1ull << i;
            if (lane == 0) {
                if (bits != 0ull) atomicOr(&f8mask, bits);
                mbar_arrive(f8ready);
            }
        }
        grid_dep_wait();  // C / partials / counters may still be in use by the preceding kernel
        uint32_t ndefer = 0;
        uint32_t lu = 0;
        for (uint32_t u = u_begin; u < u_end; ++u, ++lu) {
            uint32_t mt, ch, s0, ns;
            unit_stages<KS>(p, u, mt, ch, s0, ns);
            const uint32_t ab = lu & 1u;
            const bool f8 = unit_is_f8(u, mt);
            wait_rec(p, &accfull[ab], (lu >> 1) & 1u, 2, lu);
            if (q == 0 && lane == 0) trace_mark(p, kTrEpiFull, lu);
            tc_fence_after();
            const uint32_t m = mt * kTileM + row_l;
            const bool row_ok = m < p.rows_p;
            // kind::f8f6f4 units: A holds the bare codes, the row scale is
            // applied here; kind::f16 units: the de-quantiser warps of this
            // lane quarter took the same vote (scale_in_epilogue_ok)
            const uint16_t raw_s = 2 * mt + (q >> 1) < p.tile_rows ? __ldg(&p.scales[m]) : uint16_t(0);
            const bool epi_scale = f8 || __all_sync(0xffffffffu, scale_in_epilogue_ok(raw_s));
            const float s_row = epi_scale ? __half2float(__ushort_as_half(raw_s)) : 1.0f;
            float* part = p.ws + (static_cast<size_t>(mt) * p.split + ch) * kTileM * NPAD + row_l * 4;
            const uint32_t tacc = tmem + ((32 * q) << 16) + C::kAccCol0 + ab * C::kAccCols;
#pragma unroll
            for (uint32_t c0 = 0; c0 < NPAD; c0 += 16) {
                uint32_t v[16];
                if (ns == 0) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = 0u;  // empty K chunk contributes zero
                } else if (f8) {
                    // a = 2^-e (h0 + 2^-4 h1 + 2^-8 h2) (act_split_kernel): the part
                    // accumulators smallest first, then 2^-e of (chunk, column)
                    // and the row scale (exact powers of two / fp16 values)
                    uint32_t t[16];
                    tmem_ld_32x32b_x16(tacc + 2 * NPAD + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) t[j] = __float_as_uint(__uint_as_float(v[j]) * 0x1p-8f);
                    tmem_ld_32x32b_x16(tacc + NPAD + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        t[j] = __float_as_uint(fmaf(__uint_as_float(v[j]), 0x1p-4f, __uint_as_float(t[j])));
                    tmem_ld_32x32b_x16(tacc + c0, v);
                    tmem_ld_wait();
                    const float* cf = p.colf + ch * NPAD + c0;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        v[j] = __float_as_uint((__uint_as_float(v[j]) + __uint_as_float(t[j])) * (s_row * __ldg(cf + j)));
                } else {
                    tmem_ld_32x32b_x16(tacc + c0, v);
                    tmem_ld_wait();
                    if (epi_scale) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * s_row);
                    }
                }
                if (p.split == 1) {
                    if (c0 < p.n && row_ok) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (c0 + j < p.n) c_store(p, m, c0 + j, __uint_as_float(v[j]));
                    }
                } else if (c0 < p.n) {
                    const uint64_t pol_keep = policy_evict_last();
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        st_global_v4_hint(part + ((c0 + j) / 4) * kTileM * 4, v[j], v[j + 1], v[j + 2], v[j + 3], pol_keep);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[ab]);
            if (q == 0 && lane == 0) trace_cta(p, 1 + lu);
            if (p.split > 1) {
                __threadfence();
                __syncwarp();
                uint32_t old = 0;
                if (lane == 0) old = atomicAdd(&p.counters[mt * 4 + q], 1u);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old == p.split - 1) {
                    // last arriver of (tile, quarter): reduce in the CTA-wide pass
                    // after the main loop (in place when the list is full)
                    __threadfence();
                    if (ndefer < kMaxDefer) {
                        if (lane == 0) {
                            red_tq[q * kMaxDefer + ndefer] = mt * 4 + q;
                            p.counters[mt * 4 + q] = 0;  // self-cleaning for the next launch
                        }
                        ++ndefer;
                    } else {
                        split_reduce_rows<NPAD>(p, mt, row_l, m, row_ok);
                        if (lane == 0) p.counters[mt * 4 + q] = 0;
                    }
                }
            }
        }
        if (lane == 0) red_n[q] = ndefer;  // read only after the final __syncthreads
    } else {
        // ------------------------------------------------ de-quantiser groups
        const uint32_t g = warp >> 2;
        const uint32_t q = warp & 3u;
        const int h = static_cast<int>(q & 1u);
        const uint32_t r = q >> 1;
        const uint32_t tq = tmem + ((32 * q) << 16);  // this warp's TMEM lane quarter
        // kind::f16 units only: row scales one unit ahead (see the decode kernel)
        auto fetch_scales = [&](uint32_t uu, uint16_t (&raw)[2][2]) {
            uint32_t mt_, ch_, s0_, ns_;
            unit_stages<KS>(p, uu, mt_, ch_, s0_, ns_);
            const uint32_t tr_ = 2 * mt_ + r;
#pragma unroll
            for (int lc = 0; lc < 2; ++lc)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf)
                    raw[lc][hf] = tr_ < p.tile_rows ? __ldg(&p.scales[tr_ * 64 + 16 * (2 * h + lc) + 8 * hf + lane / 4])
                                                    : uint16_t(0);
        };
        if (p.pdl != 2u) grid_dep_wait();
        uint32_t si = 0, abase = 0;
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, s0, ns;
            unit_stages<KS>(p, u, mt, ch, s0, ns);
            const bool f8 = unit_is_f8(u, mt);
            const uint32_t w = f8 ? 1u : 2u;
            uint32_t sc[2][2] = {{0u, 0u}, {0u, 0u}};
            bool epi_scale = true;
            if (!f8) {
                uint16_t raw[2][2];
                fetch_scales(u, raw);
                bool ok_t = true;
#pragma unroll
                for (int lc = 0; lc < 2; ++lc)
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        sc[lc][hf] = row_scale_for<F, kHwCvt>(raw[lc][hf]);
                        ok_t = ok_t && scale_in_epilogue_ok(raw[lc][hf]);
                    }
                epi_scale = __all_sync(0xffffffffu, ok_t);
            }
            uint32_t ls = (g + G - si % G) % G;  // this group's stages of the unit: si % G == g
            auto stage_loop = [&](auto mode_tag) {
                constexpr int kMode = decltype(mode_tag)::value;  // 0 f16 + register scale, 1 f16, 2 f8
                for (si += ls; ls < ns; ls += G, si += G) {
                    const uint32_t ws = si % SW;
                    const uint32_t a0 = abase + ls * w;  // first A-step of the stage
                    const uint32_t wb = smem_u32(wring + ws * C::kWStageBytes);
                    if (q == 0 && lane == 0) trace_mark(p, kTrDqAempty, si);
                    wait_rec(p, &wfull[ws], (si / SW) & 1u, 3, si);
                    if (q == 0 && lane == 0) trace_mark(p, kTrDqFull, si);
                    if (warp == 0 && lane == 0 && si == 0) trace_cta(p, 14);  // first weight stage landed
                    uint32_t wd[KS][12];
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk)
                        load_ktile_words<F>(wb + (r * KS + kk) * C::kHiBytes, wb + C::kLoOff + (r * KS + kk) * C::kLoBytes,
                                            h, lane, wd[kk]);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wempty[ws]);
                    // A slots of A-steps a0 .. a0+w-1 last held A-steps a0-R ..: free once
                    // the batch of the newest of those completed (batches complete in order)
                    const uint32_t alast = a0 + w - 1;
                    if constexpr (kMode == 2) {
                        // 8-bit codes: 16 TMEM columns per k-tile, register 2s + hf of
                        // x[lc] = row 16(2h+lc) + 8hf + t/4, slice s.  A missing second
                        // tile-row arrives zero-filled by TMA: code 0.
                        const uint32_t col = (a0 % R) * 32;
#pragma unroll
                        for (int kk = 0; kk < KS; ++kk) {
                            uint32_t x0[8], x1[8];
#pragma unroll
                            for (int sl = 0; sl < 4; ++sl) {
                                uint32_t x[2][2];
                                codes8_slice_half<F>(wd[kk][3 * sl], wd[kk][3 * sl + 1], wd[kk][3 * sl + 2], h, x);
                                x0[2 * sl] = x[0][0];
                                x0[2 * sl + 1] = x[0][1];
                                x1[2 * sl] = x[1][0];
                                x1[2 * sl + 1] = x[1][1];
                            }
                            if (kk == 0) {
                                if (q == 0 && lane == 0) trace_mark(p, kTrDqDone, si);
                                if (alast >= static_cast<uint32_t>(R)) {
                                    const uint32_t b = (alast - R) / BS;
                                    wait_rec(p, &done[b % NB], (b / NB) & 1u, 6, si);
                                }
                                if (q == 0 && lane == 0) trace_mark(p, kTrDqDone1, si);
                                tc_fence_after();
                            }
                            tmem_st_16x128b_x4(tq + col + kk * 16, x0);
                            tmem_st_16x128b_x4(tq + col + kk * 16 + (16u << 16), x1);
                        }
                        tmem_st_wait();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&aready[a0 % R]);
                    } else {
                        // fp16 A-fragments, one k-tile (32 TMEM columns) per A-step
#pragma unroll
                        for (int kk = 0; kk < KS; ++kk) {
                            uint32_t o0[16], o1[16];
                            dequant_words<F, kMode == 0>(wd[kk], h, sc, o0, o1);
                            if (kk == 0) {
                                if (alast >= static_cast<uint32_t>(R)) {
                                    const uint32_t b = (alast - R) / BS;
                                    wait_rec(p, &done[b % NB], (b / NB) & 1u, 6, si);
                                }
                                tc_fence_after();
                            }
                            const uint32_t col = ((a0 + kk) % R) * 32;
                            tmem_st_16x128b_x8(tq + col, o0);
                            tmem_st_16x128b_x8(tq + col + (16u << 16), o1);
                        }
                        tmem_st_wait();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&aready[a0 % R]), mbar_arrive(&aready[(a0 + 1) % R]);
                    }
                    if (q == 0 && lane == 0) trace_mark(p, kTrMmaAfull, si);
                }
            };
            if (f8) stage_loop(std::integral_constant<int, 2>{});
            else if (epi_scale) stage_loop(std::integral_constant<int, 1>{});
            else stage_loop(std::integral_constant<int, 0>{});
            si -= ls - ns;  // back to the first stage of the next unit
            abase += ns * w;
        }
    }

    if (lane == 0) {
        if (warp == C::kMmaWarp) trace_cta(p, 9);
        else if (warp == C::kEpiWarp0) trace_cta(p, 11);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace_cta(p, 7);
    if (warp == C::kProdWarp) {
        tc_fence_after();
        if (lane == 0) trace_cta(p, 12);
        tmem_dealloc<kTmemCols>(tmem);
        if (lane == 0) trace_cta(p, 13);
    }
    if (p.split > 1) final_split_reduce<NPAD>(p, red_tq, red_n, C::kThreads);
}

// ---------------------------------------------------------------------------
// Activation split of the kind::f8f6f4 units.  Every fp16 activation a of K
// chunk ch, column n is written as three e4m3 parts
//     a = 2^-e (h0 + 2^-4 h1 + 2^-8 h2),   2^e: absmax of (ch, n) -> [128, 256)
// (RN at every step, residuals exact in fp32).  Three 4-bit significands
// cover fp16's 11, so the split is exact for every element within 2^14 of
// its chunk-column absmax; smaller ones keep an absolute error below 2^-25
// of it (e4m3 subnormal floor).  The products the MMA forms are exact, so
// the kind::f8f6f4 units compute the same sums of products as kind::f16,
// grouped into three fp32 partial sums instead of one.
// Output (workspace): B8[p * NPAD + n][logical k] (row stride cols_p bytes)
// in the logical K order of codes8_slice_half -- logical 16s + 4j + b <-
// actual 16s + {2j, 2j+1, 8+2j, 9+2j}[b] in every 16-K slice -- and
// colf[ch * NPAD + n] = 2^-e (NaN for a non-finite absmax: the column's
// outputs become NaN).  Columns n >= N are zero.  Grid (NPAD, split), 128
// threads; chunk ch covers stages [ch*nst/split, (ch+1)*nst/split) of 128 K.
__device__ __forceinline__ uint32_t cvt_e4m3x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float2 e4m3x2_to_float2(uint32_t v) {
    uint32_t h2;
    asm("{\n\t.reg .b16 t;\n\tcvt.u16.u32 t, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, t;\n\t}" : "=r"(h2) : "r"(v));
    return __half22float2(*reinterpret_cast<const __half2*>(&h2));
}

__global__ void __launch_bounds__(128) act_split_kernel(const uint16_t* __restrict__ act, uint32_t lda, uint32_t n,
                                                        uint32_t cols_p, uint32_t nst, uint32_t split, uint32_t npad,
                                                        uint8_t* __restrict__ b8, float* __restrict__ colf) {
    grid_dep_launch();  // the linear may start streaming its weights now (no-op without PDL)
    const uint32_t col = blockIdx.x, ch = blockIdx.y;
    const uint32_t g0 = (ch * nst / split) * 8u;  // 16-K groups: 8 per 128-K stage
    const uint32_t g1 = min(((ch + 1) * nst / split) * 8u, cols_p / 16u);
    const uint16_t* a = act + static_cast<size_t>(col) * lda;
    const bool live = col < n;
    grid_dep_wait();  // activations come from the preceding kernel
    __shared__ uint32_t red[4];
    uint32_t amax = 0;  // fp16 magnitude bits: integer order == value order, NaN above inf
    if (live) {
        for (uint32_t gi = g0 + threadIdx.x; gi < g1; gi += blockDim.x) {
            const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(a + 16 * gi));
            const uint4 u1 = __ldg(reinterpret_cast<const uint4*>(a + 16 * gi) + 1);
            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) amax = max(amax, max(w[i] & 0x7fffu, (w[i] >> 16) & 0x7fffu));
        }
    }
    amax = __reduce_max_sync(0xffffffffu, amax);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    amax = max(max(red[0], red[1]), max(red[2], red[3]));
    float scale = 1.0f, inv = 1.0f;
    if (amax >= 0x7c00u) {
        inv = __int_as_float(0x7fc00000);  // inf / NaN in the chunk-column
    } else if (amax != 0u) {
        int ex;
        frexpf(__half2float(__ushort_as_half(static_cast<uint16_t>(amax))), &ex);
        scale = ldexpf(1.0f, 8 - ex);
        inv = ldexpf(1.0f, ex - 8);
    }
    if (threadIdx.x == 0) colf[ch * npad + col] = inv;
    for (uint32_t gi = g0 + threadIdx.x; gi < g1; gi += blockDim.x) {
        uint32_t o[3][4] = {{0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u}};
        if (live) {
            const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(a + 16 * gi));
            const uint4 u1 = __ldg(reinterpret_cast<const uint4*>(a + 16 * gi) + 1);
            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
            float x[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int ak = b < 2 ? 2 * jj + b : 8 + 2 * jj + b - 2;  // actual k of logical 4jj + b
                    const uint16_t hb = static_cast<uint16_t>(w[ak >> 1] >> (16 * (ak & 1)));
                    x[4 * jj + b] = __half2float(__ushort_as_half(hb)) * scale;  // exact
                }
#pragma unroll
            for (int pp = 0; pp < 3; ++pp)
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    const uint32_t v = cvt_e4m3x2(x[i], x[i + 1]);
                    const float2 back = e4m3x2_to_float2(v);
                    o[pp][i >> 2] |= v << (8 * (i & 3));
                    x[i] = (x[i] - back.x) * 16.0f;  // exact residual, next part's scale
                    x[i + 1] = (x[i + 1] - back.y) * 16.0f;
                }
        }
#pragma unroll
        for (int pp = 0; pp < 3; ++pp)
            *reinterpret_cast<uint4*>(b8 + (static_cast<size_t>(pp) * npad + col) * cols_p + 16 * gi) =
                make_uint4(o[pp][0], o[pp][1], o[pp][2], o[pp][3]);
    }
}

// 2-D view of B8: {cols_p bytes, 3 NPAD rows}, box {128, 3 NPAD}, SW128: one
// stage (two k-tiles) of all part-columns, the kind::f8f6f4 B operand.
static cudaError_t make_b8_map(uint8_t* b8, uint32_t cols_p, uint32_t rows, CUtensorMap* map) {
    auto encode = encode_fn();
    if (!encode) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {cols_p, rows};
    const cuuint64_t strides[1] = {cols_p};
    const cuuint32_t box[2] = {128u, rows};
    const cuuint32_t estr[2] = {1u, 1u};
    if (encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, b8, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    return cudaSuccess;
}

template <int F, int NPAD, int G>
static cudaError_t launch_x8(const LinearLaunch& L, const KParams& kp, int grid, cudaStream_t st) {
    using C = X8Cfg<F, NPAD, G>;
    auto kern = fpx_linear_x8_kernel<F, NPAD, G>;
    KParams kq = kp;
    const uint32_t nst = (kp.kt + C::kKS - 1) / C::kKS;
    if (kq.split > nst) {  // K chunks are whole stages
        kq.split = nst;
        kq.units = (kp.rows_p + kTileM - 1) / kTileM * nst;
        grid = std::min<int>(grid, static_cast<int>(kq.units));
    }
    CUtensorMap map, hi_map, lo_map, b8_map;
    if (cudaError_t e = make_act_map(L, NPAD, C::kKS, &map)) return e;
    if (cudaError_t e = make_stream_map(L.s_hi, FmtTraits<F>::kBitsHi, L.rows_p / 64, L.cols_p / 64, C::kKS, &hi_map))
        return e;
    if (cudaError_t e = make_stream_map(L.s_lo, FmtTraits<F>::kBitsLo, L.rows_p / 64, L.cols_p / 64, C::kKS, &lo_map))
        return e;
    if (cudaError_t e = make_b8_map(L.b8, L.cols_p, 3 * NPAD, &b8_map)) return e;
    kq.colf = L.colf;
    kq.pdl = std::min(pdl_mode(), L.pdl_cap);
    // the activation split, then the linear; under programmatic dependent
    // launch the linear's weight stream starts while the split runs
    if (cudaError_t e = launch_pdl(kq.pdl != 0, act_split_kernel, dim3(NPAD, kq.split), 128, 0, st, L.act, L.lda, L.n,
                                   L.cols_p, nst, kq.split, static_cast<uint32_t>(NPAD), L.b8, L.colf))
        return e;
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), C::kSmemBytes)) return e;
    return launch_pdl(kq.pdl != 0, kern, grid, C::kThreads, C::kSmemBytes, st, map, hi_map, lo_map, b8_map, kq);
}

template <int F>
static cudaError_t launch_x8_f(const LinearLaunch& L, const KParams& kp, uint32_t npad, int grid, cudaStream_t st) {
    if (npad <= 16) return launch_x8<F, 16, 4>(L, kp, grid, st);
    if (npad == 32) return launch_x8<F, 32, 4>(L, kp, grid, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_linear_x8(const LinearLaunch& L, const KParams& kp, uint32_t npad, int grid, cudaStream_t st) {
    switch (L.fmt) {
        case kE3M2: return launch_x8_f<kE3M2>(L, kp, npad, grid, st);
        case kE2M3: return launch_x8_f<kE2M3>(L, kp, npad, grid, st);
        case kE2M2: return launch_x8_f<kE2M2>(L, kp, npad, grid, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fpxk
