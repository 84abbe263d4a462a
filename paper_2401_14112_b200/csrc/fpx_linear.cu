// fpx_linear.cu -- the hot path: fused FPx de-quantisation + tcgen05 fp16
// GEMM, C(fp32, col-major, rows_p x n) = dequant(W) x B, B fp16 col-major
// (cols x n).  Drop-in for the reference's gemm_packed (gemm.cpp:170-219).
//
// Work decomposition.  A work unit is (128-row m-tile, K chunk).  The K
// extent of an m-tile is cut into `split` chunks (chunk c covers k-tiles
// [c*KT/split, (c+1)*KT/split)); split depends only on the problem, never on
// which CTA runs a unit, so results are bit-identical however the units are
// distributed (incl. across tile-row shards on several GPUs) and whatever the
// pipeline stage depth.  A persistent grid of <= #SM CTAs takes contiguous
// unit ranges.  split > 1 units write fp32 partials; the last arriving unit
// of an m-tile sums them in chunk order (deterministic) and writes C.
//
// Pipeline stage = KS consecutive k-tiles (64 K each) of one unit: one 3-D
// TMA brings the KS activation tiles (SW128, K-major, N rows padded to NPAD
// by OOB zero fill), four 1-D bulk copies bring the two tile-rows' packed
// high/low streams (contiguous because tiles are stored row-major,
// prepack.cpp:190-191).  One mbarrier round trip per stage, not per k-tile.
//
// CTA = 4*NG + 8 warps, warp-specialised (ids chosen for the high-id-first
// issue arbiter: the single latency-critical warps on top):
//   4NG+6   producer : TMA / bulk copies into the SMEM ring
//   4NG+7   MMA      : one thread issues tcgen05.mma.kind::f16, A from TMEM,
//                      B from the SMEM descriptor, D (fp32) in TMEM
//   4NG+4   TMEM allocator
//   4NG..   epilogue : tcgen05.ld accumulators -> C / split-K partials
//   0..4NG-1 dequant : NG groups of four warps (round-robin over stages); warp
//                      q of a group owns TMEM lanes 32q..32q+31 = tile-row
//                      q/2, chunks 2(q%2), 2(q%2)+1; it LDS's its packed words
//                      (conflict-free jagged rows), runs the register-level
//                      de-quantisation and tcgen05.st's the fp16 A fragments
//                      (16x128b shape == mma A-fragment register order).
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "fpx_linear_common.cuh"

namespace fpxk {


template <int F, int NPAD, int KS_ = (NPAD <= 128 ? 2 : 1), int NG_ = 2>
struct Cfg {
    static constexpr int kKS = KS_;  // k-tiles per pipeline stage
    static constexpr int kNG = NG_;  // dequant warp groups
    static constexpr int kEpiWarp0 = 4 * kNG;     // w0 .. 4NG-1: dequant, quarter = w % 4
    static constexpr int kAllocWarp = kEpiWarp0 + 4;  // TMEM allocator (SMSP 0)
    static constexpr int kProdWarp = kEpiWarp0 + 6;   // TMA producer (SMSP 2)
    static constexpr int kMmaWarp = kEpiWarp0 + 7;    // MMA issuer (SMSP 3)
    static constexpr int kWarps = kEpiWarp0 + 8;
    static constexpr int kThreads = 32 * kWarps;
    static constexpr int kHiBytes = 512 * FmtTraits<F>::kBitsHi;  // per tile
    static constexpr int kLoBytes = 512 * FmtTraits<F>::kBitsLo;
    static constexpr int kBBytes = NPAD * 128;  // 64 k x NPAD fp16 per k-tile
    static constexpr int kHiOff = kKS * kBBytes;  // [B x KS][hi r0][hi r1][lo r0][lo r1]
    static constexpr int kLoOff = kHiOff + 2 * kKS * kHiBytes;
    static constexpr int kStageRaw = kLoOff + 2 * kKS * kLoBytes;
    static constexpr int kStageBytes = (kStageRaw + 1023) / 1024 * 1024;
    static constexpr int kStages = std::min(16, kSmemBudget / kStageBytes);
    static constexpr int kAccBufs = NPAD <= 128 ? 2 : 1;
    static constexpr int kACols = 32 * kKS;  // TMEM columns per A stage
    // A slots, at most the stage ring's depth minus the groups: a group waits
    // `full` for stage si right after its stage si - NG, whose A slot proved
    // the MMA consumed stage si - NG - kAStages; the slot's previous phase
    // (stage si - kStages) must be among those, else the parity wait aliases
    // (the decode kernel's race; here it gave the intermittent
    // NPAD=256 errors).
    static constexpr int kAStages =
        std::min(std::min(8, int((kTmemCols - kAccBufs * NPAD) / kACols)), kStages - kNG);
    static constexpr int kAccCol0 = kAStages * kACols;
    static constexpr int kBarBytes = 8 * (2 * kStages + 2 * kAStages + 4) + 16;
    static constexpr int kSmemBytes = kStages * kStageBytes + kBarBytes + 1024;
    static_assert(kStages >= 2, "smem stages");
    static_assert(kAStages >= kNG + 1, "tmem A stages");
    static_assert(kStages >= kNG + kAStages, "stage ring must cover the groups plus the A-slot ring");
    static_assert(kAccCol0 + kAccBufs * NPAD <= int(kTmemCols), "tmem budget");
};

__device__ __forceinline__ void unit_range(const KParams& p, uint32_t u, uint32_t& mt, uint32_t& ch, uint32_t& k0,
                                           uint32_t& k1) {
    mt = u / p.split;
    ch = u % p.split;
    k0 = (ch * p.kt) / p.split;
    k1 = ((ch + 1) * p.kt) / p.split;
}

// One k-tile of one dequant warp: 4 slices x (3 LDS + 4 register
// iterations) into the two 16-lane x 32-column TMEM A fragments o0 (chunk
// 2h) and o1 (chunk 2h+1), in tcgen05.st 16x128b register order.
template <int F>
__device__ __forceinline__ void dequant_ktile_regs(uint32_t hi, uint32_t lo, int h, uint32_t lane,
                                                  const uint32_t (&sc)[2][2], uint32_t (&o0)[16],
                                                  uint32_t (&o1)[16]) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        uint32_t oa, ob, oc;
        bool ah, bh, chh;
        slice_word_offsets<F>(s, h, lane, oa, ob, oc, ah, bh, chh);
        const uint32_t wa = lds32((ah ? hi : lo) + oa);
        const uint32_t wb = lds32((bh ? hi : lo) + ob);
        const uint32_t wc = lds32((chh ? hi : lo) + oc);
        uint32_t r1[4], r2[4];
        dequant_slice_half<F, kHwCvt>(wa, wb, wc, h, sc, r1, r2);
        // chunk lc = j/2; even j -> regs 4s+{0,1} (a0a1,a2a3), odd j -> 4s+{2,3} (a4a5,a6a7)
        o0[4 * s + 0] = r1[0];
        o0[4 * s + 1] = r2[0];
        o0[4 * s + 2] = r1[1];
        o0[4 * s + 3] = r2[1];
        o1[4 * s + 0] = r1[2];
        o1[4 * s + 1] = r2[2];
        o1[4 * s + 2] = r1[3];
        o1[4 * s + 3] = r2[3];
    }
}

template <int F>
__device__ __forceinline__ void dequant_ktile(uint32_t hi, uint32_t lo, int h, uint32_t lane,
                                             const uint32_t (&sc)[2][2], uint32_t taddr) {
    uint32_t o0[16], o1[16];
    dequant_ktile_regs<F>(hi, lo, h, lane, sc, o0, o1);
    tmem_st_16x128b_x8(taddr, o0);
    tmem_st_16x128b_x8(taddr + (16u << 16), o1);
}

template <int F, int NPAD, int KS_, int NG_>
__global__ void __launch_bounds__(Cfg<F, NPAD, KS_, NG_>::kThreads, 1)
    fpx_linear_kernel(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap hi_map,
                      const __grid_constant__ CUtensorMap lo_map, const KParams p) {
    using C = Cfg<F, NPAD, KS_, NG_>;
    constexpr int KS = C::kKS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = full + C::kStages;
    uint64_t* afull = empty + C::kStages;
    uint64_t* aempty = afull + C::kAStages;
    uint64_t* accfull = aempty + C::kAStages;
    uint64_t* accempty = accfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();

    const uint32_t u_begin = static_cast<uint32_t>((uint64_t)blockIdx.x * p.units / gridDim.x);
    const uint32_t u_end = static_cast<uint32_t>((uint64_t)(blockIdx.x + 1) * p.units / gridDim.x);

    if (warp == C::kProdWarp && lane == 0) prefetch_tmap(&act_map), prefetch_tmap(&hi_map), prefetch_tmap(&lo_map);
    if (warp == C::kMmaWarp && lane == 0) {
        // empty: the MMA commit (B operand read) + the group's 4 warps (packed
        // words read), so every reader of the slot arrives before the producer
        // overwrites it (a thread-visible chain compute-sanitizer can follow)
        for (int i = 0; i < C::kStages; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 5);
        for (int i = 0; i < C::kAStages; ++i) mbar_init(&afull[i], 4), mbar_init(&aempty[i], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&accfull[i], 1), mbar_init(&accempty[i], 4);
        fence_mbar_init();
    }
    if (warp == C::kAllocWarp) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The CTA owns all 512 TMEM columns of its SM (1 CTA/SM), so the
    // allocation can only start at lane 0 / column 0.  Using the constant
    // keeps every TMEM operand of the MMA loop in uniform registers
    // regardless of how the compiler judges the shared-memory load.
#ifdef FPX_TMEM_CONST
    if (*tmem_slot != 0u) __trap();
    constexpr uint32_t tmem = 0;
#else
    const uint32_t tmem = *tmem_slot;
#endif

    if (warp == C::kProdWarp) {
        // ------------------------------------------------ producer
        // One elected thread runs the whole loop: after elect.sync the
        // compiler knows a single lane is active, so every TMA operand stays
        // in uniform registers (no per-instruction broadcast loops).
        if (elect_one()) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_b = policy_evict_last();
            uint32_t si = 0;  // stage counter
            for (uint32_t u = u_begin; u < u_end; ++u) {
                uint32_t mt, ch, k0, k1;
                unit_range(p, u, mt, ch, k0, k1);
                const int32_t tr0 = static_cast<int32_t>(2 * mt);
                for (uint32_t k = k0; k < k1; k += KS, ++si) {
                    const uint32_t st = si % C::kStages, ph = (si / C::kStages) & 1u;
                    mbar_wait(&empty[st], ph ^ 1u);
                    trace_mark(p, kTrProdIssue, si);
                    uint8_t* sb = smem + st * C::kStageBytes;
                    // 3-D boxes {64w, KS, 2}: KS k-tiles of both tile-rows, landing
                    // [tile-row][k-tile][512w B]; a missing second tile-row and
                    // k-tiles past the chunk end (KS > 1) are zero-filled / unused
                    const uint32_t bytes = ((p.dbg & 8u) ? 0u : KS * C::kBBytes) +
                                           ((p.dbg & 4u) ? 0u : 2u * KS * (C::kHiBytes + C::kLoBytes));
                    mbar_arrive_expect_tx(&full[st], bytes);
                    if (!(p.dbg & 8u)) tma_load_3d(sb, &act_map, 0, 0, static_cast<int32_t>(k), &full[st], pol_b);
                    if (!(p.dbg & 4u)) {
                        tma_load_3d(sb + C::kHiOff, &hi_map, 0, static_cast<int32_t>(k), tr0, &full[st], pol_w);
                        tma_load_3d(sb + C::kLoOff, &lo_map, 0, static_cast<int32_t>(k), tr0, &full[st], pol_w);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == C::kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        // One elected thread issues every MMA and the commits that track
        // them (same single-lane / uniform-register reasoning as above).
        if (elect_one()) {
            constexpr uint32_t idesc = umma_idesc_f16(kTileM, NPAD);
            uint32_t si = 0, lu = 0;
            for (uint32_t u = u_begin; u < u_end; ++u, ++lu) {
                uint32_t mt, ch, k0, k1;
                unit_range(p, u, mt, ch, k0, k1);
                const uint32_t ab = lu % C::kAccBufs, abph = (lu / C::kAccBufs) & 1u;
                mbar_wait(&accempty[ab], abph ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem + C::kAccCol0 + ab * NPAD;
                for (uint32_t k = k0; k < k1; k += KS, ++si) {
                    const uint32_t cnt = min(static_cast<uint32_t>(KS), k1 - k);
                    const uint32_t st = si % C::kStages;
                    const uint32_t as = si % C::kAStages, aph = (si / C::kAStages) & 1u;
                    // afull(si) implies full(si): every dequant warp waited on
                    // full[st] (TMA complete_tx) before arriving on afull[as],
                    // so the B tile is visible to the MMA through that chain.
                    mbar_wait(&afull[as], aph);
                    tc_fence_after();
                    trace_mark(p, kTrMmaAfull, si);
                    const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(smem + st * C::kStageBytes));
                    const uint32_t a_tmem = tmem + as * C::kACols;
                    if (!(p.dbg & 2u)) {
#pragma unroll
                        for (int kk = 0; kk < KS; ++kk) {
                            if (kk < static_cast<int>(cnt)) {
#pragma unroll
                                for (uint32_t ks = 0; ks < 4; ++ks)
                                    umma_f16_ts(d_tmem, a_tmem + kk * 32 + ks * 8,
                                                bdesc + static_cast<uint64_t>((kk * C::kBBytes + ks * 32) >> 4), idesc,
                                                (k > k0 || kk > 0 || ks > 0) ? 1u : 0u);
                            }
                        }
                    }
                    trace_mark(p, kTrMmaIssued, si);
                    umma_commit(&empty[st]);
                    umma_commit(&aempty[as]);
                }
                umma_commit(&accfull[ab]);
            }
        }
        __syncwarp();
    } else if (warp >= C::kEpiWarp0 && warp < C::kEpiWarp0 + 4) {
        // ------------------------------------------------ epilogue
        const uint32_t q = warp & 3u;
        const uint32_t row_l = 32 * q + lane;
        uint32_t lu = 0;
        for (uint32_t u = u_begin; u < u_end; ++u, ++lu) {
            uint32_t mt, ch, k0, k1;
            unit_range(p, u, mt, ch, k0, k1);
            const uint32_t ab = lu % C::kAccBufs, abph = (lu / C::kAccBufs) & 1u;
            if (p.dbg & 16u) mbar_wait_sleep(&accfull[ab], abph, 256);
            else mbar_wait(&accfull[ab], abph);
            if (q == 0 && lane == 0) trace_mark(p, kTrEpiFull, lu);
            tc_fence_after();
            const uint32_t m = mt * kTileM + row_l;
            const bool row_ok = m < p.rows_p;
            float* part = p.ws + (static_cast<size_t>(mt) * p.split + ch) * NPAD * kTileM;
#pragma unroll 1
            for (uint32_t c0 = 0; c0 < NPAD; c0 += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tmem + ((32 * q) << 16) + C::kAccCol0 + ab * NPAD + c0, v);
                tmem_ld_wait();
                if (c0 < p.n) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t col = c0 + j;
                        if (col < p.n) {
                            if (p.split == 1) {
                                if (row_ok) c_store(p, m, col, __uint_as_float(v[j]));
                            } else {
                                part[static_cast<size_t>(col) * kTileM + row_l] = __uint_as_float(v[j]);
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[ab]);
            if (p.split > 1) {
                __threadfence();
                __syncwarp();
                uint32_t old = 0;
                if (lane == 0) old = atomicAdd(&p.counters[mt * 4 + q], 1u);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old == p.split - 1) {
                    // last arriver: C = ((P0 + P1) + P2) + ... in chunk order
                    __threadfence();
                    const float* base = p.ws + static_cast<size_t>(mt) * p.split * NPAD * kTileM + row_l;
                    for (uint32_t c0 = 0; c0 < p.n; c0 += 16) {
                        float acc[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[j] = 0.0f;
                        for (uint32_t cc = 0; cc < p.split; ++cc) {
                            const float* pc = base + (static_cast<size_t>(cc) * NPAD + c0) * kTileM;
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (c0 + j < p.n) acc[j] += __ldcg(pc + j * kTileM);
                        }
                        if (row_ok) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (c0 + j < p.n) c_store(p, m, c0 + j, acc[j]);
                        }
                    }
                    if (lane == 0) p.counters[mt * 4 + q] = 0;  // self-cleaning for the next launch
                }
            }
        }
    } else if (warp < C::kEpiWarp0) {
        // ------------------------------------------------ de-quantisers
        const uint32_t g = warp >> 2;
        const uint32_t q = warp & 3u;
        const int h = static_cast<int>(q & 1u);
        const uint32_t r = q >> 1;
        uint32_t si = 0;
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, k0, k1;
            unit_range(p, u, mt, ch, k0, k1);
            const uint32_t tr = 2 * mt + r;
            const bool valid = tr < p.tile_rows;
            uint32_t sc[2][2] = {{0, 0}, {0, 0}};
            if (valid) {
#pragma unroll
                for (int lc = 0; lc < 2; ++lc)
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        const uint32_t row = tr * 64 + 16 * (2 * h + lc) + 8 * hf + lane / 4;
                        sc[lc][hf] = row_scale_for<F, kHwCvt>(p.scales[row]);
                    }
            }
            for (uint32_t k = k0; k < k1; k += KS, ++si) {
                if (si % C::kNG != g) continue;
                const uint32_t cnt = min(static_cast<uint32_t>(KS), k1 - k);
                const uint32_t st = si % C::kStages, ph = (si / C::kStages) & 1u;
                const uint32_t as = si % C::kAStages, aph = (si / C::kAStages) & 1u;
                if (p.dbg & 32u) mbar_wait_sleep(&aempty[as], aph ^ 1u, 32);
                else mbar_wait(&aempty[as], aph ^ 1u);
                if (q == 0 && lane == 0) trace_mark(p, kTrDqAempty, si);
                mbar_wait(&full[st], ph);
                if (q == 0 && lane == 0) trace_mark(p, kTrDqFull, si);
                tc_fence_after();
                if (valid && !(p.dbg & 1u)) {
                    const uint32_t sb = smem_u32(smem + st * C::kStageBytes);
                    const uint32_t ta = tmem + ((32 * q) << 16) + as * C::kACols;
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk) {
                        if (kk < static_cast<int>(cnt))
                            dequant_ktile<F>(sb + C::kHiOff + (r * KS + kk) * C::kHiBytes,
                                             sb + C::kLoOff + (r * KS + kk) * C::kLoBytes, h, lane, sc, ta + kk * 32);
                    }
                    tmem_st_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) trace_mark(p, q == 0 ? kTrDqDone : kTrDqDone1 + q - 1, si);
                if (lane == 0) mbar_arrive(&afull[as]), mbar_arrive(&empty[st]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == C::kAllocWarp) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

// ===========================================================================
// Decode kernel (batch <= 32, the memory-bound regime).
//
// Measured constraints that shape it (tools/micro/, B200):
//  * a kind::f16 tcgen05.mma with M=128, K=16 occupies the tensor pipe for
//    ~44 cycles for ANY N <= 128 (operand fetch, not math, bounds it), i.e.
//    at most ~46 fp16 weights/clk/SM -- only ~1.5x the ~31 weights/clk/SM
//    the HBM roofline needs;
//  * every tcgen05.commit costs ~300 tensor-pipe cycles, so commits are
//    batched (one per kBS stages);
//  * tcgen05.commit from several concurrently issuing threads loses
//    arrivals, so exactly one thread issues all MMAs and commits;
//  * loops that issue TMA / MMA run warp-wide with warp-uniform control flow
//    (bookkeeping in uniform registers) and elect one lane per instruction
//    inside the asm.
//
// Pipeline (one persistent CTA per SM, units = (128-row tile, K chunk)):
//  producers (one weight warp, one activation warp) --TMA--> weight ring (SW stages: KS k-tiles of packed
//    weights for the unit's 2 tile-rows) and activation ring (SB stages: KS
//    activation k-tiles, the MMA's B operand)
//  de-quantiser groups (G x 4 warps; stage si -> group si % G): LDS the
//    stage's packed words, release the weight stage at once (it is consumed
//    in registers), de-quantise, tcgen05.st into the TMEM A ring (R slots)
//  MMA warp: stages in order, KS x 4 MMAs each into the unit's single fp32
//    accumulator (double-buffered across units); one commit per kBS stages
//    releases their activation stages and A slots; one commit per unit
//    hands the accumulator to the epilogue
//  epilogue (4 warps): tcgen05.ld -> C, or split-K partials + fixed-order
//    last-arriver reduction.
// The weight ring -- where the bytes are -- recycles as soon as the packed
// words are in registers; only the small activation and A rings wait for
// MMA completion.  The k-tiles of a unit are accumulated in K order by one
// issuer, so the result is a pure function of (W, act, split):
// deterministic and independent of the grid and of the group count.
// Every stage is a full KS k-tiles: a K tail beyond the last k-tile is
// zero-filled by TMA (weights and activations), contributing exact zeros.
//
// Warps: 0 .. 4G-1 de-quantisers (group w/4, TMEM lane quarter w%4),
// 4G .. 4G+3 epilogue (quarter w%4), 4G+4 MMA issuer, 4G+5 .. 4G+4+P weight
// producers (the first also allocates TMEM), 4G+5+P activation producer.
#ifndef FPX_DEC_PW
#define FPX_DEC_PW 1
#endif
template <int F, int NPAD, int KS_, int G_, int P_ = FPX_DEC_PW>
struct GCfg {
    static constexpr int kKS = KS_;
    static constexpr int kG = G_;
    static constexpr int kP = P_;
    static constexpr int kEpiWarp0 = 4 * kG;
    static constexpr int kMmaWarp = kEpiWarp0 + 4;
    static constexpr int kProdWarp = kMmaWarp + 1;
    static constexpr int kActWarp = kProdWarp + kP;  // kP weight producers, then the activation producer
    static constexpr int kWarps = kActWarp + 1;
    static constexpr int kThreads = 32 * kWarps;
    static constexpr int kHiBytes = 512 * FmtTraits<F>::kBitsHi;  // per 64x64 tile
    static constexpr int kLoBytes = 512 * FmtTraits<F>::kBitsLo;
    static constexpr int kBBytes = NPAD * 128;                    // per activation k-tile
    // weight stage: [hi r0 x KS][hi r1 x KS][lo r0 x KS][lo r1 x KS]
    static constexpr int kLoOff = 2 * kKS * kHiBytes;
    static constexpr int kWStageBytes = (2 * kKS * (kHiBytes + kLoBytes) + 1023) / 1024 * 1024;
    static constexpr int kBStageBytes = (kKS * kBBytes + 1023) / 1024 * 1024;
    // Wide batches (NPAD >= 64): the MMA warp itself waits for each stage's
    // activations, so the activation ring (16-32 KB stages) need not be as
    // deep as the A-slot ring, and one accumulator buffer leaves TMEM for
    // more A slots (a CTA runs one long unit at the default splits; a
    // second unit waits for the epilogue to drain the first).  Narrow
    // batches keep the de-quantisers' activation wait (one MMA-loop wait
    // less) and double-buffered accumulators.
    static constexpr bool kMmaWaitsB = NPAD >= 64;
#ifndef FPX_DEC_WIDE_ACCBUFS
#define FPX_DEC_WIDE_ACCBUFS 2
#endif
    static constexpr int kAccBufs = NPAD >= 64 ? FPX_DEC_WIDE_ACCBUFS : 2;
    static constexpr int kAccCol0 = int(kTmemCols) - kAccBufs * NPAD;  // accumulator buffer(s) at the top
    static constexpr int kASlotsMax = (kAccCol0 / 32) / kKS;      // A stage slots the TMEM budget allows
#ifndef FPX_DEC_SB
#define FPX_DEC_SB 12
#endif
#ifndef FPX_DEC_SB32
#define FPX_DEC_SB32 FPX_DEC_SB
#endif
#ifndef FPX_DEC_SB64
#define FPX_DEC_SB64 4
#endif
#ifndef FPX_DEC_SB128
#define FPX_DEC_SB128 3
#endif
#ifndef FPX_DEC_SMEM_KB
#define FPX_DEC_SMEM_KB 216
#endif
    // The activation ring only has to outlast a commit batch; everything else
    // goes to the weight ring, whose depth (bytes in flight per SM) sets the
    // sustainable HBM rate against the ~2.5 us loaded TMA latency.
    static constexpr int kBStages =
        NPAD <= 16 ? FPX_DEC_SB : (NPAD == 32 ? FPX_DEC_SB32 : (NPAD == 64 ? FPX_DEC_SB64 : FPX_DEC_SB128));
    // Weight producer i issues stages i, i+P, ... into slots it alone owns
    // (SW % P == 0), so it only ever waits on the consumption of its own
    // previous use of a slot: no parity aliasing.  Several producers because
    // one warp issues a TMA only every ~0.1 us (measured), below the rate the
    // HBM roofline needs in bursts.
    static constexpr int kWStages =
        std::min(24, (FPX_DEC_SMEM_KB * 1024 - 2048 - kBStages * kBStageBytes) / kWStageBytes) / kP * kP;
    // TMEM A stage slots, at most the activation ring's depth and the weight
    // ring's depth minus the groups (see the SB >= R and SW >= G + R
    // assertions below).
    static constexpr int kASlots = std::min(std::min(kASlotsMax, kMmaWaitsB ? 16 : kBStages), kWStages - kG);
#ifndef FPX_DEC_BS
#define FPX_DEC_BS 3
#endif
    // stages per commit batch; with R >= G + BS a group never waits for the
    // batch holding its own previous stage (R = 6, G = 3 or 4 at NPAD 64 /
    // 128 takes BS = 2)
    static constexpr int kBS =
        std::max(1, std::min(std::min(std::min(FPX_DEC_BS, kASlots / 2), std::max(1, kASlots - kG)), kBStages - 1));
    static constexpr int kNB = (std::max(kBStages, kASlots) + kBS - 1) / kBS + 3;  // batch barriers (no aliasing)
    static constexpr int kBarBytes = 8 * (2 * kWStages + kBStages + kNB + kASlots + 5) + 16;
    static constexpr int kSmemBytes = kWStages * kWStageBytes + kBStages * kBStageBytes + kBarBytes + 1024;
    static constexpr uint32_t kWTx = 2 * kKS * (kHiBytes + kLoBytes);
    static constexpr uint32_t kBTx = kKS * kBBytes;
    static_assert(kBStages >= kBS + 1 && kASlots >= kBS + 1 && kWStages >= kG + 1, "ring depths");
    // A de-quantiser group waits bfull for stage si with a parity wait.  That
    // is only unambiguous if the activation producer has already issued stage
    // si - SB into the same slot; it has issued at least stage si - R (the
    // MMA consumed it, which freed this group's A slot).  Hence SB >= R.
    // (SB < R let a group pass the wait on the slot's older phase: wrong
    // results with SB=6, faults with smaller rings.)
    static_assert(kMmaWaitsB || kBStages >= kASlots, "activation ring must be at least as deep as the A-slot ring");
    // The same argument for the weight ring: a group waits wfull for stage si
    // right after finishing its stage si - G, whose A slot required the MMA to
    // have consumed stage si - G - R -- so every stage up to there has landed.
    // The slot's previous phase (stage si - SW) must be among them:
    // SW >= G + R.  (NPAD=64 had SW 9 < 4 + 6.)
    static_assert(kWStages >= kG + kASlots, "weight ring must cover the groups plus the A-slot ring");
    static_assert(kWStages % kP == 0, "each weight slot is owned by one producer warp");
    static_assert(NPAD <= 128, "double-buffered NPAD-column accumulators + A ring must fit 512 TMEM columns");
};





template <int F, int NPAD, int KS_, int G_>
__global__ void __launch_bounds__(GCfg<F, NPAD, KS_, G_>::kThreads, 1)
    fpx_linear_decode_kernel(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap hi_map,
                             const __grid_constant__ CUtensorMap lo_map, const KParams p) {
    using C = GCfg<F, NPAD, KS_, G_>;
    constexpr int KS = C::kKS, G = C::kG, SW = C::kWStages, SB = C::kBStages, R = C::kASlots, BS = C::kBS,
                  NB = C::kNB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bring = smem;                              // [SB] activation stages (SW128 K-major)
    uint8_t* wring = smem + SB * C::kBStageBytes;       // [SW] packed weight stages
    uint64_t* bars = reinterpret_cast<uint64_t*>(wring + SW * C::kWStageBytes);
    uint64_t* wfull = bars;            // [SW] weights landed               (tx bytes)
    uint64_t* wempty = wfull + SW;     // [SW] group's 4 warps read the stage (arrivals)
    uint64_t* bfull = wempty + SW;     // [SB] activations landed           (tx bytes)
    uint64_t* done = bfull + SB;       // [NB] MMAs of a batch of BS stages complete (commit)
    uint64_t* aready = done + NB;      // [R]  group's 4 warps stored the stage's A tiles
    uint64_t* accfull = aready + R;    // [2]  unit's MMAs complete (commit)
    uint64_t* accempty = accfull + 2;  // [2]  epilogue drained the accumulator
    uint64_t* sready = accempty + 2;   // [1]  the 128 epilogue threads staged the units' row scales (uscale)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sready + 1);
    // [4] per epilogue lane quarter: 1 + tile of a deferred last-unit
    // reduction, or 0.  A separate static array: stores next to tmem_slot
    // cost the MMA loop its uniform-register TMEM operands (ptxas).
    __shared__ uint32_t red_tq[4 * kMaxDefer];  // per quarter: tile * 4 + quarter of each deferred reduction
    __shared__ uint32_t red_n[4];
    // Unit table: the CTA's units resolved once in the prologue (tile, chunk,
    // first stage, stages) and their tiles' row scales staged in shared memory
    // by the epilogue warps, so a unit boundary costs no integer divisions
    // and no dependent global load on any role's critical path (it cost
    // every de-quantiser group ~0.5 us per boundary).  More than kMaxUnits
    // units per CTA (tiny grids) fall back to computing both on the spot.
    __shared__ uint4 utab[kMaxUnits];
    __shared__ uint16_t uscale[kMaxUnits][kTileM];

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();
    const uint32_t u_begin = static_cast<uint32_t>((uint64_t)blockIdx.x * p.units / gridDim.x);
    const uint32_t u_end = static_cast<uint32_t>((uint64_t)(blockIdx.x + 1) * p.units / gridDim.x);
    const bool tab = u_end - u_begin <= kMaxUnits;
    if (threadIdx.x == 0) trace_cta(p, 15);  // kernel entry, before the prologue
    if (tab && threadIdx.x < u_end - u_begin) {
        uint32_t mt, ch, s0, ns;
        unit_stages<KS>(p, u_begin + threadIdx.x, mt, ch, s0, ns);
        utab[threadIdx.x] = make_uint4(mt, ch, s0, ns);
    }
    auto unit_of = [&](uint32_t u, uint32_t& mt, uint32_t& ch, uint32_t& s0, uint32_t& ns) {
        if (tab) {
            const uint4 e = utab[u - u_begin];
            mt = e.x, ch = e.y, s0 = e.z, ns = e.w;
        } else {
            unit_stages<KS>(p, u, mt, ch, s0, ns);
        }
    };

    if (warp == C::kEpiWarp0 && lane == 0) {
        for (int i = 0; i < SW; ++i) mbar_init(&wfull[i], 1), mbar_init(&wempty[i], 4);
        for (int i = 0; i < SB; ++i) mbar_init(&bfull[i], 1);
        for (int i = 0; i < NB; ++i) mbar_init(&done[i], 1);
        for (int i = 0; i < R; ++i) mbar_init(&aready[i], 4);
        for (int i = 0; i < 2; ++i) mbar_init(&accfull[i], 1), mbar_init(&accempty[i], 4);
        for (int i = 0; i < 4; ++i) red_n[i] = 0;
        mbar_init(sready, 128);
        fence_mbar_init();
    }
    if (warp == C::kProdWarp) {
        if (lane == 0) prefetch_tmap(&act_map), prefetch_tmap(&hi_map), prefetch_tmap(&lo_map);
        tmem_alloc<kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The CTA owns all 512 TMEM columns of its SM (1 CTA/SM), so the
    // allocation can only start at lane 0 / column 0.  Using the constant
    // keeps every TMEM operand of the MMA loop in uniform registers
    // regardless of how the compiler judges the shared-memory load.
#ifdef FPX_TMEM_CONST
    if (*tmem_slot != 0u) __trap();
    constexpr uint32_t tmem = 0;
#else
    const uint32_t tmem = *tmem_slot;
#endif
    if (threadIdx.x == 0) trace_cta(p, 0);
    // PDL only: let the next launch be scheduled (its CTAs still need this
    // CTA's shared memory / TMEM, so they start as these exit).
    if (p.pdl) grid_dep_launch();

    if (p.dbg & 256u) {
        // FPX_LINEAR_DBG=256: launch + prologue + teardown only (bring-up)
    } else if (warp >= C::kProdWarp && warp < C::kActWarp) {
        // ------------------------------------------------ weight producers
        // Weights only, producer pw every P-th stage: the sole throttle is the weight ring
        // (slots come back as soon as a group has the words in registers),
        // so up to SW stages of HBM reads stay in flight.  Sharing a warp with
        // the activation loads -- whose slots come back only with MMA
        // completion -- capped the weight prefetch depth at the activation
        // ring's.  Weights are immutable during the call, so under PDL they
        // are requested BEFORE waiting for the preceding kernel.
        // PDL mode 2 (default): packed weights are immutable while linears run
        // (inference), so the weight stream starts before the preceding kernel
        // has finished; mode 1 waits for it like every other global read.
        if (p.pdl != 2u) grid_dep_wait();
        const bool leader = lane == 0;
        const uint32_t pw = warp - C::kProdWarp;
        const uint64_t pol_w = policy_evict_first();
        const uint32_t wtx = (p.dbg & 4u) ? 0u : C::kWTx;
        uint32_t si = 0, ws = pw, wph = 0;  // stage, weight slot, slot parity
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, s0, ns;
            unit_of(u, mt, ch, s0, ns);
            const int32_t tr0 = static_cast<int32_t>(2 * mt);
            for (uint32_t ls = 0; ls < ns; ++ls, ++si) {
                if (si % C::kP != pw) continue;
                const int32_t k = static_cast<int32_t>((s0 + ls) * KS);
                // slot free once the group that read it (stage si - SW) released it
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
                ws += C::kP;
                if (ws >= static_cast<uint32_t>(SW)) ws -= SW, wph ^= 1u;
            }
        }
    } else if (warp == C::kActWarp) {
        // ------------------------------------------------ activation producer
        // Activations may be written by the preceding kernel: wait for it.
        grid_dep_wait();
        const bool leader = lane == 0;
        const uint64_t pol_b = policy_evict_last();
        uint32_t si = 0, bs = 0;
        uint32_t b = 0, bb = 0, nbs = 0, nph = 0;  // batch releasing slot bs: stage si - SB
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, s0, ns;
            unit_of(u, mt, ch, s0, ns);
            const uint32_t btx = (p.dbg & 8u) ? 0u : C::kBTx;
            for (uint32_t ls = 0; ls < ns; ++ls, ++si) {
                const int32_t k = static_cast<int32_t>((s0 + ls) * KS);
                if (si >= static_cast<uint32_t>(SB)) {
                    // stage si - SB belongs to MMA batch b = (si - SB) / BS
                    wait_rec(p, &done[nbs], nph, 7, si);
                    if (++bb == static_cast<uint32_t>(BS)) {
                        bb = 0;
                        ++b;
                        if (++nbs == static_cast<uint32_t>(NB)) nbs = 0, nph ^= 1u;
                    }
                }
                if (leader) {
                    mbar_arrive_expect_tx(&bfull[bs], btx);
                    if (!(p.dbg & 8u))
                        tma_load_3d(bring + bs * C::kBStageBytes, &act_map, 0, 0, k, &bfull[bs], pol_b);
                }
                __syncwarp();
                if (++bs == static_cast<uint32_t>(SB)) bs = 0;
            }
        }
        (void)b;
    } else if (warp == C::kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = umma_idesc_f16(kTileM, NPAD);
        const bool leader = lane == 0;
        // ring positions advance incrementally (no divisions on this
        // single-issue critical path)
        uint32_t si = 0, lu = 0;
        uint32_t as = 0, aph = 0;   // A slot and its phase parity
        uint32_t bsl = 0;           // activation slot
        uint32_t nb = 0, nbs = 0;   // stages in the open commit batch, batch barrier slot
        uint32_t nbatch = 0;        // batch commits issued
        uint32_t bph = 0;           // activation slot parity (kMmaWaitsB)
        for (uint32_t u = u_begin; u < u_end; ++u, ++lu) {
            uint32_t mt, ch, s0, ns;
            unit_of(u, mt, ch, s0, ns);
            constexpr uint32_t AB = C::kAccBufs;
            const uint32_t ab = lu % AB;
            wait_rec(p, &accempty[ab], ((lu / AB) & 1u) ^ 1u, 5, lu);  // epilogue done with unit lu - AB
            tc_fence_after();
            const uint32_t d_tmem = tmem + C::kAccCol0 + ab * NPAD;
            for (uint32_t ls = 0; ls < ns; ++ls, ++si) {
                if (leader) trace_mark(p, kTrMmaWait, si);
                // narrow batches: aready implies the activation stage landed (the
                // group waited bfull first); wide batches wait for it here
                if constexpr (C::kMmaWaitsB) wait_rec(p, &bfull[bsl], bph, 8, si);
                wait_rec(p, &aready[as], aph, 4, si);
                tc_fence_after();
                if (leader) trace_mark(p, kTrMmaGo, si);
                const uint32_t a_tmem = tmem + as * KS * 32;
                const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bring + bsl * C::kBStageBytes));
                const uint32_t acc0 = ls > 0 ? 1u : 0u;  // the unit's first k-tile overwrites
                if (p.dbg & 2u) {
                } else {
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
                        for (uint32_t ks = 0; ks < 4; ++ks)
                            umma_f16_ts_warp(d_tmem, a_tmem + kk * 32 + ks * 8,
                                             bdesc + static_cast<uint64_t>((kk * C::kBBytes + ks * 32) >> 4), idesc,
                                             (kk > 0 || ks > 0) ? 1u : acc0);
                }
                if (++nb == static_cast<uint32_t>(BS)) {
                    umma_commit_warp(&done[nbs]);
                    ++nbatch;
                    nb = 0;
                    nbs = (nbs + 1 == static_cast<uint32_t>(NB)) ? 0u : nbs + 1;
                }
                if (leader) trace_mark(p, kTrMmaIssued, si);
                if (++as == static_cast<uint32_t>(R)) as = 0, aph ^= 1u;
                if (++bsl == static_cast<uint32_t>(SB)) bsl = 0, bph ^= 1u;
            }
            umma_commit_warp(&accfull[ab]);
        }
        if (nb != 0) umma_commit_warp(&done[nbs]), ++nbatch;  // final partial batch
        // The last batch commits have no consumer (no later stage reuses
        // their slots) and the final partial one is even issued after the
        // last accfull commit: wait for the newest so that no tcgen05.commit
        // arrival can land in this CTA's shared memory after it exits -- i.e.
        // in the barriers of the next CTA placed on this SM.
        if (nbatch != 0) {
            const uint32_t b = nbatch - 1;
            mbar_wait(&done[b % NB], (b / NB) & 1u);
        }
    } else if (warp >= C::kEpiWarp0) {
        // ------------------------------------------------ epilogue
        const uint32_t q = warp & 3u;
        const uint32_t row_l = 32 * q + lane;
        if (tab) {
            // stage the row scales of the CTA's units (zero past the last
            // tile-row); immutable like the weights under PDL mode 2
            if (p.pdl != 2u) grid_dep_wait();
            for (uint32_t i = 0; i < u_end - u_begin; ++i) {
                const uint32_t m = utab[i].x * kTileM + row_l;
                uscale[i][row_l] = m < p.rows_p ? __ldg(&p.scales[m]) : uint16_t(0);
            }
            mbar_arrive(sready);  // every writer arrives: its stores are released by its own arrive
        }
        grid_dep_wait();  // C / partials / counters may still be in use by the preceding kernel
        uint32_t ndefer = 0;  // this quarter's deferred reductions (red_n[q] after the loop)
        uint32_t lu = 0;
        for (uint32_t u = u_begin; u < u_end; ++u, ++lu) {
            uint32_t mt, ch, s0, ns;
            unit_of(u, mt, ch, s0, ns);
            const uint32_t ab = lu % C::kAccBufs;
            wait_rec(p, &accfull[ab], (lu / C::kAccBufs) & 1u, 2, lu);
            if (q == 0 && lane == 0) trace_mark(p, kTrEpiFull, lu);
            tc_fence_after();
            const uint32_t m = mt * kTileM + row_l;
            const bool row_ok = m < p.rows_p;
            // the de-quantiser warps of this lane quarter took the same vote
            // (scale_in_epilogue_ok): if it passed, apply the row scale here
            const uint16_t raw_s = tab ? uscale[lu][row_l]
                                       : (2 * mt + (q >> 1) < p.tile_rows ? __ldg(&p.scales[m]) : uint16_t(0));
            const bool epi_scale = __all_sync(0xffffffffu, scale_in_epilogue_ok(raw_s));
            const float s_row = epi_scale ? __half2float(__ushort_as_half(raw_s)) : 1.0f;
            // split-K partials: [unit][col/4][row][4] fp32 -- a lane's 4 columns
            // are one 16-byte vector and a warp's 32 rows are contiguous, so the
            // stores here and the loads of the reduction are coalesced float4s
            float* part = p.ws + (static_cast<size_t>(mt) * p.split + ch) * kTileM * NPAD + row_l * 4;
            const uint32_t tacc = tmem + ((32 * q) << 16) + C::kAccCol0 + ab * NPAD;
#pragma unroll
            for (uint32_t c0 = 0; c0 < NPAD; c0 += 16) {
                uint32_t v[16];
                if (ns > 0) {
                    tmem_ld_32x32b_x16(tacc + c0, v);
                    tmem_ld_wait();
                    if (epi_scale) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * s_row);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = 0u;  // empty K chunk contributes zero
                }
                if (p.split == 1) {
                    if (c0 < p.n && row_ok) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (c0 + j < p.n) c_store(p, m, c0 + j, __uint_as_float(v[j]));
                    }
                } else if (c0 < p.n) {
                    // columns >= n hold exact zeros (zero-filled activations)
                    // kept in L2 (evict_last) against the evict_first weight stream:
                    // the last arriver reads them back on the launch's tail
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
        }
        if (p.split > 1) {
            // Split-K arrivals for all of the CTA's chunks at once, after its
            // last unit: one release fence per epilogue warp instead of one
            // per unit (a MEMBAR under full HBM load stalls the warp for
            // microseconds, and the accumulator it holds stalls the MMA two
            // units later).  The last arriver of a (tile, quarter) reduces it
            // in the CTA-wide pass after the main loop (final_split_reduce),
            // or here when its deferral list is full.
            __threadfence();
            __syncwarp();
            bool acquired = false;
            // lane i arrives for the CTA's unit ub + i: one atomic round trip per 32 units
            for (uint32_t ub = u_begin; ub < u_end; ub += 32) {
                const uint32_t u = ub + lane;
                uint32_t mt = 0, ch, s0, ns;
                bool last = false;
                if (u < u_end) {
                    unit_of(u, mt, ch, s0, ns);
                    last = atomicAdd(&p.counters[mt * 4 + q], 1u) == p.split - 1;
                }
                uint32_t lasts = __ballot_sync(0xffffffffu, last);
                if (lasts != 0u && !acquired) {
                    __threadfence();  // acquire side of the counters (the other chunks' partials)
                    acquired = true;
                }
                if (last) p.counters[mt * 4 + q] = 0;  // self-cleaning for the next launch
                while (lasts != 0u) {
                    const uint32_t i = __ffs(lasts) - 1;
                    lasts &= lasts - 1;
                    const uint32_t mti = __shfl_sync(0xffffffffu, mt, i);
                    if (ndefer < kMaxDefer) {
                        if (lane == 0) red_tq[q * kMaxDefer + ndefer] = mti * 4 + q;
                        ++ndefer;
                    } else {
                        const uint32_t m = mti * kTileM + row_l;
                        split_reduce_rows<NPAD>(p, mti, row_l, m, m < p.rows_p);
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
        // Row scales: from uscale (unit table), else fetched one unit ahead
        // (a dependent global load at every unit start would stall all
        // groups at the same moment).
        auto fetch_scales = [&](uint32_t uu, uint16_t (&raw)[2][2]) {
            if (tab) {
#pragma unroll
                for (int lc = 0; lc < 2; ++lc)
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf)
                        raw[lc][hf] = uscale[uu - u_begin][64 * r + 16 * (2 * h + lc) + 8 * hf + lane / 4];
                return;
            }
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
        // PDL mode 2: the row scales are immutable like the weights, so the
        // groups de-quantise their first stages while the preceding kernel
        // drains; they block on bfull until the activations (loaded after
        // griddepcontrol.wait) land.  That wait is unambiguous because SB >= R
        // (GCfg); with SB < R it aliased and this early start exposed it.
        if (p.pdl != 2u) grid_dep_wait();
        if (tab) mbar_wait(sready, 0);
        uint16_t nxt[2][2] = {{0, 0}, {0, 0}};
        if (u_begin < u_end) fetch_scales(u_begin, nxt);
        uint32_t si = 0;
        for (uint32_t u = u_begin; u < u_end; ++u) {
            uint32_t mt, ch, s0, ns;
            unit_of(u, mt, ch, s0, ns);
            uint32_t sc[2][2];  // zero for a missing tile-row (fetch_scales)
            bool ok_t = true;
#pragma unroll
            for (int lc = 0; lc < 2; ++lc)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    sc[lc][hf] = row_scale_for<F, kHwCvt>(nxt[lc][hf]);
                    ok_t = ok_t && scale_in_epilogue_ok(nxt[lc][hf]);
                }
            // warp-uniform: the scale goes to the epilogue for this unit's 32 rows
            const bool epi_scale = __all_sync(0xffffffffu, ok_t);
            if (u + 1 < u_end) fetch_scales(u + 1, nxt);
            // this group's stages of the unit: si % G == g
            uint32_t ls = (g + G - si % G) % G;
            // Two copies of the stage loop (scale in registers / in the
            // epilogue), selected once per unit: a per-stage select was
            // if-converted by ptxas into executing both.
            auto stage_loop = [&](auto scale_tag) {
                constexpr bool kScale = decltype(scale_tag)::value;
                for (si += ls; ls < ns; ls += G, si += G) {
                    const uint32_t ws = si % SW, as = si % R;
                    const uint32_t wb = smem_u32(wring + ws * C::kWStageBytes);
                    if (q == 0 && lane == 0) trace_mark(p, kTrDqAempty, si);
                    wait_rec(p, &wfull[ws], (si / SW) & 1u, 3, si);
                    if (q == 0 && lane == 0) trace_mark(p, kTrDqFull, si);
                    if (warp == 0 && lane == 0 && si == 0) trace_cta(p, 14);  // first weight stage landed
                    // all of the stage's packed words into registers, then hand the
                    // weight stage back to the producers
                    uint32_t w[KS][12];
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk)
                        load_ktile_words<F>(wb + (r * KS + kk) * C::kHiBytes, wb + C::kLoOff + (r * KS + kk) * C::kLoBytes,
                                            h, lane, w[kk]);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wempty[ws]);
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk) {
                        // A missing second tile-row (odd tile_rows) arrives zero-filled
                        // by TMA and is multiplied by a zero scale: every A-slot lane
                        // an MMA reads holds an exact zero.  (No separate zeroing
                        // path: ptxas if-converted it into every stage.)
                        uint32_t o0[16], o1[16];
                        dequant_words<F, kScale>(w[kk], h, sc, o0, o1);
                        if (kk == 0) {
                            // A slot `as` last held stage si - R: free once that stage's batch completed
                            if (q == 0 && lane == 0) trace_mark(p, kTrDqDone, si);
                            if (si >= static_cast<uint32_t>(R)) {
                                const uint32_t b = (si - R) / BS;
                                wait_rec(p, &done[b % NB], (b / NB) & 1u, 6, si);
                            }
                            if (q == 0 && lane == 0) trace_mark(p, kTrDqDone1, si);
                            tc_fence_after();
                        }
                        tmem_st_16x128b_x8(tq + (as * KS + kk) * 32, o0);
                        tmem_st_16x128b_x8(tq + (as * KS + kk) * 32 + (16u << 16), o1);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    // the MMA reads this stage's activations: make sure they landed
                    // (wide batches: the MMA warp waits for them itself)
                    if constexpr (!C::kMmaWaitsB) wait_rec(p, &bfull[si % SB], (si / SB) & 1u, 8, si);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aready[as]);
                    if (q == 0 && lane == 0) trace_mark(p, kTrMmaAfull, si);
                }
            };
            if (epi_scale) stage_loop(std::false_type{});
            else stage_loop(std::true_type{});
            si -= ls - ns;  // back to the first stage of the next unit
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
        if (lane == 0) trace_cta(p, 12);  // teardown: every warp of the CTA is done
        tmem_dealloc<kTmemCols>(tmem);
        if (lane == 0) trace_cta(p, 13);  // after TMEM dealloc
    }
    if (p.split > 1) final_split_reduce<NPAD>(p, red_tq, red_n, C::kThreads);
    if (FPX_TRACE && threadIdx.x == 0) trace_cta(p, 8);  // kernel exit (after the deferred reductions)
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-(function, device)
// setting: a process driving several GPUs sets it once on each device it
// launches on, and a failed attempt is retried on the next call.
cudaError_t ensure_smem_attr(const void* kern, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;  // (kernel, device) pairs already configured
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& d : done)
        if (d.first == kern && d.second == dev) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.emplace_back(kern, dev);
    return e;
}

// Programmatic dependent launch (FPX_LINEAR_PDL, read once):
//   2 (default) the kernel may start while the preceding kernel in the stream
//     drains: prologue, TMEM allocation, the weight ring's first pass and the
//     de-quantisation of the first stages (weights + row scales) begin at
//     once; activations, C, partials and counters wait for
//     griddepcontrol.wait.  Requires that the packed weights and scales are
//     not written by a preceding kernel that triggers dependents early
//     (inference: weights are static).  Measured ~3 us per launch.
//   1 PDL with every global access after griddepcontrol.wait (hides the
//     launch latency and prologue only, ~1.2 us).
//   0 plain stream order.
uint32_t pdl_mode() {
    static const uint32_t mode = [] {
        const char* e = std::getenv("FPX_LINEAR_PDL");
        const int v = e != nullptr ? std::atoi(e) : 2;
        return static_cast<uint32_t>(v < 0 ? 0 : (v > 2 ? 2 : v));
    }();
    return mode;
}


// 3-D view of the activations: {64 k, n, k-tile} with strides {lda, 64}
// elements; box {64, NPAD, KS} -> KS consecutive SW128 [NPAD x 128 B] tiles.
cudaError_t make_act_map(const LinearLaunch& L, uint32_t npad, uint32_t ks, CUtensorMap* map) {
    auto encode = encode_fn();
    if (!encode) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {64u, L.n, L.cols_p / 64u};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(L.lda) * 2u, 128u};
    const cuuint32_t box[3] = {64u, npad, ks};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(L.act), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    return cudaSuccess;
}

// 3-D view of one packed stream (w bits/code, 512*w bytes per 64x64 tile,
// tiles row-major, prepack.cpp:190-191): {64*w u64 words, k-tile, tile-row};
// box {64*w, KS, 2} = KS consecutive tiles of the two tile-rows of a 128-row
// unit, landing as [tile-row][k-tile][512*w B] in shared memory.
cudaError_t make_stream_map(const uint8_t* base, int w, uint32_t tile_rows, uint32_t kt, uint32_t ks,
                            CUtensorMap* map) {
    auto encode = encode_fn();
    if (!encode) return cudaErrorNotSupported;
    const cuuint64_t tile_bytes = 512u * static_cast<cuuint64_t>(w);
    const cuuint64_t dims[3] = {tile_bytes / 8u, kt, tile_rows};
    const cuuint64_t strides[2] = {tile_bytes, tile_bytes * kt};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(tile_bytes / 8u), ks, 2u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    if (encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    return cudaSuccess;
}

template <int F, int NPAD, int KS_, int NG_>
cudaError_t launch_t(const LinearLaunch& L, const KParams& kp, int grid, cudaStream_t st) {
    using C = Cfg<F, NPAD, KS_, NG_>;
    auto kern = fpx_linear_kernel<F, NPAD, KS_, NG_>;
    CUtensorMap map;
    if (cudaError_t e = make_act_map(L, NPAD, C::kKS, &map)) return e;
    CUtensorMap hi_map, lo_map;
    if (cudaError_t e = make_stream_map(L.s_hi, FmtTraits<F>::kBitsHi, L.rows_p / 64, L.cols_p / 64, C::kKS, &hi_map))
        return e;
    if (cudaError_t e = make_stream_map(L.s_lo, FmtTraits<F>::kBitsLo, L.rows_p / 64, L.cols_p / 64, C::kKS, &lo_map))
        return e;
    // NPAD = 256 (single accumulator buffer): the intermittent wrong results
    // once measured at split 9 were the stage-ring parity aliasing now ruled
    // out by Cfg (kStages >= NG + kAStages).
    KParams kq = kp;
    if (C::kAccBufs == 1) grid = static_cast<int>(kq.units);
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), C::kSmemBytes)) return e;
    kern<<<grid, C::kThreads, C::kSmemBytes, st>>>(map, hi_map, lo_map, kq);
    return cudaGetLastError();
}

template <int F, int NPAD, int KS_, int G_>
cudaError_t launch_g(const LinearLaunch& L, const KParams& kp, int grid, cudaStream_t st) {
    using C = GCfg<F, NPAD, KS_, G_>;
    auto kern = fpx_linear_decode_kernel<F, NPAD, KS_, G_>;
    // K chunks are whole stages: at most ceil(KT/KS) of them
    KParams kq = kp;
    const uint32_t nst = (kp.kt + C::kKS - 1) / C::kKS;
    if (kq.split > nst) {
        kq.split = nst;
        kq.units = (kp.rows_p + kTileM - 1) / kTileM * nst;
        grid = std::min<int>(grid, static_cast<int>(kq.units));
    }
    CUtensorMap map, hi_map, lo_map;
    if (cudaError_t e = make_act_map(L, NPAD, C::kKS, &map)) return e;
    if (cudaError_t e = make_stream_map(L.s_hi, FmtTraits<F>::kBitsHi, L.rows_p / 64, L.cols_p / 64, C::kKS, &hi_map))
        return e;
    if (cudaError_t e = make_stream_map(L.s_lo, FmtTraits<F>::kBitsLo, L.rows_p / 64, L.cols_p / 64, C::kKS, &lo_map))
        return e;
    kq.pdl = std::min(pdl_mode(), L.pdl_cap);
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), C::kSmemBytes)) return e;
    return launch_pdl(kq.pdl != 0, kern, grid, C::kThreads, C::kSmemBytes, st, map, hi_map, lo_map, kq);
}

// Pipeline shape per batch width.  N <= 128: the decode kernel, KS k-tiles
// per stage, G de-quantiser groups (8192x22016: N=64 35.0 us vs 37.8 us,
// N=128 53.0 us vs 56.7 us for the single-issuer kernel at its best split;
// NPAD=128 runs 3 groups, 4 measured equal).  N > 128: the single-issuer
// kernel in 256-column chunks.  Tuning override (instantiated subset only):
// FPX_LINEAR_CFG="KS,G" at NPAD 16 / 32.
#ifndef FPX_N64_KS
#define FPX_N64_KS 2
#endif
#ifndef FPX_N64_G
#define FPX_N64_G 4
#endif
#ifndef FPX_N128_KS
#define FPX_N128_KS 2
#endif
#ifndef FPX_N128_G
#define FPX_N128_G 3
#endif
template <int F>
cudaError_t launch_f(const LinearLaunch& L, const KParams& kp, uint32_t npad, int grid, cudaStream_t st) {
    int ks = 0, ng = 0;
    if (const char* c = std::getenv("FPX_LINEAR_CFG")) std::sscanf(c, "%d,%d", &ks, &ng);
    // FPX_LINEAR_X8=1 (opt-in, measured slower -- DESIGN.md): N <= 32 on the
    // kind::f8f6f4 kernel of fpx_linear_x8.cu when the caller provided the
    // activation-split workspace.
    if (linear_x8_enabled() && L.b8 != nullptr && L.colf != nullptr && ks == 0 && npad <= 32)
        return launch_linear_x8(L, kp, npad, grid, st);
    if (npad <= 16) {
        if (ks == 1 && ng == 4) return launch_g<F, 16, 1, 4>(L, kp, grid, st);
        if (ks == 2 && ng == 3) return launch_g<F, 16, 2, 3>(L, kp, grid, st);
        if (ks == 2 && ng == 5) return launch_g<F, 16, 2, 5>(L, kp, grid, st);
        return launch_g<F, 16, 2, 4>(L, kp, grid, st);
    }
    if (npad == 32) {
        if (ks == 2 && ng == 3) return launch_g<F, 32, 2, 3>(L, kp, grid, st);
        return launch_g<F, 32, 2, 4>(L, kp, grid, st);
    }
    if (npad == 64) return launch_g<F, 64, FPX_N64_KS, FPX_N64_G>(L, kp, grid, st);
    if (npad == 128) return launch_g<F, 128, FPX_N128_KS, FPX_N128_G>(L, kp, grid, st);
    if (npad == 256) return launch_t<F, 256, 1, 2>(L, kp, grid, st);
    return cudaErrorInvalidValue;
}

}  // namespace fpxk

using namespace fpxk;

// FPX_LINEAR_X8=1 (read once): route N <= 32 to the kind::f8f6f4 kernel.
bool linear_x8_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FPX_LINEAR_X8");
        return e != nullptr && std::atoi(e) != 0;
    }();
    return on;
}

static uint32_t npad_for(uint32_t n) {
    uint32_t p = 16;
    while (p < n) p *= 2;
    return p;
}

// Bytes of fp32 split-K partials (0 for split 1).  The C-ABI lays the
// workspace out as [arrival counters at offset 0, always reserved,
// self-cleaning][partials][staged activations], so a workspace zero-filled
// once stays valid across calls of any shape.
size_t linear_workspace_bytes(uint32_t rows_p, uint32_t n, int split) {
    if (split <= 1) return 0;
    const uint32_t tiles_m = (rows_p + kTileM - 1) / kTileM;
    const size_t part = static_cast<size_t>(tiles_m) * split * npad_for(n) * kTileM * sizeof(float);
    return (part + 255) / 256 * 256;
}

// Workspace of the activation split (act_split_kernel) for N <= 32: B8
// [3 npad][cols_p] bytes, then colf [split][npad] floats.
size_t linear_split_bytes(uint32_t cols_p, uint32_t n, int split) {
    if (n == 0 || n > 32) return 0;
    const uint32_t npad = npad_for(n);
    const size_t b8 = (static_cast<size_t>(3) * npad * cols_p + 255) / 256 * 256;
    return b8 + (static_cast<size_t>(std::max(split, 1)) * npad * sizeof(float) + 255) / 256 * 256;
}

// Smallest estimated makespan in k-tile units: ceil(units / SMs) units per
// CTA, each ceil(KT/split) k-tiles plus a per-unit cost (pipeline ramp and
// the fp32 partial round trip, in weight-tile-byte equivalents).
int linear_default_split(uint32_t rows_p, uint32_t cols_p, uint32_t n, int num_sms) {
    const uint32_t tiles_m = (rows_p + kTileM - 1) / kTileM;
    const uint32_t kt = cols_p / 64;
    if (kt == 0 || tiles_m == 0) return 1;
    double best = 1e30;
    int best_s = 1;
    const int smax = static_cast<int>(std::min<uint32_t>(kt, 64));
    // Waves x (k-tiles per unit + per-unit overhead).  The overhead, ~10
    // k-tiles (pipeline drain/refill around the accumulator hand-off and the
    // epilogue), was fitted on B200 to the measured best splits of SURVEY
    // §8d's shapes (bench_configs.py --sweep-splits: 8192x22016, 22016x8192,
    // the five 70B linears, 4096^2); it makes fewer, longer units win over
    // finer load balance.  Split-K partial traffic adds a little per unit.
    auto pick = [&](double unit_pen, double part_w, bool finer_on_tie) {
        double b = 1e30;
        int bs = 1;
        for (int s = 1; s <= smax; ++s) {
            const double per_cta = std::ceil(double(tiles_m) * s / num_sms);
            const double pen = unit_pen + (s > 1 ? part_w * (2.0 * kTileM * n * 4.0) / 6144.0 : 0.0);
            const double est = per_cta * (std::ceil(double(kt) / s) + pen);
            if (est < b - 1e-9 || (finer_on_tie && est <= b + 1e-9)) b = est, bs = s;
        }
        return bs;
    };
    best_s = pick(10.0, 0.25, false);
    // Where even that split gives CTAs several units, their boundaries cost
    // less than the fit above assumes (the round-2 unit table and deferred
    // reductions): re-pick with a 2-k-tile penalty, half the partial-traffic
    // weight and ties to the finer split (N=16: 70B QKV 10240x8192 split 3 -> 5, 16.4 -> 15.9
    // us; gate/up 28672x8192 3 -> 5, 33.1 -> 32.5 us; 22016x8192 4 -> 5,
    // 26.8 -> 26.0 us).  One-unit-per-CTA shapes, the headline among them,
    // keep the first pick.
    if (std::ceil(double(tiles_m) * best_s / num_sms) > 1.0) best_s = pick(2.0, 0.125, true);
    (void)best;
    return best_s;
}

cudaError_t launch_linear(const LinearLaunch& L, cudaStream_t st) {
    const uint32_t npad = npad_for(L.n);
    const uint32_t tiles_m = (L.rows_p + kTileM - 1) / kTileM;
    KParams kp{};
    kp.s_hi = L.s_hi;
    kp.s_lo = L.s_lo;
    kp.scales = L.scales;
    kp.c = L.c;
    kp.ldc = L.ldc;
    kp.out_f16 = L.out_f16;
    kp.bias = L.bias;
    kp.act = L.act_fn;
    kp.resid = L.resid;
    kp.epi = (L.out_f16 || L.bias != nullptr || L.act_fn != 0 || L.resid != nullptr) ? 1u : 0u;
    kp.rows_p = L.rows_p;
    kp.tile_rows = L.rows_p / 64;
    kp.kt = L.cols_p / 64;
    kp.n = L.n;
    kp.split = static_cast<uint32_t>(L.split);
    kp.units = tiles_m * kp.split;
    kp.ws = L.ws;
    kp.counters = L.counters;
    if (const char* d = std::getenv("FPX_LINEAR_DBG")) kp.dbg = static_cast<uint32_t>(std::atoi(d));
    kp.trace = L.trace;
    kp.prog = L.prog;
    int grid = L.grid > 0 ? L.grid : 148;
    grid = std::min<int>(grid, static_cast<int>(kp.units));
    if (grid <= 0) return cudaSuccess;
    switch (L.fmt) {
        case kE3M2: return launch_f<kE3M2>(L, kp, npad, grid, st);
        case kE2M3: return launch_f<kE2M3>(L, kp, npad, grid, st);
        case kE2M2: return launch_f<kE2M2>(L, kp, npad, grid, st);
    }
    return cudaErrorInvalidValue;
}
