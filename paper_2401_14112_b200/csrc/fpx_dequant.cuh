// fpx_dequant.cuh -- register-level de-quantisation of the packed FPx
// streams into fp16 mma A-fragments.  Shared by the fused linear kernel
// (fpx_linear.cu) and the bit-exact verification kernel (fpx_codec.cu), so
// the dequant bits the GEMM consumes are exactly the bits the parity tests
// compare against the reference's dequantize_reference (codec.cpp:179-193).
//
// Packed layout (reference prepack.cpp:29-134): per 64x64
// tile, per segment width w, thread t's word j lives at byte (j*32+t)*4 of
// the tile's 512*w-byte block; code k of thread t sits in iteration k/4,
// byte lane {1,3,0,2}[k%4], group (k/4) % (8/w) of word (k/4)/(8/w), at bits
// [8*lane+8-w*(g+1), 8*lane+8-w*g).
//
// A warp of the linear kernel owns 32 rows of a 64-row tile: half h (0/1)
// covers chunks 2h and 2h+1 of every slice, i.e. iterations i = 4h+j,
// j = 0..3, of the reference's 8-iteration loop (simt.cpp:21-42).  For one
// slice s the thread needs:
//   [2,4] split (FP6 e3m2/e2m3): 2-bit word 2s+h, 4-bit words 4s+2h, 4s+2h+1
//   [4,1] split (FP5 e2m2)     : 4-bit words 4s+2h, 4s+2h+1, 1-bit word s
// and produces, per j, R1 (pair rows 16c+t/4) and R2 (rows 16c+8+t/4),
// c = 2h + j/2, each an f16x2 register in mma A-fragment order.
//
// Two register paths, both bit-exact with the reference oracle:
//  * kHwCvt (default, B200-native): pair the byte lanes of each packed word
//    with one PRMT ({1,3} -> R1, {0,2} -> R2, matching the reference's lane
//    permutation prepack.cpp:17), stitch the four codes of iteration j into
//    the low 6 bits of each byte lane (one LOP3 + shifts), convert with the sm_100a hardware
//    FP6 -> f16x2 unpack (cvt.rn.f16x2.e3m2x2 / e2m3x2, SASS F2FP ... UNPACK_B,
//    which ignores bits 7:6 of each byte) and multiply by the RAW fp16 row
//    scale.  cvt yields fp16(decode(code)) exactly, so the product is the
//    oracle's half_mul(float_to_half(decode), scale) by definition.  FP5
//    e2m2 codes become e2m3 codes by appending a zero mantissa bit (same
//    bias, exactly representable).  ALU work ~2.5x below the SWAR path and
//    the converts issue outside the ALU pipe.
//  * kSwar: the paper's Algorithm 1 (simt.hpp:26-45, simt.cpp:13-44) --
//    stitch, bias-deferred 4-way cast into fp16 top bits, multiply by the
//    effective scale fp16(s * 2^(15-bias)) (codec.cpp:195-199).
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "ptx_sm100.cuh"

namespace fpxk {

enum FmtId : int { kE3M2 = 0, kE2M3 = 1, kE2M2 = 2 };
enum DqPath : int { kHwCvt = 0, kSwar = 1 };

template <int F>
struct FmtTraits;

// e3m2: S|EEE|MM, bias 3.
template <>
struct FmtTraits<kE3M2> {
    static constexpr int kBitsHi = 2, kBitsLo = 4;  // stream widths (hi first)
    static constexpr int kRebias = 12;              // 15 - bias (SWAR path)
};
// e2m3: S|EE|MMM, bias 1.
template <>
struct FmtTraits<kE2M3> {
    static constexpr int kBitsHi = 2, kBitsLo = 4;
    static constexpr int kRebias = 14;
};
// e2m2: S|EE|MM, bias 1, split [4,1].
template <>
struct FmtTraits<kE2M2> {
    static constexpr int kBitsHi = 4, kBitsLo = 1;
    static constexpr int kRebias = 14;
};

// (mask_src & kMask) | (other & ~kMask) as ONE LOP3 (LUT 0xE2 over
// (a, mask, c)); left to itself nvcc splits it into two.
template <uint32_t kMask>
FPX_DEV uint32_t lop3_sel(uint32_t mask_src, uint32_t other) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(d) : "r"(mask_src), "n"(kMask), "r"(other));
    return d;
}

FPX_DEV uint32_t prmt(uint32_t a, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
    return d;
}

// Hardware FP6x2 -> f16x2 (exact).  F = kE3M2 uses e3m2, else e2m3.
template <int F>
FPX_DEV void cvt_pairs(uint32_t paired, uint32_t& lo, uint32_t& hi) {
    if constexpr (F == kE3M2) {
        asm("{\n\t.reg .b16 l, h;\n\t"
            "mov.b32 {l, h}, %2;\n\t"
            "cvt.rn.f16x2.e3m2x2 %0, l;\n\t"
            "cvt.rn.f16x2.e3m2x2 %1, h;\n\t}"
            : "=r"(lo), "=r"(hi)
            : "r"(paired));
    } else {
        asm("{\n\t.reg .b16 l, h;\n\t"
            "mov.b32 {l, h}, %2;\n\t"
            "cvt.rn.f16x2.e2m3x2 %0, l;\n\t"
            "cvt.rn.f16x2.e2m3x2 %1, h;\n\t}"
            : "=r"(lo), "=r"(hi)
            : "r"(paired));
    }
}

// ------------------------------------------------------------ kHwCvt path
// Right shift on the FMA pipe (IMAD.HI) instead of the ALU pipe (SHF).  The
// ALU pipe (LOP3/SHF/PRMT/F2FP, 16 lanes/clk/SMSP on B200) is what bounds
// the de-quantiser; HMUL2/IMAD issue to the FMA pipe.  Measured by
// tools/micro/pipe_bench.cu.
#ifndef FPX_SHR_ON_FMA
#define FPX_SHR_ON_FMA 0
#endif
template <int K>
FPX_DEV uint32_t shr(uint32_t x) {
#if FPX_SHR_ON_FMA
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(1u << (32 - K)));
    return d;
#else
    return x >> K;
#endif
}

FPX_DEV uint32_t prmt2(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// Codes of iteration j in bits [5:0] of each byte lane (bits 7:6 junk,
// ignored by the converts and by tcgen05.mma kind::f8f6f4), in the byte-lane
// order of the inputs.  Every operation is byte-local, so permuting the
// input words' bytes permutes the outputs' bytes the same way.
template <int F>
FPX_DEV void codes_low6_raw(uint32_t pa, uint32_t pb, uint32_t pc, int h, uint32_t (&c)[4]) {
    if constexpr (FmtTraits<F>::kBitsHi == 2) {
        // 2-bit group j (bits 7-2j..6-2j) -> bits 5:4; 4-bit group j%2 -> bits 3:0
        c[0] = lop3_sel<0x30303030u>(shr<2>(pa), shr<4>(pb));
        c[1] = lop3_sel<0x30303030u>(pa, pb);
        c[2] = lop3_sel<0x30303030u>(pa << 2, shr<4>(pc));
        c[3] = lop3_sel<0x30303030u>(pa << 4, pc);
    } else {
        // e2m2 [4,1] -> e2m3 code (c << 1): 4-bit group j%2 (S E1 E0 M1) -> bits 5:2,
        // 1-bit group g = 4h+j (bit 7-g, M0) -> bit 1, bit 0 = 0 (bits 7:6
        // are ignored by the conversion, as on the [2,4] path).
        // * The half h's four 1-bit groups are brought to bits 7:4 of every
        //   byte (x 16 for h = 1, an IMAD; bits 3:0 then hold the byte
        //   below's groups and are never selected).
        // * They are split into even / odd bit positions, so that whatever
        //   lands next to a selected bit is zero, and each split is shifted
        //   once for two code words: x (bits 7, 5 -> 3, 1) and y (bits 6, 4
        //   -> 1 and bit 7 of the byte below; a rotate, so byte 0 gets byte
        //   3's).
        // * One select LOP3 per code word, plus one shift for words 0 and 3,
        //   whose nibble and 1-bit group are merged before moving together.
        const uint32_t pch = pc * (h ? 16u : 1u);
        const uint32_t x = (pch & 0xaaaaaaaau) >> 4;
        const uint32_t y = __funnelshift_r(pch & 0x55555555u, pch & 0x55555555u, 5);
        c[0] = shr<2>(lop3_sel<0xf0f0f0f0u>(pa, x));
        c[1] = lop3_sel<0x3c3c3c3cu>(pa << 2, y);
        c[2] = lop3_sel<0x3c3c3c3cu>(shr<2>(pb), x);
        const uint32_t t3 = lop3_sel<0x0f0f0f0fu>(pb, y);
        c[3] = __funnelshift_l(t3, t3, 2);
    }
}

// The fp16 path: byte lanes permuted {1,3,0,2} first so that the low half of
// c[j] feeds R1 (codes 4j+0, 4j+1) and the high half R2 (4j+2, 4j+3); the
// permutation is applied once to each of the three packed words (3 PRMT per
// slice rather than one per iteration).
template <int F>
FPX_DEV void codes_low6(uint32_t wa, uint32_t wb, uint32_t wc, int h, uint32_t (&c)[4]) {
    codes_low6_raw<F>(prmt(wa, 0x2031u), prmt(wb, 0x2031u), prmt(wc, 0x2031u), h, c);
}

// ------------------------------------------------------------ 8-bit A path
// The A operand of tcgen05.mma kind::f8f6f4 straight from the packed words:
// FP6 codes (FP5 e2m2 as e2m3, see codes_low6_raw) in 8-bit containers, no
// conversion at all.  In the raw byte-lane order, c[j] holds (lane 1, lane 3)
// = row 16c + t/4 and (lane 0, lane 2) = row 16c + 8 + t/4, columns
// 8(j%2) + 2(t%4) + {0, 1} of the slice (c = 2h + j/2; prepack.cpp:17, 29-58).
// One PRMT per output gathers the four codes of one row:
//   x[lc][hf] = row 16(2h+lc) + 8hf + t/4, slice columns
//               {2j, 2j+1, 8+2j, 9+2j} (j = t % 4) in bytes 0..3.
// 4 LOP3 + 5 shifts + 4 PRMT per 16 weights, vs 3 PRMT + 4 LOP3 + 5 shifts +
// 8 F2FP on the fp16 path.  The TMEM cell (row, column 4s + t%4) of a k-tile
// then holds logical k = 16s + 4(t%4) + b <- actual slice column
// {2j, 2j+1, 8+2j, 9+2j}[b]; the activations' e4m3 parts are laid out in
// the same logical K order (act_split_kernel), so the products pair up.
template <int F>
FPX_DEV void codes8_slice_half(uint32_t wa, uint32_t wb, uint32_t wc, int h, uint32_t (&x)[2][2]) {
    uint32_t c[4];
    codes_low6_raw<F>(wa, wb, wc, h, c);
    x[0][0] = prmt2(c[0], c[1], 0x7531u);
    x[0][1] = prmt2(c[0], c[1], 0x6420u);
    x[1][0] = prmt2(c[2], c[3], 0x7531u);
    x[1][1] = prmt2(c[2], c[3], 0x6420u);
}

// ------------------------------------------------------------ kSwar path
// Reference stitch_step with the register advance of simt.cpp:25-32 folded
// into constant shifts: four codes left-aligned at bit 7 of each byte.
template <int F>
FPX_DEV uint32_t stitch_hi(uint32_t wa, uint32_t wb, uint32_t wc, int j, int h) {
    if constexpr (FmtTraits<F>::kBitsHi == 2) {
        (void)h;
        const uint32_t f1 = wa << (2 * j);
        const uint32_t f2 = (j < 2 ? wb : wc) << (4 * (j & 1));
        return (f1 & 0xc0c0c0c0u) | ((f2 & 0xf0f0f0f0u) >> 2);
    } else {
        const uint32_t hi = ((j < 2 ? wa : wb) << (4 * (j & 1))) & 0xf0f0f0f0u;
        const int g = 4 * h + j;
        return hi | (((wc << g) & 0x80808080u) >> 4);
    }
}

// Bias-deferred cast (Eq. 3): R1 = lanes {1 lo, 3 hi}, R2 = lanes {0, 2}.
template <int F>
FPX_DEV void swar_to_half2(uint32_t x, uint32_t& r1, uint32_t& r2) {
    if constexpr (F == kE3M2) {
        // reference dequant4 (simt.hpp:40-45)
        const uint32_t v = (x & 0x80808080u) | ((x >> 2) & 0x1f1f1f1fu);
        r1 = v & 0x9f009f00u;
        r2 = (v & 0x009f009fu) << 8;
    } else if constexpr (F == kE2M3) {
        r1 = (x & 0x80008000u) | ((x >> 3) & 0x0f800f80u);
        const uint32_t y = x << 8;
        r2 = (y & 0x80008000u) | ((y >> 3) & 0x0f800f80u);
    } else {
        r1 = (x & 0x80008000u) | ((x >> 3) & 0x0f000f00u);
        const uint32_t y = x << 8;
        r2 = (y & 0x80008000u) | ((y >> 3) & 0x0f000f00u);
    }
}

// One slice of one half-warp-tile: 4 iterations -> {R1, R2} per j, by
// default multiplied (fp16 RNE) by the row scales.  sc[lc][0] = scale (both halves)
// of row 16(2h+lc)+t/4, sc[lc][1] of +8: RAW scales for kHwCvt, effective
// scales for kSwar (see row_scale_for).
//
// kScale = false (kHwCvt only): skip the multiply and return fp16(decode)
// exactly; the caller applies the row scale later in fp32 (the linear
// kernel's epilogue, for rows whose scales make fp16(decode * s) a normal,
// finite number -- see fpx_linear.cu).
template <int F, int P = kHwCvt, bool kScale = true>
FPX_DEV void dequant_slice_half(uint32_t wa, uint32_t wb, uint32_t wc, int h, const uint32_t (&sc)[2][2],
                                uint32_t (&r1)[4], uint32_t (&r2)[4]) {
    if constexpr (P == kHwCvt) {
        uint32_t c[4];
        codes_low6<F>(wa, wb, wc, h, c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t a, b;
            cvt_pairs<F == kE3M2 ? kE3M2 : kE2M3>(c[j], a, b);
            if constexpr (kScale) {
                r1[j] = hmul2_rn(a, sc[j >> 1][0]);
                r2[j] = hmul2_rn(b, sc[j >> 1][1]);
            } else {
                r1[j] = a;
                r2[j] = b;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t a, b;
            swar_to_half2<F>(stitch_hi<F>(wa, wb, wc, j, h), a, b);
            r1[j] = hmul2_rn(a, sc[j >> 1][0]);
            r2[j] = hmul2_rn(b, sc[j >> 1][1]);
        }
    }
}

// Byte offsets (within a tile's stream block) of the three words one thread
// needs for slice s, half h: {wa, wb, wc} per the table at the top.
template <int F>
FPX_DEV void slice_word_offsets(int s, int h, uint32_t t, uint32_t& oa, uint32_t& ob, uint32_t& oc, bool& a_in_hi,
                                bool& b_in_hi, bool& c_in_hi) {
    if constexpr (FmtTraits<F>::kBitsHi == 2) {
        oa = ((2 * s + h) * 32 + t) * 4;          // 2-bit stream
        ob = ((4 * s + 2 * h) * 32 + t) * 4;      // 4-bit stream
        oc = ((4 * s + 2 * h + 1) * 32 + t) * 4;  // 4-bit stream
        a_in_hi = true, b_in_hi = false, c_in_hi = false;
    } else {
        oa = ((4 * s + 2 * h) * 32 + t) * 4;      // 4-bit stream (hi)
        ob = ((4 * s + 2 * h + 1) * 32 + t) * 4;  // 4-bit stream (hi)
        oc = (s * 32 + t) * 4;                    // 1-bit stream (lo)
        a_in_hi = true, b_in_hi = true, c_in_hi = false;
    }
}

// fp16 bits -> fp16 bits, fp16(x * 2^k) computed exactly in fp32 then RNE
// (codec.cpp:195-199 effective_scale).
FPX_DEV uint16_t effective_scale_dev(uint16_t s, int rebias) {
    const float v = __half2float(__ushort_as_half(s)) * __int_as_float((127 + rebias) << 23);
    return __half_as_ushort(__float2half_rn(v));
}

FPX_DEV uint32_t bcast_half2(uint16_t h) { return static_cast<uint32_t>(h) * 0x10001u; }

// The per-row multiplier a path expects, broadcast to both halves.
template <int F, int P = kHwCvt>
FPX_DEV uint32_t row_scale_for(uint16_t raw) {
    if constexpr (P == kHwCvt) return bcast_half2(raw);
    else return bcast_half2(effective_scale_dev(raw, FmtTraits<F>::kRebias));
}

}  // namespace fpxk
