/*
 * fpx_oracle.c -- CPU restatement of the reference's FPx weight path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The shipped path (paper_2401_14112_b200/) never links or calls
 * anything under oracle/.
 *
 * Every function restates the algorithm of the reference C++ library at
 * /root/reference/proj (cited file:line) in plain C so that the parity tests
 * have an independent scalar model of:
 *   soft fp16 (half.cpp), FpxFormat/SplitScheme (format.cpp), the codec
 *   (codec.cpp), the pre-packer (prepack.cpp), Algorithm-1 SWAR dequant
 *   (simt.cpp) and the tile/slice/chunk/panel GEMM order (gemm.cpp).
 *
 * Parity pinning: the restatement is checked byte-for-byte against the
 * reference itself (oracle/_ref/libfpxref.so built from the unmodified
 * reference sources by oracle/Makefile) and against the committed golden
 * vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Status codes: 0 = ok, otherwise 1 + fpx::ErrorCode (error.hpp:10-24).
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction, matching the
 * reference build which has no FMA in its x86-64 baseline ISA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID_FORMAT 1
#define ORC_INVALID_CODE 2
#define ORC_INVALID_VALUE 3
#define ORC_SCALE_OVERFLOW 4
#define ORC_SHAPE_MISMATCH 5
#define ORC_RAGGED_INPUT 6
#define ORC_UNSUPPORTED_SPLIT 7

typedef union { float f; uint32_t u; } f32bits;

/* ---------------------------------------------------------------- fp16 */

/* half.cpp:7-28 -- exact binary16 -> binary32 (subnormals renormalised,
 * inf/nan payload carried). */
float orc_half_to_float(uint16_t h) {
    f32bits r;
    uint32_t s = (uint32_t)(h >> 15) << 31;
    uint32_t ex = (h >> 10) & 0x1fu;
    uint32_t mant = h & 0x3ffu;
    if (ex == 31u) {
        r.u = s | 0x7f800000u | (mant << 13);
    } else if (ex != 0u) {
        r.u = s | ((ex + 112u) << 23) | (mant << 13);
    } else if (mant == 0u) {
        r.u = s;
    } else {
        /* mant * 2^-24 is exact in fp32 */
        r.f = ldexpf((float)mant, -24);
        r.u |= s;
    }
    return r.f;
}

/* half.cpp:30-66 -- binary32 -> binary16, round-to-nearest-even, gradual
 * underflow, overflow to inf, NaN keeps sign + top payload with quiet bit. */
uint16_t orc_float_to_half(float f) {
    f32bits in;
    in.f = f;
    uint16_t s = (uint16_t)((in.u >> 16) & 0x8000u);
    uint32_t a = in.u & 0x7fffffffu;
    if (a >= 0x7f800000u) {
        uint32_t payload = a & 0x7fffffu;
        return payload ? (uint16_t)(s | 0x7e00u | (payload >> 13)) : (uint16_t)(s | 0x7c00u);
    }
    int e16 = (int)(a >> 23) - 112;          /* biased fp16 exponent */
    uint32_t sig = (a & 0x7fffffu) | 0x800000u;
    if (e16 >= 31) return (uint16_t)(s | 0x7c00u);
    int drop;                                 /* low significand bits dropped */
    uint32_t base;
    if (e16 >= 1) {
        drop = 13;
        base = ((uint32_t)e16 << 10) | ((sig >> 13) & 0x3ffu);
    } else {
        if (e16 < -10) return s;              /* below half of min subnormal */
        drop = 14 - e16;                      /* 14..24 */
        base = sig >> drop;
    }
    uint32_t rem = sig & ((1u << drop) - 1u);
    uint32_t halfway = 1u << (drop - 1);
    /* carry out of the mantissa rolls into the exponent (and to inf) */
    if (rem > halfway || (rem == halfway && (base & 1u))) base += 1u;
    return (uint16_t)(s | base);
}

/* half.cpp:68-70 -- fp16 multiply: exact fp32 product, one RNE rounding. */
uint16_t orc_half_mul(uint16_t a, uint16_t b) {
    return orc_float_to_half(orc_half_to_float(a) * orc_half_to_float(b));
}

/* ---------------------------------------------------------- FpxFormat */

/* format.cpp:30-39 -- E in 1..5, M in 0..6, 3..8 total bits. */
int orc_format_ok(int e, int m) {
    int t = 1 + e + m;
    return (e >= 1 && e <= 5 && m >= 0 && m <= 6 && t >= 3 && t <= 8) ? 1 : 0;
}

static int fmt_bias(int e) { return (1 << (e - 1)) - 1; }  /* format.hpp:21 */

/* format.cpp:8-12 -- (2 - 2^-M) * 2^(emax - bias), emax = all-ones field. */
float orc_max_rep(int e, int m) {
    double frac = 2.0 - ldexp(1.0, -m);
    return (float)ldexp(frac, ((1 << e) - 1) - fmt_bias(e));
}

/* format.cpp:59-69 -- preset split by total width (high bits first). */
int orc_split_for(int e, int m, int* widths) {
    static const int table[9][3] = {{0}, {0}, {0}, {2, 1}, {4}, {4, 1}, {2, 4}, {4, 2, 1}, {4, 4}};
    static const int count[9] = {0, 0, 0, 2, 1, 2, 2, 3, 2};
    int t = 1 + e + m;
    if (t < 3 || t > 8) return 0;
    for (int i = 0; i < count[t]; ++i) widths[i] = table[t][i];
    return count[t];
}

/* -------------------------------------------------------------- codec */

/* codec.cpp:49-68 -- exact value of a code. */
float orc_decode(uint32_t code, int e, int m) {
    int bias = fmt_bias(e);
    uint32_t sgn = (code >> (e + m)) & 1u;
    uint32_t ef = (code >> m) & ((1u << e) - 1u);
    uint32_t mf = code & ((1u << m) - 1u);
    double v = (ef == 0u) ? ldexp((double)mf, 1 - bias - m)
                          : ldexp((double)((1u << m) | mf), (int)ef - bias - m);
    float f = (float)v;
    return sgn ? -f : f;
}

/* codec.cpp:70-103 -- RNE encode on the 2^(e-M) grid, saturating. NaN is
 * rejected by the caller (quantize checks rows first). */
uint32_t orc_encode(double v, int e, int m) {
    int bias = fmt_bias(e);
    uint32_t smask = 1u << (e + m);
    uint32_t sign = signbit(v) ? smask : 0u;
    double a = fabs(v);
    if (a > (double)orc_max_rep(e, m)) return sign | (smask - 1u);
    int emin = 1 - bias;
    int ex = (a >= ldexp(1.0, emin)) ? ilogb(a) : emin;
    uint32_t k = (uint32_t)nearbyint(ldexp(a, m - ex));   /* ties-to-even */
    uint32_t unit = 1u << m;
    if (k == 2u * unit) { k = unit; ++ex; }               /* binade carry */
    if (k < unit) return sign | k;                        /* subnormal */
    return sign | ((uint32_t)(ex + bias) << m) | (k - unit);
}

/* codec.cpp:195-199 -- fp16(scale * 2^(15 - bias)). */
uint16_t orc_effective_scale(uint16_t s, int e, int m) {
    (void)m;
    double v = (double)orc_half_to_float(s) * ldexp(1.0, 15 - fmt_bias(e));
    return orc_float_to_half((float)v);
}

static uint32_t pad64(uint32_t n) { return (n + 63u) & ~63u; }

/* codec.cpp:105-177 -- row-wise quantization of an fp32 row-major matrix.
 * codes: pad64(rows) x pad64(cols) bytes (zero padded); scales: pad64(rows).
 * On failure returns the status of the FIRST failing row (row order) and
 * writes that row index to *fail_row. */
int orc_quantize(const float* w, uint32_t rows, uint32_t cols, int e, int m,
                 uint8_t* codes, uint16_t* scales, int64_t* fail_row) {
    if (!orc_format_ok(e, m)) return ORC_INVALID_FORMAT;
    if (rows == 0 || cols == 0) return ORC_SHAPE_MISMATCH;
    uint32_t rp = pad64(rows), cp = pad64(cols);
    memset(codes, 0, (size_t)rp * cp);
    for (uint32_t r = 0; r < rp; ++r) scales[r] = 0x3c00u;
    double maxrep = (double)orc_max_rep(e, m);
    int rebias = 15 - fmt_bias(e);
    if (fail_row) *fail_row = -1;
    for (uint32_t r = 0; r < rows; ++r) {
        const float* row = w + (size_t)r * cols;
        double amax = 0.0;
        int nan = 0;
        for (uint32_t c = 0; c < cols; ++c) {
            double a = fabs((double)row[c]);
            if (isnan(a)) nan = 1;
            if (a > amax) amax = a;
        }
        int st = ORC_OK;
        uint16_t s16 = 0;
        if (nan) {
            st = ORC_INVALID_VALUE;
        } else if (amax != 0.0) {
            s16 = orc_float_to_half((float)(amax / maxrep));
            if ((s16 & 0x7c00u) == 0x7c00u) {
                st = ORC_SCALE_OVERFLOW;
            } else {
                if ((s16 & 0x7fffu) == 0u) s16 = (uint16_t)((s16 & 0x8000u) | 1u);
                double sv = (double)orc_half_to_float(s16);
                uint16_t eff = orc_float_to_half((float)(sv * ldexp(1.0, rebias)));
                if ((eff & 0x7c00u) == 0x7c00u) st = ORC_SCALE_OVERFLOW;
            }
        } else {
            continue;  /* all-zero row: scale 1.0, codes 0 */
        }
        if (st != ORC_OK) {
            if (fail_row) *fail_row = (int64_t)r;
            return st;
        }
        scales[r] = s16;
        double sv = (double)orc_half_to_float(s16);
        uint8_t* out = codes + (size_t)r * cp;
        for (uint32_t c = 0; c < cols; ++c)
            out[c] = (uint8_t)orc_encode((double)row[c] / sv, e, m);
    }
    return ORC_OK;
}

/* codec.cpp:179-193 -- the scalar de-quantization oracle:
 * fp16(decode(code)) * raw row scale, fp16 RNE. Row-major fp16 out. */
void orc_dequantize(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p,
                    uint32_t cols_p, int e, int m, uint16_t* out) {
    uint16_t lut[256];
    for (uint32_t c = 0; c < (1u << (1 + e + m)); ++c) lut[c] = orc_float_to_half(orc_decode(c, e, m));
    for (uint32_t r = 0; r < rows_p; ++r)
        for (uint32_t c = 0; c < cols_p; ++c) {
            size_t i = (size_t)r * cols_p + c;
            out[i] = orc_half_mul(lut[codes[i]], scales[r]);
        }
}

/* ------------------------------------------------------------ prepack */

/* prepack.cpp:17 -- byte lane receiving code j of a group of four. */
static const uint32_t kLaneOfCode[4] = {1u, 3u, 0u, 2u};

/* prepack.cpp:29-38 -- (slice, chunk, thread, pair, lane) -> tile (row, col). */
void orc_fragment_coords(uint32_t s, uint32_t c, uint32_t t, uint32_t p, uint32_t l,
                         uint32_t* row, uint32_t* col) {
    *row = 16u * c + 8u * (p & 1u) + t / 4u;
    *col = 16u * s + 8u * (p >> 1) + 2u * (t % 4u) + l;
}

/* Consumption-order index k (0..127) of thread t -> tile (row, col).
 * prepack.cpp:40-58: order is slice, chunk, pair, lane. */
static void code_position(uint32_t t, uint32_t k, uint32_t* row, uint32_t* col) {
    orc_fragment_coords(k >> 5, (k >> 3) & 3u, t, (k >> 1) & 3u, k & 1u, row, col);
}

/* Bit position of segment `seg` of code k inside its word, per
 * prepack.cpp:71-86: group g of a width-w word sits at bits
 * [8*lane + 8 - w*(g+1), 8*lane + 8 - w*g) of the word. */
static void segment_slot(uint32_t k, int w, uint32_t* word, uint32_t* shift) {
    uint32_t it = k >> 2, per_word = 8u / (uint32_t)w;
    *word = it / per_word;
    *shift = 8u * kLaneOfCode[k & 3u] + 8u - (uint32_t)w * (it % per_word + 1u);
}

/* prepack.cpp:153-209 -- pack a padded code grid. streams[seg] must hold
 * tiles * 512 * widths[seg] bytes; tile t = tr * (cols_p/64) + tc;
 * word j of thread i lands at byte offset (j*32 + i)*4 of the tile block,
 * little-endian (prepack.cpp:115-134). */
int orc_pack(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
             int e, int m, const int* widths, int nseg, uint8_t* const* streams) {
    if (rows_p == 0 || cols_p == 0 || (rows_p & 63u) || (cols_p & 63u)) return ORC_SHAPE_MISMATCH;
    int tot = 0;
    for (int i = 0; i < nseg; ++i) tot += widths[i];
    if (tot != 1 + e + m) return ORC_UNSUPPORTED_SPLIT;
    for (uint32_t r = 0; r < rows_p; ++r)
        if ((orc_effective_scale(scales[r], e, m) & 0x7c00u) == 0x7c00u) return ORC_SCALE_OVERFLOW;
    uint32_t gc = cols_p / 64u, ntiles = (rows_p / 64u) * gc;
    for (uint32_t tile = 0; tile < ntiles; ++tile) {
        uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
        for (int sg = 0; sg < nseg; ++sg)
            memset(streams[sg] + (size_t)tile * 512u * widths[sg], 0, 512u * (size_t)widths[sg]);
        for (uint32_t t = 0; t < 32u; ++t)
            for (uint32_t k = 0; k < 128u; ++k) {
                uint32_t rr, cc;
                code_position(t, k, &rr, &cc);
                uint32_t code = codes[(size_t)(r0 + rr) * cols_p + c0 + cc];
                int low = 1 + e + m;
                for (int sg = 0; sg < nseg; ++sg) {
                    int w = widths[sg];
                    low -= w;
                    uint32_t val = (code >> low) & ((1u << w) - 1u);
                    uint32_t word, sh;
                    segment_slot(k, w, &word, &sh);
                    size_t byte = (size_t)tile * 512u * w + ((size_t)word * 32u + t) * 4u;
                    uint32_t cur;
                    memcpy(&cur, streams[sg] + byte, 4);   /* host is little-endian */
                    cur |= val << sh;
                    memcpy(streams[sg] + byte, &cur, 4);
                }
            }
    }
    return ORC_OK;
}

/* prepack.cpp:211-260 -- exact inverse of orc_pack. */
int orc_unpack(uint8_t const* const* streams, uint32_t rows_p, uint32_t cols_p, int e, int m,
               const int* widths, int nseg, uint8_t* codes) {
    if (rows_p == 0 || cols_p == 0 || (rows_p & 63u) || (cols_p & 63u)) return ORC_SHAPE_MISMATCH;
    uint32_t gc = cols_p / 64u, ntiles = (rows_p / 64u) * gc;
    for (uint32_t tile = 0; tile < ntiles; ++tile) {
        uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
        for (uint32_t t = 0; t < 32u; ++t)
            for (uint32_t k = 0; k < 128u; ++k) {
                uint32_t code = 0;
                int low = 1 + e + m;
                for (int sg = 0; sg < nseg; ++sg) {
                    int w = widths[sg];
                    low -= w;
                    uint32_t word, sh, cur;
                    segment_slot(k, w, &word, &sh);
                    memcpy(&cur, streams[sg] + (size_t)tile * 512u * w + ((size_t)word * 32u + t) * 4u, 4);
                    code |= ((cur >> sh) & ((1u << w) - 1u)) << low;
                }
                uint32_t rr, cc;
                code_position(t, k, &rr, &cc);
                codes[(size_t)(r0 + rr) * cols_p + c0 + cc] = (uint8_t)code;
            }
    }
    return ORC_OK;
}

/* ------------------------------------------------- Algorithm 1 (SWAR) */

/* simt.hpp:26-45 + simt.cpp:7-44 -- one thread's slice: 2 words of 2-bit
 * segments, 4 words of 4-bit segments, 8 effective scales -> 32 fp16 in
 * consumption order. Only meaningful for e3m2 with the [2,4] split
 * (simt.cpp:51-53). */
void orc_swar_thread_slice(const uint32_t f1in[2], const uint32_t f2in[4], const uint16_t sc[8],
                           uint16_t out[32]) {
    uint32_t f1[2] = {f1in[0], f1in[1]}, f2[4] = {f2in[0], f2in[1], f2in[2], f2in[3]};
    int i1 = 0, i2 = 0;
    for (int i = 0; i < 8; ++i) {
        uint32_t x = (f1[i1] & 0xc0c0c0c0u) | ((f2[i2] & 0xf0f0f0f0u) >> 2);
        if ((i & 3) == 3) ++i1; else f1[i1] <<= 2;
        if (i & 1) ++i2; else f2[i2] <<= 4;
        uint32_t v = (x & 0x80808080u) | ((x >> 2) & 0x1f1f1f1fu);
        uint32_t r1 = v & 0x9f009f00u, r2 = (v & 0x009f009fu) << 8;
        uint16_t s1 = sc[(i / 2) * 2], s2 = sc[(i / 2) * 2 + 1];
        out[4 * i + 0] = orc_half_mul((uint16_t)(r1 & 0xffffu), s1);
        out[4 * i + 1] = orc_half_mul((uint16_t)(r1 >> 16), s1);
        out[4 * i + 2] = orc_half_mul((uint16_t)(r2 & 0xffffu), s2);
        out[4 * i + 3] = orc_half_mul((uint16_t)(r2 >> 16), s2);
    }
}

/* gemm.cpp:67-85 driven over a whole packed matrix: de-quantize every tile
 * through the SWAR path (e3m2/[2,4]) and scatter to a row-major fp16 grid.
 * This is the packed-path counterpart of orc_dequantize; the two must agree
 * bit-for-bit (SPEC acceptance #1). */
void orc_dequant_packed_e3m2(const uint8_t* s2, const uint8_t* s4, const uint16_t* scales,
                             uint32_t rows_p, uint32_t cols_p, uint16_t* out) {
    uint32_t gc = cols_p / 64u, ntiles = (rows_p / 64u) * gc;
    for (uint32_t tile = 0; tile < ntiles; ++tile) {
        uint32_t tr = tile / gc, tc = tile % gc;
        for (uint32_t sl = 0; sl < 4u; ++sl)
            for (uint32_t t = 0; t < 32u; ++t) {
                uint32_t f1[2], f2[4];
                uint16_t sc[8], o[32];
                for (int j = 0; j < 2; ++j)
                    memcpy(&f1[j], s2 + (size_t)tile * 1024u + (((2u * sl + j) * 32u + t) * 4u), 4);
                for (int j = 0; j < 4; ++j)
                    memcpy(&f2[j], s4 + (size_t)tile * 2048u + (((4u * sl + j) * 32u + t) * 4u), 4);
                for (uint32_t c = 0; c < 4u; ++c) {
                    sc[2 * c] = orc_effective_scale(scales[tr * 64u + 16u * c + t / 4u], 3, 2);
                    sc[2 * c + 1] = orc_effective_scale(scales[tr * 64u + 16u * c + 8u + t / 4u], 3, 2);
                }
                orc_swar_thread_slice(f1, f2, sc, o);
                for (uint32_t k = 0; k < 32u; ++k) {
                    uint32_t rr, cc;
                    code_position(t, sl * 32u + k, &rr, &cc);
                    out[(size_t)(tr * 64u + rr) * cols_p + tc * 64u + cc] = o[k];
                }
            }
    }
}

/* --------------------------------------------------------------- GEMM */

/* gemm.cpp:221-252 with mma_emulate (gemm.cpp:154-168): C(fp32 col-major,
 * rows_p x n) = dequant(W) x B, B fp16 col-major (b_rows x n) zero-padded
 * beyond b_rows / n (gemm.cpp:15-18). Order per output element: k-tiles,
 * slices, k inside the 16-wide mma, each product fp32 then fp32 add. */
int orc_gemm_reference(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p,
                       uint32_t cols_p, uint32_t orig_cols, int e, int m, const uint16_t* b,
                       uint32_t b_rows, uint32_t n, float* c) {
    if (b_rows != cols_p && b_rows != orig_cols) return ORC_SHAPE_MISMATCH;
    uint16_t* w = (uint16_t*)malloc((size_t)rows_p * cols_p * 2u);
    float* bf = (float*)malloc((size_t)cols_p * (n ? n : 1) * sizeof(float));
    if (!w || !bf) { free(w); free(bf); return ORC_INVALID_VALUE; }
    orc_dequantize(codes, scales, rows_p, cols_p, e, m, w);
    for (uint32_t j = 0; j < n; ++j)
        for (uint32_t k = 0; k < cols_p; ++k)
            bf[(size_t)j * cols_p + k] = k < b_rows ? orc_half_to_float(b[(size_t)j * b_rows + k]) : 0.0f;
    memset(c, 0, (size_t)rows_p * n * sizeof(float));
    for (uint32_t r = 0; r < rows_p; ++r) {
        float wr[64];
        for (uint32_t k0 = 0; k0 < cols_p; k0 += 16u) {
            for (uint32_t k = 0; k < 16u; ++k) wr[k] = orc_half_to_float(w[(size_t)r * cols_p + k0 + k]);
            for (uint32_t j = 0; j < n; ++j) {
                float acc = c[(size_t)j * rows_p + r];
                const float* bj = bf + (size_t)j * cols_p + k0;
                for (uint32_t k = 0; k < 16u; ++k) acc += wr[k] * bj[k];
                c[(size_t)j * rows_p + r] = acc;
            }
        }
    }
    free(w);
    free(bf);
    return ORC_OK;
}

/* ------------------------------------------------------------- helpers */

/* FNV-1a 64 over a byte buffer, chainable (for golden pins). */
uint64_t orc_fnv1a64(const uint8_t* p, size_t n, uint64_t h) {
    if (h == 0) h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) { h ^= p[i]; h *= 0x100000001b3ull; }
    return h;
}
