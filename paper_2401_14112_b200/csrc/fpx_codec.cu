// fpx_codec.cu -- sm_100a kernels for the ahead-of-time half of the path:
//   K0 quantize  (reference codec.cpp:105-177, bit-exact incl. error order)
//   K1 prepack   (reference prepack.cpp:153-209, bit-exact bytes)
//      unpack    (reference prepack.cpp:211-260)
//   K3 dequant   (reference codec.cpp:179-193 values via the runtime SWAR
//                 path of fpx_dequant.cuh, or a LUT path for other formats)
// plus two small data-movement helpers used by the C-ABI (activation
// staging for unaligned K, and the sharded-output gather permute).
#include <cuda_fp16.h>

#include <cstdint>

#include "fpx_dequant.cuh"
#include "fpx_kernels.h"

namespace fpxk {

// ------------------------------------------------------------------ K0
// One CTA per padded row.  Row r < rows: absmax (NaN-aware), fp16 scale via
// double -> float -> half (codec.cpp:145), zero-scale bump (:153), effective
// scale check (:155-164), then codes = RNE-encode(double(v) / s) (:168-170).
// Failures are folded into one 64-bit atomicMin key (row << 8 | status) so
// the host sees the FIRST failing row in row order (:173-174).

__device__ __forceinline__ uint32_t encode_dev(double v, int e, int m, int bias, double maxrep) {
    const uint32_t smask = 1u << (e + m);
    const uint32_t sign = signbit(v) ? smask : 0u;
    const double a = fabs(v);
    if (a > maxrep) return sign | (smask - 1u);
    const int emin = 1 - bias;
    int ex = (a >= ldexp(1.0, emin)) ? ilogb(a) : emin;
    uint32_t k = static_cast<uint32_t>(rint(ldexp(a, m - ex)));  // ties-to-even
    const uint32_t unit = 1u << m;
    if (k == 2u * unit) {
        k = unit;
        ++ex;
    }
    if (k < unit) return sign | k;
    return sign | (static_cast<uint32_t>(ex + bias) << m) | (k - unit);
}

template <typename T>
__device__ __forceinline__ float load_w(const T* p);
template <>
__device__ __forceinline__ float load_w<float>(const float* p) {
    return *p;
}
template <>
__device__ __forceinline__ float load_w<uint16_t>(const uint16_t* p) {
    return __half2float(__ushort_as_half(*p));  // exact (codec.cpp:35-40)
}

// codes == nullptr: row scales, status and the per-row skip flag only (pass 1
// of the fused quantize+pack, whose tile kernel encodes and packs).
template <typename T>
__global__ void __launch_bounds__(256) quantize_kernel(const T* __restrict__ w, uint32_t rows,
                                                       uint32_t cols, uint32_t cols_p, int e, int m,
                                                       double maxrep, uint8_t* __restrict__ codes,
                                                       uint16_t* __restrict__ scales,
                                                       unsigned long long* __restrict__ status,
                                                       uint8_t* __restrict__ row_skip) {
    const uint32_t r = blockIdx.x;
    uint8_t* out = codes ? codes + static_cast<size_t>(r) * cols_p : nullptr;
    if (codes == nullptr && r >= rows) {
        if (threadIdx.x == 0) scales[r] = 0x3c00u, row_skip[r] = 1;
        return;
    }
    __shared__ float red[8];
    __shared__ int nan_flag;
    __shared__ double s_val;
    __shared__ int skip;
    if (r >= rows) {  // padding rows: codes 0, scale 1.0
        for (uint32_t c = threadIdx.x; c < cols_p; c += blockDim.x) out[c] = 0;
        if (threadIdx.x == 0) scales[r] = 0x3c00u;
        return;
    }
    const T* row = w + static_cast<size_t>(r) * cols;
    if (threadIdx.x == 0) nan_flag = 0;
    __syncthreads();
    float amax = 0.0f;
    bool nan = false;
    for (uint32_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const float a = fabsf(load_w(row + c));
        nan |= isnan(a);
        amax = fmaxf(amax, a);  // fmaxf drops NaN; tracked separately
    }
    if (nan) nan_flag = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.0f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a = fmaxf(a, red[i]);
        int st = 0;
        uint16_t s16 = 0x3c00u;
        skip = 0;
        if (nan_flag) {
            st = 3;  // InvalidValue
        } else if (a == 0.0f) {
            skip = 1;  // all-zero row: scale 1.0, codes 0
        } else {
            const double q = static_cast<double>(a) / maxrep;
            s16 = __half_as_ushort(__float2half_rn(__double2float_rn(q)));
            if ((s16 & 0x7c00u) == 0x7c00u) {
                st = 4;  // ScaleOverflow
            } else {
                if ((s16 & 0x7fffu) == 0u) s16 = static_cast<uint16_t>((s16 & 0x8000u) | 1u);
                const double sv = static_cast<double>(__half2float(__ushort_as_half(s16)));
                const double ev = sv * ldexp(1.0, 15 - ((1 << (e - 1)) - 1));
                const uint16_t eff = __half_as_ushort(__float2half_rn(__double2float_rn(ev)));
                if ((eff & 0x7c00u) == 0x7c00u) st = 4;
            }
        }
        if (st) {
            atomicMin(status, (static_cast<unsigned long long>(r) << 8) | static_cast<unsigned>(st));
            skip = 1;
            s16 = 0x3c00u;
        }
        scales[r] = s16;
        if (row_skip) row_skip[r] = static_cast<uint8_t>(skip);
        s_val = static_cast<double>(__half2float(__ushort_as_half(s16)));
    }
    if (codes == nullptr) return;
    __syncthreads();
    const int bias = (1 << (e - 1)) - 1;
    const double sv = s_val;
    const bool zero = skip != 0;
    for (uint32_t c = threadIdx.x; c < cols_p; c += blockDim.x) {
        uint8_t code = 0;
        if (!zero && c < cols) code = static_cast<uint8_t>(encode_dev(static_cast<double>(load_w(row + c)) / sv, e, m, bias, maxrep));
        out[c] = code;
    }
}

// ------------------------------------------------------------------ K1
// One warp per 64x64 tile.  The tile's codes are staged in shared memory
// with coalesced 16-byte row loads; thread t then walks its 128 codes in
// consumption order (slice, chunk, pair, lane -> prepack.cpp:29-58) and
// ORs each segment into its word (prepack.cpp:71-86); word j is stored at
// (j*32+t)*4 of the tile block -- every store instruction is one coalesced
// 128-byte row (prepack.cpp:115-134).
struct SplitDesc {
    int nseg;
    int width[3];
    uint8_t* stream[3];
};
struct SplitDescC {
    int nseg;
    int width[3];
    const uint8_t* stream[3];
};

constexpr int kPackWarps = 4;

__device__ __forceinline__ void code_rc(uint32_t t, uint32_t k, uint32_t& r, uint32_t& c) {
    const uint32_t s = k >> 5, ch = (k >> 3) & 3u, p = (k >> 1) & 3u, l = k & 1u;
    r = 16u * ch + 8u * (p & 1u) + t / 4u;
    c = 16u * s + 8u * (p >> 1) + 2u * (t % 4u) + l;
}

__constant__ uint32_t kLane[4] = {1u, 3u, 0u, 2u};

__global__ void __launch_bounds__(32 * kPackWarps) prepack_kernel(const uint8_t* __restrict__ codes,
                                                                  uint32_t cols_p, uint32_t ntiles,
                                                                  int bits, SplitDesc sd) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * 64];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t tile = blockIdx.x * kPackWarps + warp;
    if (tile >= ntiles) return;
    const uint32_t gc = cols_p / 64u;
    const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
    uint8_t* ts = tile_s[warp];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t chunk = i * 32u + t;  // 256 x 16-byte chunks
        const uint32_t rr = chunk >> 2, cc = (chunk & 3u) * 16u;
        *reinterpret_cast<uint4*>(ts + rr * 64u + cc) =
            *reinterpret_cast<const uint4*>(codes + static_cast<size_t>(r0 + rr) * cols_p + c0 + cc);
    }
    __syncwarp();
    int low = bits;
    for (int sg = 0; sg < sd.nseg; ++sg) {
        const int w = sd.width[sg];
        low -= w;
        const uint32_t per_word = 8u / w, nwords = 4u * w;
        const uint32_t vmask = (1u << w) - 1u;
        uint8_t* blk = sd.stream[sg] + static_cast<size_t>(tile) * 512u * w;
        for (uint32_t j = 0; j < nwords; ++j) {
            uint32_t word = 0;
            // codes whose segment lands in word j: iterations j*per_word .. +per_word-1
            for (uint32_t g = 0; g < per_word; ++g) {
                const uint32_t it = j * per_word + g;
#pragma unroll
                for (uint32_t q = 0; q < 4u; ++q) {
                    uint32_t rr, cc;
                    code_rc(t, it * 4u + q, rr, cc);
                    const uint32_t v = (static_cast<uint32_t>(ts[rr * 64u + cc]) >> low) & vmask;
                    word |= v << (8u * kLane[q] + 8u - w * (g + 1u));
                }
            }
            reinterpret_cast<uint32_t*>(blk)[j * 32u + t] = word;
        }
    }
}

// ------------------------------------------------------------------ K0+K1 fused
// Pass 2 of fpx_quantize_pack: one warp per 64x64 tile encodes its codes
// straight from the weights (the same fp64 RNE encode of double(w) / s as
// quantize_kernel, codec.cpp:168-170, with the row scales and skip flags of
// pass 1) into shared memory, then packs them exactly like prepack_kernel.
// The code matrix never exists in HBM.
template <typename T>
__global__ void __launch_bounds__(32 * kPackWarps) quantize_pack_kernel(const T* __restrict__ w, uint32_t rows,
                                                                        uint32_t cols, uint32_t cols_p,
                                                                        uint32_t ntiles, int e, int m,
                                                                        double maxrep,
                                                                        const uint16_t* __restrict__ scales,
                                                                        const uint8_t* __restrict__ row_skip,
                                                                        int bits, SplitDesc sd) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * 64];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t tile = blockIdx.x * kPackWarps + warp;
    if (tile >= ntiles) return;
    const uint32_t gc = cols_p / 64u;
    const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
    uint8_t* ts = tile_s[warp];
    const int bias = (1 << (e - 1)) - 1;
    // two rows per pass: lanes 0-15 row 2i, 16-31 row 2i+1, 4 consecutive columns each
    for (uint32_t i = 0; i < 32u; ++i) {
        const uint32_t rr = 2u * i + (t >> 4), cc = (t & 15u) * 4u;
        const uint32_t r = r0 + rr;
        uint32_t packed4 = 0;
        if (r < rows && !row_skip[r]) {
            const double sv = static_cast<double>(__half2float(__ushort_as_half(scales[r])));
            const T* row = w + static_cast<size_t>(r) * cols;
#pragma unroll
            for (uint32_t q = 0; q < 4u; ++q) {
                const uint32_t c = c0 + cc + q;
                if (c < cols)
                    packed4 |= encode_dev(static_cast<double>(load_w(row + c)) / sv, e, m, bias, maxrep) << (8u * q);
            }
        }
        *reinterpret_cast<uint32_t*>(ts + rr * 64u + cc) = packed4;
    }
    __syncwarp();
    int low = bits;
    for (int sg = 0; sg < sd.nseg; ++sg) {
        const int wd = sd.width[sg];
        low -= wd;
        const uint32_t per_word = 8u / wd, nwords = 4u * wd;
        const uint32_t vmask = (1u << wd) - 1u;
        uint8_t* blk = sd.stream[sg] + static_cast<size_t>(tile) * 512u * wd;
        for (uint32_t j = 0; j < nwords; ++j) {
            uint32_t word = 0;
            for (uint32_t g = 0; g < per_word; ++g) {
                const uint32_t it = j * per_word + g;
#pragma unroll
                for (uint32_t q = 0; q < 4u; ++q) {
                    uint32_t rr, cc;
                    code_rc(t, it * 4u + q, rr, cc);
                    const uint32_t v = (static_cast<uint32_t>(ts[rr * 64u + cc]) >> low) & vmask;
                    word |= v << (8u * kLane[q] + 8u - wd * (g + 1u));
                }
            }
            reinterpret_cast<uint32_t*>(blk)[j * 32u + t] = word;
        }
    }
}

// Exact inverse: words -> codes -> tile positions.
__global__ void __launch_bounds__(32 * kPackWarps) unpack_kernel(uint8_t* __restrict__ codes, uint32_t cols_p,
                                                                 uint32_t ntiles, int bits, SplitDescC sd) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * 64];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t tile = blockIdx.x * kPackWarps + warp;
    if (tile >= ntiles) return;
    const uint32_t gc = cols_p / 64u;
    const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
    uint8_t* ts = tile_s[warp];
    for (uint32_t k = 0; k < 128u; ++k) {
        const uint32_t it = k >> 2;
        uint32_t code = 0;
        int low = bits;
        for (int sg = 0; sg < sd.nseg; ++sg) {
            const int w = sd.width[sg];
            low -= w;
            const uint32_t per_word = 8u / w;
            const uint32_t word = reinterpret_cast<const uint32_t*>(sd.stream[sg] + static_cast<size_t>(tile) * 512u * w)[(it / per_word) * 32u + t];
            const uint32_t sh = 8u * kLane[k & 3u] + 8u - w * (it % per_word + 1u);
            code |= ((word >> sh) & ((1u << w) - 1u)) << low;
        }
        uint32_t rr, cc;
        code_rc(t, k, rr, cc);
        ts[rr * 64u + cc] = static_cast<uint8_t>(code);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t chunk = i * 32u + t;
        const uint32_t rr = chunk >> 2, cc = (chunk & 3u) * 16u;
        *reinterpret_cast<uint4*>(codes + static_cast<size_t>(r0 + rr) * cols_p + c0 + cc) =
            *reinterpret_cast<const uint4*>(ts + rr * 64u + cc);
    }
}

// ------------------------------------------------------------------ K3
// Verification de-quantiser.  Block = 2 warps = one 64x64 tile; warp h runs
// exactly a register path of the fused kernel (dequant_slice_half<F, P>:
// P = kHwCvt is what fpx_linear runs, P = kSwar the paper's Algorithm 1) and
// scatters the fp16 results (thread t's R1 of iteration j covers consumption
// indices 32s + 4(4h+j) + {0,1}, R2 the next two) into a shared tile that is
// then written as coalesced rows of the row-major fp16 W.
template <int F, int P>
__global__ void __launch_bounds__(64) dequant_reg_kernel(const uint8_t* __restrict__ s_hi,
                                                          const uint8_t* __restrict__ s_lo,
                                                          const uint16_t* __restrict__ scales,
                                                          uint32_t cols_p, uint16_t* __restrict__ out) {
    __shared__ __align__(16) uint16_t tile_s[64 * 64];
    constexpr int kHi = FmtTraits<F>::kBitsHi, kLo = FmtTraits<F>::kBitsLo;
    const uint32_t tile = blockIdx.x;
    const uint32_t h = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t gc = cols_p / 64u;
    const uint32_t tr = tile / gc, tc = tile % gc;
    const uint8_t* hi = s_hi + static_cast<size_t>(tile) * 512u * kHi;
    const uint8_t* lo = s_lo + static_cast<size_t>(tile) * 512u * kLo;
    uint32_t sc[2][2];
#pragma unroll
    for (int lc = 0; lc < 2; ++lc)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const uint32_t row = tr * 64u + 16u * (2u * h + lc) + 8u * hf + t / 4u;
            sc[lc][hf] = row_scale_for<F, P>(scales[row]);
        }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        uint32_t oa, ob, oc;
        bool ah, bh, ch;
        slice_word_offsets<F>(s, h, t, oa, ob, oc, ah, bh, ch);
        const uint32_t wa = *reinterpret_cast<const uint32_t*>((ah ? hi : lo) + oa);
        const uint32_t wb = *reinterpret_cast<const uint32_t*>((bh ? hi : lo) + ob);
        const uint32_t wc = *reinterpret_cast<const uint32_t*>((ch ? hi : lo) + oc);
        uint32_t r1[4], r2[4];
        dequant_slice_half<F, P>(wa, wb, wc, h, sc, r1, r2);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t k0 = 32u * s + 4u * (4u * h + j);
            uint32_t rr, cc;
            code_rc(t, k0, rr, cc);  // pair of (k0, k0+1): same row, cols cc, cc+1
            *reinterpret_cast<uint32_t*>(&tile_s[rr * 64u + cc]) = r1[j];
            code_rc(t, k0 + 2u, rr, cc);
            *reinterpret_cast<uint32_t*>(&tile_s[rr * 64u + cc]) = r2[j];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 64u * 8u; i += 64u) {  // 64 rows x 8 uint4
        const uint32_t rr = i >> 3, cc = (i & 7u) * 8u;
        *reinterpret_cast<uint4*>(out + static_cast<size_t>(tr * 64u + rr) * cols_p + tc * 64u + cc) =
            *reinterpret_cast<const uint4*>(&tile_s[rr * 64u + cc]);
    }
}

// Any format/split: unsplit -> fp16(decode) LUT -> fp16 multiply by the RAW
// row scale, i.e. literally the oracle's definition (codec.cpp:186-188).
__global__ void __launch_bounds__(32 * kPackWarps) dequant_lut_kernel(SplitDescC sd, int e, int m,
                                                                      const uint16_t* __restrict__ scales,
                                                                      uint32_t cols_p, uint32_t ntiles,
                                                                      uint16_t* __restrict__ out) {
    __shared__ uint16_t lut[256];
    const int bits = 1 + e + m, bias = (1 << (e - 1)) - 1;
    for (int c = threadIdx.x; c < (1 << bits); c += blockDim.x) {
        // fp16(decode_scalar(c)) (codec.cpp:49-68 + half.cpp:30-66), exact in fp32
        const int sg = (c >> (e + m)) & 1, ef = (c >> m) & ((1 << e) - 1), mf = c & ((1 << m) - 1);
        const float v = ef == 0 ? ldexpf(static_cast<float>(mf), 1 - bias - m)
                                : ldexpf(static_cast<float>((1 << m) | mf), ef - bias - m);
        lut[c] = __half_as_ushort(__float2half_rn(sg ? -v : v));
    }
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t tile = blockIdx.x * kPackWarps + warp;
    if (tile >= ntiles) return;
    const uint32_t gc = cols_p / 64u;
    const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
    for (uint32_t k = 0; k < 128u; ++k) {
        const uint32_t it = k >> 2;
        uint32_t code = 0;
        int low = bits;
        for (int sg = 0; sg < sd.nseg; ++sg) {
            const int w = sd.width[sg];
            low -= w;
            const uint32_t per_word = 8u / w;
            const uint32_t word = reinterpret_cast<const uint32_t*>(sd.stream[sg] + static_cast<size_t>(tile) * 512u * w)[(it / per_word) * 32u + t];
            code |= ((word >> (8u * kLane[k & 3u] + 8u - w * (it % per_word + 1u))) & ((1u << w) - 1u)) << low;
        }
        uint32_t rr, cc;
        code_rc(t, k, rr, cc);
        const __half v = __hmul_rn(__ushort_as_half(lut[code]), __ushort_as_half(scales[r0 + rr]));
        out[static_cast<size_t>(r0 + rr) * cols_p + c0 + cc] = __half_as_ushort(v);
    }
}

// dequantize_reference straight from the code matrix (codec.cpp:179-193):
// W[r][c] = half_mul(fp16(decode(code)), scale[r]) for every padded element.
// HBM-bound (1 B in, 2 B out per element): each thread turns 16 codes (one
// 16-byte load) into 16 fp16 (two 16-byte stores) through a shared LUT of
// fp16(decode(code)); a code with bits above the format's width (the
// reference's decode_scalar InvalidCode, codec.cpp:50-53) folds its row into
// the atomicMin error key like quantize.
__global__ void __launch_bounds__(256) dequant_codes_kernel(const uint8_t* __restrict__ codes,
                                                            const uint16_t* __restrict__ scales, uint32_t cols_p,
                                                            size_t nvec, int e, int m,
                                                            unsigned long long* __restrict__ status,
                                                            uint16_t* __restrict__ out) {
    __shared__ uint16_t lut[256];
    const int bits = 1 + e + m, bias = (1 << (e - 1)) - 1;
    for (int c = threadIdx.x; c < 256; c += blockDim.x) {
        const int sg = (c >> (e + m)) & 1, ef = (c >> m) & ((1 << e) - 1), mf = c & ((1 << m) - 1);
        const float v = ef == 0 ? ldexpf(static_cast<float>(mf), 1 - bias - m)
                                : ldexpf(static_cast<float>((1 << m) | mf), ef - bias - m);
        lut[c] = __half_as_ushort(__float2half_rn(sg ? -v : v));
    }
    __syncthreads();
    const uint32_t bad_mask = ~((1u << bits) - 1u) & 0xffu;
    const uint32_t vec_per_row = cols_p / 16u;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nvec;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint4 cw = __ldcs(reinterpret_cast<const uint4*>(codes) + i);
        const size_t row = i / vec_per_row;
        const uint16_t sraw = __ldg(&scales[row]);
        const __half2 s2 = __half2half2(__ushort_as_half(sraw));
        // NaN results follow the reference's host arithmetic (fp32 product on
        // x86, half.cpp:68-70): a NaN scale propagates quieted with its sign
        // and payload; inf x 0 is the default NaN 0xFE00.  (Only reachable
        // with hand-made non-finite scales: quantize never produces them.)
        const uint32_t nan_fix = (sraw & 0x7fffu) > 0x7c00u ? (sraw | 0x0200u) : 0xfe00u;
        const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
        uint32_t o[8];
        uint32_t any_bad = 0;
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
            const uint32_t w = words[wi];
            any_bad |= w & (bad_mask * 0x01010101u);
#pragma unroll
            for (int hp = 0; hp < 2; ++hp) {
                const uint32_t lo = lut[(w >> (16 * hp)) & 0xffu], hi = lut[(w >> (16 * hp + 8)) & 0xffu];
                const __half2 d = __halves2half2(__ushort_as_half(static_cast<uint16_t>(lo)),
                                                 __ushort_as_half(static_cast<uint16_t>(hi)));
                const __half2 r = __hmul2_rn(d, s2);  // fp16 RNE product, subnormals kept (half.cpp:68-70)
                uint32_t v = *reinterpret_cast<const uint32_t*>(&r);
                if ((v & 0x7fffu) > 0x7c00u) v = (v & 0xffff0000u) | nan_fix;
                if (((v >> 16) & 0x7fffu) > 0x7c00u) v = (v & 0xffffu) | (nan_fix << 16);
                o[2 * wi + hp] = v;
            }
        }
        if (any_bad) atomicMin(status, (static_cast<unsigned long long>(row) << 8) | 2ull /* FPX_ERR_INVALID_CODE */);
        uint4* dst = reinterpret_cast<uint4*>(out) + 2 * i;
        __stcs(dst, make_uint4(o[0], o[1], o[2], o[3]));
        __stcs(dst + 1, make_uint4(o[4], o[5], o[6], o[7]));
    }
}

// Scale-validity scan for pack (prepack.cpp:165-168): flags any row whose
// effective scale is not finite.
__global__ void check_scales_kernel(const uint16_t* __restrict__ scales, uint32_t n, int rebias,
                                    unsigned int* __restrict__ bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && (effective_scale_dev(scales[i], rebias) & 0x7c00u) == 0x7c00u) atomicOr(bad, 1u);
}

// Copy col-major activations (k_act x n, arbitrary k_act) into a K_pad-strided
// zero-padded buffer so the tensor map has 16-byte aligned rows.
__global__ void stage_act_kernel(const uint16_t* __restrict__ src, uint32_t k_act, uint32_t n,
                                 uint32_t k_pad, uint16_t* __restrict__ dst) {
    const size_t total = static_cast<size_t>(k_pad) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t j = static_cast<uint32_t>(i / k_pad), k = static_cast<uint32_t>(i % k_pad);
        dst[i] = k < k_act ? src[static_cast<size_t>(j) * k_act + k] : 0;
    }
}

// Gathered [world][n][m_slot] -> col-major [n][ldc] with per-rank row ranges.
__global__ void gather_permute_kernel(const float* __restrict__ g, const uint32_t* __restrict__ row0,
                                      const uint32_t* __restrict__ nrows, int world, uint32_t m_slot,
                                      uint32_t n, float* __restrict__ c, uint32_t ldc) {
    const size_t total = static_cast<size_t>(world) * n * m_slot;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t m = static_cast<uint32_t>(i % m_slot);
        const size_t rest = i / m_slot;
        const uint32_t j = static_cast<uint32_t>(rest % n);
        const int r = static_cast<int>(rest / n);
        if (m < nrows[r]) c[static_cast<size_t>(j) * ldc + row0[r] + m] = g[i];
    }
}

// gathered [world][n][m_slot] -> col-major C, with each rank's tile-row range
// recomputed from fpx_shard_rows' formula (no host-side tables).
__global__ void gather_shards_kernel(const float* __restrict__ g, uint32_t rows_p, int world, uint32_t m_slot,
                                     uint32_t n, float* __restrict__ c, uint32_t ldc) {
    const uint64_t trs = rows_p / 64u;
    const size_t total = static_cast<size_t>(world) * n * m_slot;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t m = static_cast<uint32_t>(i % m_slot);
        const size_t rest = i / m_slot;
        const uint32_t j = static_cast<uint32_t>(rest % n);
        const int r = static_cast<int>(rest / n);
        const uint32_t tr0 = static_cast<uint32_t>(trs * r / world), tr1 = static_cast<uint32_t>(trs * (r + 1) / world);
        if (m < (tr1 - tr0) * 64u) c[static_cast<size_t>(j) * ldc + tr0 * 64u + m] = g[i];
    }
}

}  // namespace fpxk

cudaError_t launch_dequant_codes(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p, int e,
                                 int m, unsigned long long* status, uint16_t* out, cudaStream_t st) {
    const size_t nvec = static_cast<size_t>(rows_p) * cols_p / 16u;
    fpxk::dequant_codes_kernel<<<148 * 8, 256, 0, st>>>(codes, scales, cols_p, nvec, e, m, status, out);
    return cudaGetLastError();
}

cudaError_t launch_gather_shards(const float* g, uint32_t rows_p, int world, uint32_t m_slot, uint32_t n, float* c,
                                 uint32_t ldc, cudaStream_t st) {
    fpxk::gather_shards_kernel<<<592, 256, 0, st>>>(g, rows_p, world, m_slot, n, c, ldc);
    return cudaGetLastError();
}

// ------------------------------------------------------------ launchers
using namespace fpxk;

static SplitDesc make_sd(int nseg, const int* widths, uint8_t* const* streams) {
    SplitDesc sd{};
    sd.nseg = nseg;
    for (int i = 0; i < nseg; ++i) sd.width[i] = widths[i], sd.stream[i] = streams[i];
    return sd;
}
static SplitDescC make_sdc(int nseg, const int* widths, const uint8_t* const* streams) {
    SplitDescC sd{};
    sd.nseg = nseg;
    for (int i = 0; i < nseg; ++i) sd.width[i] = widths[i], sd.stream[i] = streams[i];
    return sd;
}

cudaError_t launch_quantize(const void* w, int w_dtype, uint32_t rows, uint32_t cols, uint32_t rows_p,
                            uint32_t cols_p, int e, int m, double maxrep, uint8_t* codes,
                            uint16_t* scales, unsigned long long* status, cudaStream_t st) {
    if (w_dtype == 0)
        quantize_kernel<float><<<rows_p, 256, 0, st>>>(static_cast<const float*>(w), rows, cols, cols_p, e, m,
                                                       maxrep, codes, scales, status, nullptr);
    else
        quantize_kernel<uint16_t><<<rows_p, 256, 0, st>>>(static_cast<const uint16_t*>(w), rows, cols, cols_p,
                                                          e, m, maxrep, codes, scales, status, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_quantize_pack(const void* w, int w_dtype, uint32_t rows, uint32_t cols, uint32_t rows_p,
                                 uint32_t cols_p, int e, int m, double maxrep, uint16_t* scales,
                                 unsigned long long* status, uint8_t* row_skip, int nseg, const int* widths,
                                 uint8_t* const* streams, cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    const int bits = 1 + e + m;
    const SplitDesc sd = make_sd(nseg, widths, streams);
    const uint32_t grid = (ntiles + kPackWarps - 1) / kPackWarps;
    if (w_dtype == 0) {
        quantize_kernel<float><<<rows_p, 256, 0, st>>>(static_cast<const float*>(w), rows, cols, cols_p, e, m,
                                                       maxrep, nullptr, scales, status, row_skip);
        quantize_pack_kernel<float><<<grid, 32 * kPackWarps, 0, st>>>(
            static_cast<const float*>(w), rows, cols, cols_p, ntiles, e, m, maxrep, scales, row_skip, bits, sd);
    } else {
        quantize_kernel<uint16_t><<<rows_p, 256, 0, st>>>(static_cast<const uint16_t*>(w), rows, cols, cols_p, e,
                                                          m, maxrep, nullptr, scales, status, row_skip);
        quantize_pack_kernel<uint16_t><<<grid, 32 * kPackWarps, 0, st>>>(static_cast<const uint16_t*>(w), rows,
                                                                         cols, cols_p, ntiles, e, m, maxrep,
                                                                         scales, row_skip, bits, sd);
    }
    return cudaGetLastError();
}

cudaError_t launch_prepack(const uint8_t* codes, uint32_t rows_p, uint32_t cols_p, int bits, int nseg,
                           const int* widths, uint8_t* const* streams, cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    if (ntiles == 0) return cudaSuccess;
    prepack_kernel<<<(ntiles + kPackWarps - 1) / kPackWarps, 32 * kPackWarps, 0, st>>>(
        codes, cols_p, ntiles, bits, make_sd(nseg, widths, streams));
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint8_t* const* streams, uint32_t rows_p, uint32_t cols_p, int bits, int nseg,
                          const int* widths, uint8_t* codes, cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    if (ntiles == 0) return cudaSuccess;
    unpack_kernel<<<(ntiles + kPackWarps - 1) / kPackWarps, 32 * kPackWarps, 0, st>>>(
        codes, cols_p, ntiles, bits, make_sdc(nseg, widths, streams));
    return cudaGetLastError();
}

template <int F>
static void launch_reg(int path, uint32_t ntiles, const uint8_t* const* streams, const uint16_t* scales,
                       uint32_t cols_p, uint16_t* out, cudaStream_t st) {
    if (path == 1)
        dequant_reg_kernel<F, kSwar><<<ntiles, 64, 0, st>>>(streams[0], streams[1], scales, cols_p, out);
    else
        dequant_reg_kernel<F, kHwCvt><<<ntiles, 64, 0, st>>>(streams[0], streams[1], scales, cols_p, out);
}

// path: 0 = the fused kernel's hardware-convert register path, 1 = SWAR
// (Algorithm 1), 2 = LUT (any format).  Formats without a register path
// always use the LUT.
cudaError_t launch_dequant(const uint8_t* const* streams, int nseg, const int* widths, const uint16_t* scales,
                           uint32_t rows_p, uint32_t cols_p, int e, int m, uint16_t* out, int path,
                           cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    if (ntiles == 0) return cudaSuccess;
    const bool s24 = nseg == 2 && widths[0] == 2 && widths[1] == 4;
    const bool s41 = nseg == 2 && widths[0] == 4 && widths[1] == 1;
    if (path != 2 && e == 3 && m == 2 && s24) {
        launch_reg<kE3M2>(path, ntiles, streams, scales, cols_p, out, st);
    } else if (path != 2 && e == 2 && m == 3 && s24) {
        launch_reg<kE2M3>(path, ntiles, streams, scales, cols_p, out, st);
    } else if (path != 2 && e == 2 && m == 2 && s41) {
        launch_reg<kE2M2>(path, ntiles, streams, scales, cols_p, out, st);
    } else {
        dequant_lut_kernel<<<(ntiles + kPackWarps - 1) / kPackWarps, 32 * kPackWarps, 0, st>>>(
            make_sdc(nseg, widths, streams), e, m, scales, cols_p, ntiles, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_check_scales(const uint16_t* scales, uint32_t n, int rebias, unsigned int* bad,
                                cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    check_scales_kernel<<<(n + 255) / 256, 256, 0, st>>>(scales, n, rebias, bad);
    return cudaGetLastError();
}

cudaError_t launch_stage_act(const uint16_t* src, uint32_t k_act, uint32_t n, uint32_t k_pad, uint16_t* dst,
                             cudaStream_t st) {
    stage_act_kernel<<<592, 256, 0, st>>>(src, k_act, n, k_pad, dst);
    return cudaGetLastError();
}

cudaError_t launch_gather_permute(const float* g, const uint32_t* row0, const uint32_t* nrows, int world,
                                  uint32_t m_slot, uint32_t n, float* c, uint32_t ldc, cudaStream_t st) {
    gather_permute_kernel<<<592, 256, 0, st>>>(g, row0, nrows, world, m_slot, n, c, ldc);
    return cudaGetLastError();
}
