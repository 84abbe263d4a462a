// fpx_codec.cu -- sm_100a kernels for the ahead-of-time half of the path:
//   K0 quantize  (reference codec.cpp:105-177, bit-exact incl. error order)
//   K1 prepack   (reference prepack.cpp:153-209, bit-exact bytes)
//      unpack    (reference prepack.cpp:211-260)
//   K3 dequant   (reference codec.cpp:179-193 values via the runtime SWAR
//                 path of fpx_dequant.cuh, or a LUT path for other formats)
// plus two small data-movement helpers used by the C-ABI (activation
// staging for unaligned K, and the sharded-output gather permute).
#include <cuda_fp16.h>

#include <algorithm>
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
//
// The encode runs without any division (encode_exact).  The reference rounds
// q = double(w) / s to nearest in double, then rounds q to the format:
// ex = floor(log2 q) (>= emin), k = rint(q * 2^(m - ex)) ties-to-even,
// saturating at max_rep.  Here q is formed in fp32 as |w| * fp32(1/s), whose
// relative error (<= 2^-23) moves y = q * 2^(m - ex) < 2^(m+1) by at most
// 2^(m-22); so rint(y) is the reference's k unless y lies within
// eps = 2^(m-20) of a half-integer, and those rare cases are decided
// exactly: the midpoint T = (floor(y) + 1/2) * 2^(ex - m) * s has at most
// m + 2 + 11 significant bits, so it is exact in fp32, and |w| compares
// exactly against it (the double quotient of the reference cannot make a
// tie out of |w| != T: both sit on |w|'s ulp grid, >= 2^-24 |w| apart).  An
// exact tie goes to the even k, like the reference's rint.  A quotient that
// rounds across a power of two only moves k to the next binade's first
// code, which is the same code.  Values above the largest code round to it
// (min with cmax), which is the reference's saturation.

// The reference's encode(double(w) / s) for s > 0 (sv = s, inv = fp32 1/s).
__device__ __forceinline__ uint32_t encode_exact(float w, float sv, float inv, int e, int m, int bias,
                                                 uint32_t cmax) {
    const uint32_t sign = (__float_as_uint(w) >> 31) << (e + m);
    const float a = fabsf(w);
    const float q = a * inv;
    int ex = static_cast<int>((__float_as_uint(q) >> 23) & 0xffu) - 127;
    ex = min(max(ex, 1 - bias), 120);
    const float y = q * __uint_as_float(static_cast<uint32_t>(127 + m - ex) << 23);  // q * 2^(m - ex), exact
    float kf = rintf(y);
    const float eps = __uint_as_float(static_cast<uint32_t>(127 + m - 20) << 23);
    if (fabsf(y - kf) > 0.5f - eps) {
        // near a tie: compare against the exact midpoint
        const float fl = floorf(y);
        const float t = (fl + 0.5f) * __uint_as_float(static_cast<uint32_t>(127 + ex - m) << 23) * sv;
        kf = a > t ? fl + 1.0f : (a < t ? fl : fl + (fmodf(fl, 2.0f) != 0.0f ? 1.0f : 0.0f));
    }
    const uint32_t k = static_cast<uint32_t>(kf);
    const uint32_t unit = 1u << m;
    uint32_t c = k < unit ? k : (static_cast<uint32_t>(ex + bias) << m) + k - unit;
    return sign | min(c, cmax);
}

// Four weights at once.  For the FP6 formats the candidate comes from the
// sm_100a hardware conversion (cvt.rn.satfinite.e3m2x2 / e2m3x2.f32, two
// codes per instruction) applied to q * (1 + 2^-20) and q * (1 - 2^-20):
// where both agree no rounding boundary lies within 2^-20 of q -- wider than
// q's own error -- so that is the reference's code; otherwise (near a tie,
// rare) encode_exact decides.
//
// FP5 e2m2 rides on the e3m2 conversion: e2m2(q) = 4 * e3m2(q / 4) for
// q / 4 <= 1.75.  Both keep 2 mantissa bits; e3m2's normal range starts at
// 2^-2 (q >= 1, e2m2's normal range) with the same exponent field (bias 3
// vs 1 absorbs the factor 4), and its subnormal step 2^-4 is e2m2's 2^-2 / 4.
// So the e2m2 magnitude code is the e3m2 one, saturated at 15 (7.0) where
// the quotient rounds to 2.0 or above.
enum EncMode { kEncGeneric = 0, kEncHwE3M2 = 1, kEncHwE2M3 = 2, kEncHwE2M2 = 3 };

template <int MODE>
__device__ __forceinline__ uint32_t cvt_fp6x2(float lo, float hi) {
    uint16_t r;
    if constexpr (MODE == kEncHwE3M2 || MODE == kEncHwE2M2)
        asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    else
        asm("cvt.rn.satfinite.e2m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __noinline__ uint32_t encode4_exact_slow(float4 v, float sv, float inv, int e, int m, int bias,
                                                    uint32_t cmax) {
    return encode_exact(v.x, sv, inv, e, m, bias, cmax) | encode_exact(v.y, sv, inv, e, m, bias, cmax) << 8 |
           encode_exact(v.z, sv, inv, e, m, bias, cmax) << 16 | encode_exact(v.w, sv, inv, e, m, bias, cmax) << 24;
}

template <int MODE>
__device__ __forceinline__ uint32_t encode4(float4 v, float sv, float inv, int e, int m, int bias, uint32_t cmax) {
    if constexpr (MODE == kEncGeneric) {
        return encode_exact(v.x, sv, inv, e, m, bias, cmax) | encode_exact(v.y, sv, inv, e, m, bias, cmax) << 8 |
               encode_exact(v.z, sv, inv, e, m, bias, cmax) << 16 | encode_exact(v.w, sv, inv, e, m, bias, cmax) << 24;
    } else {
        // Signed quotients: the conversion rounds magnitudes and carries the
        // sign (also of zero and of underflow to zero), exactly the
        // reference's sign | magnitude code, so no sign bits are assembled.
        constexpr bool k5 = MODE == kEncHwE2M2;
        const float iv = k5 ? inv * 0.25f : inv;  // exact: a power-of-two factor
        const float qa = v.x * iv, qb = v.y * iv, qc = v.z * iv, qd = v.w * iv;
        constexpr float kUp = 1.0f + 0x1p-20f, kDn = 1.0f - 0x1p-20f;
        const uint32_t up = cvt_fp6x2<MODE>(qa * kUp, qb * kUp) | cvt_fp6x2<MODE>(qc * kUp, qd * kUp) << 16;
        const uint32_t dn = cvt_fp6x2<MODE>(qa * kDn, qb * kDn) | cvt_fp6x2<MODE>(qc * kDn, qd * kDn) << 16;
        if (up != dn)  // a quotient near a rounding boundary (rare: kept out of line)
            return encode4_exact_slow(v, sv, inv, e, m, bias, cmax);
        // e2m2: sign bit 5 -> 4, magnitude saturated at 15 (7.0)
        if constexpr (k5) return __vminu4(up & 0x1f1f1f1fu, 0x0f0f0f0fu) | ((up >> 1) & 0x10101010u);
        return up & 0x3f3f3f3fu;
    }
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

// Four consecutive weights of a row (vector load when aligned).
template <typename T>
__device__ __forceinline__ float4 load_w4(const T* p, bool vec);
template <>
__device__ __forceinline__ float4 load_w4<float>(const float* p, bool vec) {
    if (vec) return __ldcs(reinterpret_cast<const float4*>(p));
    return make_float4(p[0], p[1], p[2], p[3]);
}
template <>
__device__ __forceinline__ float4 load_w4<uint16_t>(const uint16_t* p, bool vec) {
    uint32_t lo, hi;
    if (vec) {
        const uint2 v = __ldcs(reinterpret_cast<const uint2*>(p));
        lo = v.x, hi = v.y;
    } else {
        lo = p[0] | (static_cast<uint32_t>(p[1]) << 16), hi = p[2] | (static_cast<uint32_t>(p[3]) << 16);
    }
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&lo));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&hi));
    return make_float4(a.x, a.y, b.x, b.y);
}

// 16 bytes of a row (16-byte aligned) as groups of 4 weights.
__device__ __forceinline__ void load_w16(const float* p, float4 (&v)[1]) {
    v[0] = __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void load_w16(const uint16_t* p, float4 (&v)[2]) {
    const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
    const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
    v[0] = make_float4(a.x, a.y, b.x, b.y);
    v[1] = make_float4(c.x, c.y, d.x, d.y);
}

// The 16 bytes of a row at column c when they run past `cols` (or are not
// 16-byte aligned): element-wise, +0.0 past the end.
__device__ __forceinline__ uint4 load_raw16_ragged(const float* row, uint32_t c, uint32_t cols) {
    uint32_t x[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) x[q] = c + q < cols ? __float_as_uint(row[c + q]) : 0u;
    return make_uint4(x[0], x[1], x[2], x[3]);
}
__device__ __forceinline__ uint4 load_raw16_ragged(const uint16_t* row, uint32_t c, uint32_t cols) {
    uint32_t x[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t a = c + 2 * q < cols ? row[c + 2 * q] : 0u;
        const uint32_t b = c + 2 * q + 1 < cols ? row[c + 2 * q + 1] : 0u;
        x[q] = a | (b << 16);
    }
    return make_uint4(x[0], x[1], x[2], x[3]);
}

// 16 raw bytes of a row as groups of 4 weights (exact widening).
__device__ __forceinline__ void raw16_to_float4(const uint4& u, float4 (&v)[1]) {
    v[0] = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w));
}
__device__ __forceinline__ void raw16_to_float4(const uint4& u, float4 (&v)[2]) {
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
    const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
    v[0] = make_float4(a.x, a.y, b.x, b.y);
    v[1] = make_float4(c.x, c.y, d.x, d.y);
}

// Thread 0 of a row's CTA, after the row max: fp16 scale via
// double -> float -> half (codec.cpp:145), zero-scale bump (:153), effective
// scale check (:155-164); failures folded into the status key (:173-174).
__device__ __forceinline__ void decide_row_scale(uint32_t r, float a, bool nan, int e, double maxrep,
                                                 uint16_t* scales, unsigned long long* status, uint8_t* row_skip,
                                                 int& skip, float& s_val) {
    int st = 0;
    uint16_t s16 = 0x3c00u;
    skip = 0;
    if (nan) {
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
    s_val = __half2float(__ushort_as_half(s16));
}

// Row pass: scale + status (+ the row's codes when codes != nullptr).
// codes == nullptr: row scales, status and the per-row skip flag only (pass 1
// of the fused quantize+pack, whose tile kernel encodes and packs).
template <typename T, int MODE>
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
    __shared__ float s_val;
    __shared__ int skip;
    if (r >= rows) {  // padding rows: codes 0, scale 1.0
        for (uint32_t c = threadIdx.x * 16; c < cols_p; c += blockDim.x * 16)
            *reinterpret_cast<uint4*>(out + c) = make_uint4(0u, 0u, 0u, 0u);
        if (threadIdx.x == 0) scales[r] = 0x3c00u;
        return;
    }
    const T* row = w + static_cast<size_t>(r) * cols;
    // vector loads when the row start is 16-byte (fp32) / 8-byte (fp16) aligned
    const bool vec = (reinterpret_cast<uintptr_t>(row) % (4 * sizeof(T))) == 0;
    const uint32_t c4 = cols & ~3u;
    if (threadIdx.x == 0) nan_flag = 0;
    __syncthreads();
    float amax = 0.0f;
    bool nan = false;
    // eight independent vector loads in flight per thread (the row is
    // streamed once here and once more, mostly from L2, by the encode)
    // 16-byte loads (kG groups of 4 weights) when the rows are 16-byte aligned
    constexpr uint32_t kG = 16u / (4u * sizeof(T));
    const bool vec16 = (reinterpret_cast<uintptr_t>(w) % 16u) == 0 && (static_cast<size_t>(cols) * sizeof(T)) % 16u == 0;
    constexpr uint32_t kU = 8;
    uint32_t c = threadIdx.x * 4;
    if (vec16 && kG > 1) {
        const uint32_t stp = blockDim.x * 4 * kG;
        for (c = threadIdx.x * 4 * kG; c + (kU / kG - 1) * stp + 4 * kG <= c4; c += (kU / kG) * stp) {
            float4 v[kU / kG][kG];
#pragma unroll
            for (uint32_t u = 0; u < kU / kG; ++u) load_w16(row + c + u * stp, v[u]);
#pragma unroll
            for (uint32_t u = 0; u < kU / kG; ++u)
#pragma unroll
                for (uint32_t gq = 0; gq < kG; ++gq) {
                    const float4 x = v[u][gq];
                    nan |= isnan(x.x) | isnan(x.y) | isnan(x.z) | isnan(x.w);
                    amax = fmaxf(fmaxf(amax, fmaxf(fabsf(x.x), fabsf(x.y))), fmaxf(fabsf(x.z), fabsf(x.w)));
                }
        }
        // the rest 4 at a time, continuing where each thread's 16-byte walk stopped
        for (uint32_t cq = c; cq < c4; cq += stp)
            for (uint32_t gq = 0; gq < kG && cq + 4 * gq < c4; ++gq) {
                const float4 x = load_w4(row + cq + 4 * gq, vec);
                nan |= isnan(x.x) | isnan(x.y) | isnan(x.z) | isnan(x.w);
                amax = fmaxf(fmaxf(amax, fmaxf(fabsf(x.x), fabsf(x.y))), fmaxf(fabsf(x.z), fabsf(x.w)));
            }
        c = c4;
    }
    for (; c + (kU - 1) * blockDim.x * 4 < c4; c += kU * blockDim.x * 4) {
        float4 v[kU];
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) v[u] = load_w4(row + c + u * blockDim.x * 4, vec);
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            nan |= isnan(v[u].x) | isnan(v[u].y) | isnan(v[u].z) | isnan(v[u].w);
            amax = fmaxf(fmaxf(amax, fmaxf(fabsf(v[u].x), fabsf(v[u].y))), fmaxf(fabsf(v[u].z), fabsf(v[u].w)));
        }
    }
    for (; c < c4; c += blockDim.x * 4) {
        const float4 v = load_w4(row + c, vec);
        nan |= isnan(v.x) | isnan(v.y) | isnan(v.z) | isnan(v.w);
        amax = fmaxf(fmaxf(amax, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));  // fmaxf drops NaN
    }
    for (uint32_t c = c4 + threadIdx.x; c < cols; c += blockDim.x) {
        const float a = fabsf(load_w(row + c));
        nan |= isnan(a);
        amax = fmaxf(amax, a);
    }
    if (nan) nan_flag = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.0f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a = fmaxf(a, red[i]);
        decide_row_scale(r, a, nan_flag != 0, e, maxrep, scales, status, row_skip, skip, s_val);
    }
    if (codes == nullptr) return;
    __syncthreads();
    const int bias = (1 << (e - 1)) - 1;
    const float sv = s_val, inv = __frcp_rn(s_val);
    const uint32_t cmax = (1u << (e + m)) - 1u;
    const bool zero = skip != 0;
    // 4 codes (one 32-bit store) per thread and vector; four vectors in
    // flight per iteration over the row's full-width part, then the tail
    constexpr uint32_t kE = 4;
    const uint32_t step = blockDim.x * 4;
    uint32_t c0 = threadIdx.x * 4;
    if (!zero) {
        for (; c0 + (kE - 1) * step + 4 <= cols; c0 += kE * step) {
            float4 v[kE];
#pragma unroll
            for (uint32_t u = 0; u < kE; ++u) v[u] = load_w4(row + c0 + u * step, vec);
#pragma unroll
            for (uint32_t u = 0; u < kE; ++u) {
                *reinterpret_cast<uint32_t*>(out + c0 + u * step) = encode4<MODE>(v[u], sv, inv, e, m, bias, cmax);
            }
        }
    }
    for (uint32_t c = c0; c < cols_p; c += step) {
        uint32_t packed = 0;
        if (!zero && c < cols) {
            float4 v;
            if (c + 4 <= cols) {
                v = load_w4(row + c, vec);
            } else {
                v.x = load_w(row + c);
                v.y = c + 1 < cols ? load_w(row + c + 1) : 0.0f;
                v.z = c + 2 < cols ? load_w(row + c + 2) : 0.0f;
                v.w = c + 3 < cols ? load_w(row + c + 3) : 0.0f;
            }
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c + j < cols) packed |= encode_exact(vv[j], sv, inv, e, m, bias, cmax) << (8 * j);
        }
        *reinterpret_cast<uint32_t*>(out + c) = packed;
    }
}

// K0 with the row staged in shared memory (rows of at most kStageMax
// bytes, 16-byte aligned): one bulk copy brings the whole row in -- up to
// ~88 KB in flight per CTA with no per-thread load slots -- and both the max
// and the encode read it from shared memory, so HBM sees each weight once
// (the two-pass kernel above re-reads most rows from DRAM: ~1.3 GB of reads
// for 0.72 GB of fp32 weights at 8192 x 22016).
cudaError_t ensure_smem_attr(const void* kern, int bytes);  // fpx_linear.cu (per device)
constexpr uint32_t kStageMax = 200u * 1024u;
constexpr uint32_t kStageChunk = 32u * 1024u;

template <typename T, int MODE>
__global__ void __launch_bounds__(256) quantize_staged_kernel(const T* __restrict__ w, uint32_t cols, uint32_t cols_p,
                                                              int e, int m, double maxrep, uint8_t* __restrict__ codes,
                                                              uint16_t* __restrict__ scales,
                                                              unsigned long long* __restrict__ status) {
    extern __shared__ __align__(16) uint8_t srow[];
    __shared__ uint64_t full;
    __shared__ float red[8];
    __shared__ int nan_flag;
    __shared__ float s_val;
    __shared__ int skip;
    const uint32_t r = blockIdx.x;
    const uint32_t bytes = cols * sizeof(T);  // % 16 == 0 (host check)
    if (threadIdx.x == 0) {
        nan_flag = 0;
        mbar_init(&full, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&full, bytes);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(w + static_cast<size_t>(r) * cols);
        const uint64_t pol = policy_evict_first();
        for (uint32_t o = 0; o < bytes; o += kStageChunk)
            bulk_g2s(srow + o, src + o, min(kStageChunk, bytes - o), &full, pol);
    }
    __syncthreads();
    mbar_wait(&full, 0);
    constexpr uint32_t kG = 16u / (4u * sizeof(T));  // groups of 4 weights per 16 bytes
    const uint32_t n16 = bytes / 16u;
    float amax = 0.0f;
    bool nan = false;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
        float4 v[kG];
        raw16_to_float4(reinterpret_cast<const uint4*>(srow)[i], v);
#pragma unroll
        for (uint32_t gq = 0; gq < kG; ++gq) {
            const float4 x = v[gq];
            nan |= isnan(x.x) | isnan(x.y) | isnan(x.z) | isnan(x.w);
            amax = fmaxf(fmaxf(amax, fmaxf(fabsf(x.x), fabsf(x.y))), fmaxf(fabsf(x.z), fabsf(x.w)));
        }
    }
    if (nan) nan_flag = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.0f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a = fmaxf(a, red[i]);
        decide_row_scale(r, a, nan_flag != 0, e, maxrep, scales, status, nullptr, skip, s_val);
    }
    __syncthreads();
    const int bias = (1 << (e - 1)) - 1;
    const float sv = s_val, inv = __frcp_rn(s_val);
    const uint32_t cmax = (1u << (e + m)) - 1u;
    uint8_t* out = codes + static_cast<size_t>(r) * cols_p;
    // 16 bytes of weights -> kG code words; columns past cols (to cols_p) get code 0
    if (skip) {
        for (uint32_t c = threadIdx.x * 4; c < cols_p; c += blockDim.x * 4) *reinterpret_cast<uint32_t*>(out + c) = 0u;
        return;
    }
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
        float4 v[kG];
        raw16_to_float4(reinterpret_cast<const uint4*>(srow)[i], v);
        uint32_t packed[kG];
#pragma unroll
        for (uint32_t gq = 0; gq < kG; ++gq) packed[gq] = encode4<MODE>(v[gq], sv, inv, e, m, bias, cmax);
        if constexpr (kG == 1)
            *reinterpret_cast<uint32_t*>(out + 4 * i) = packed[0];
        else
            *reinterpret_cast<uint2*>(out + 8 * i) = make_uint2(packed[0], packed[kG - 1]);
    }
    for (uint32_t c = cols + threadIdx.x * 4; c < cols_p; c += blockDim.x * 4)
        *reinterpret_cast<uint32_t*>(out + c) = 0u;
}

// ------------------------------------------------------------------ K1
// One warp per 64x64 tile.  The tile's codes are staged in shared memory
// (coalesced 16-byte row loads; row stride 80 bytes so the eight rows one
// gather instruction touches fall on eight different bank groups).  Thread t
// then builds its words iteration by iteration: iteration it = (slice s,
// chunk c, column half ph) holds the four codes (rows r0, r0 + 8) x (columns
// c0, c0 + 1), r0 = 16c + t/4, c0 = 16s + 8ph + 2(t%4) (prepack.cpp:29-58),
// fetched with two 16-bit shared loads and placed into byte lanes {1, 3, 0,
// 2} (prepack.cpp:17) with one PRMT.  Each segment of width w is then cut out
// of all four lanes at once (SWAR: shift, mask) and shifted to bits
// 8 - w(g+1) of its lane (prepack.cpp:71-86); word j is stored at
// (j*32+t)*4 of the tile block, one coalesced 128-byte row per store
// instruction (prepack.cpp:115-134).
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
constexpr int kTileStride = 80;  // bytes per staged 64-code row

__device__ __forceinline__ void code_rc(uint32_t t, uint32_t k, uint32_t& r, uint32_t& c) {
    const uint32_t s = k >> 5, ch = (k >> 3) & 3u, p = (k >> 1) & 3u, l = k & 1u;
    r = 16u * ch + 8u * (p & 1u) + t / 4u;
    c = 16u * s + 8u * (p >> 1) + 2u * (t % 4u) + l;
}

__constant__ uint32_t kLane[4] = {1u, 3u, 0u, 2u};

// The four codes of iteration `it` of thread t in byte lanes {1, 3, 0, 2}:
// lane 1 (r0, c0), lane 3 (r0, c0+1), lane 0 (r0+8, c0), lane 2 (r0+8, c0+1).
__device__ __forceinline__ uint32_t iter_codes(const uint8_t* ts, uint32_t t, uint32_t it) {
    const uint32_t s = it >> 3, ch = (it >> 1) & 3u, ph = it & 1u;
    const uint32_t r0 = 16u * ch + t / 4u, c0 = 16u * s + 8u * ph + 2u * (t % 4u);
    const uint32_t a = *reinterpret_cast<const uint16_t*>(ts + r0 * kTileStride + c0);
    const uint32_t b = *reinterpret_cast<const uint16_t*>(ts + (r0 + 8u) * kTileStride + c0);
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, 0x1504;" : "=r"(d) : "r"(a), "r"(b));  // bytes {b.lo, a.lo, b.hi, a.hi}
    return d;
}

// Pack a staged tile (stride kTileStride) into its stream blocks: segment
// of width W at bit `low`, words built in registers from all 32 iterations.
template <int W>
__device__ __forceinline__ void pack_segment(const uint32_t (&x)[32], int low, uint8_t* stream, uint32_t t,
                                             uint32_t tile) {
    constexpr uint32_t kPer = 8u / W, kWords = 4u * W;
    constexpr uint32_t kMask = ((1u << W) - 1u) * 0x01010101u;
    uint32_t* blk = reinterpret_cast<uint32_t*>(stream + static_cast<size_t>(tile) * 512u * W);
#pragma unroll
    for (uint32_t j = 0; j < kWords; ++j) {
        uint32_t word = 0;
#pragma unroll
        for (uint32_t g = 0; g < kPer; ++g) word |= ((x[j * kPer + g] >> low) & kMask) << (8u - W * (g + 1u));
        blk[j * 32u + t] = word;
    }
}

__device__ __forceinline__ void pack_tile(const uint8_t* ts, uint32_t t, uint32_t tile, int bits, const SplitDesc& sd) {
    uint32_t x[32];
#pragma unroll
    for (uint32_t it = 0; it < 32u; ++it) x[it] = iter_codes(ts, t, it);
    int low = bits;
    for (int sg = 0; sg < sd.nseg; ++sg) {
        const int w = sd.width[sg];
        low -= w;
        switch (w) {
            case 1: pack_segment<1>(x, low, sd.stream[sg], t, tile); break;
            case 2: pack_segment<2>(x, low, sd.stream[sg], t, tile); break;
            case 4: pack_segment<4>(x, low, sd.stream[sg], t, tile); break;
            default: break;  // the C-ABI admits widths 1, 2 and 4 only
        }
    }
}

// Persistent warps: each walks tiles gw, gw + nw, ... with the next tile's
// 4 KB of codes already in flight (registers) while it packs the current one.
__global__ void __launch_bounds__(32 * kPackWarps) prepack_kernel(const uint8_t* __restrict__ codes,
                                                                  uint32_t cols_p, uint32_t ntiles,
                                                                  int bits, SplitDesc sd) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * kTileStride];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t nw = gridDim.x * kPackWarps;
    const uint32_t gc = cols_p / 64u;
    uint8_t* ts = tile_s[warp];
    auto load = [&](uint32_t tile, uint4 (&v)[8]) {
        const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t chunk = i * 32u + t;  // 256 x 16-byte chunks
            v[i] = __ldcs(reinterpret_cast<const uint4*>(codes + static_cast<size_t>(r0 + (chunk >> 2)) * cols_p + c0 +
                                                         (chunk & 3u) * 16u));
        }
    };
    uint32_t tile = blockIdx.x * kPackWarps + warp;
    uint4 cur[8];
    if (tile < ntiles) load(tile, cur);
    for (; tile < ntiles; tile += nw) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t chunk = i * 32u + t;
            *reinterpret_cast<uint4*>(ts + (chunk >> 2) * kTileStride + (chunk & 3u) * 16u) = cur[i];
        }
        if (tile + nw < ntiles) load(tile + nw, cur);  // next tile in flight
        __syncwarp();
        pack_tile(ts, t, tile, bits, sd);
        __syncwarp();  // ts is rewritten next iteration
    }
}

// ------------------------------------------------------------------ K0+K1 fused
// Pass 2 of fpx_quantize_pack: one warp per 64x64 tile encodes its codes
// straight from the weights (encode_exact with the row scales and skip flags
// of pass 1) into shared memory, then packs them exactly like
// prepack_kernel.  The code matrix never touches HBM.
template <typename T, int MODE>
__global__ void __launch_bounds__(32 * kPackWarps) quantize_pack_kernel(const T* __restrict__ w, uint32_t rows,
                                                                        uint32_t cols, uint32_t cols_p,
                                                                        uint32_t ntiles, int e, int m,
                                                                        double maxrep,
                                                                        const uint16_t* __restrict__ scales,
                                                                        const uint8_t* __restrict__ row_skip,
                                                                        int bits, SplitDesc sd) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * kTileStride];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t tile = blockIdx.x * kPackWarps + warp;
    if (tile >= ntiles) return;
    const uint32_t gc = cols_p / 64u;
    const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
    uint8_t* ts = tile_s[warp];
    const int bias = (1 << (e - 1)) - 1;
    const uint32_t cmax = (1u << (e + m)) - 1u;
    (void)maxrep;
    // Each lane reads 16 bytes of one row per pass -- kG groups of 4 weights
    // (fp32: 1, fp16: 2) -- so kLpr lanes cover a 64-weight tile row and a
    // pass covers kRpp rows.  Passes run in chunks of kChunk with every load
    // of the chunk issued first, kept as raw 16-byte words (converted to fp32
    // only at the encode), so both dtypes keep 128 bytes per lane in flight;
    // row scales and skip flags load alongside and apply after.
    constexpr uint32_t kG = 16u / (4u * sizeof(T)), kLpr = 16u / kG, kRpp = 32u / kLpr;
    // 16-byte words in flight per lane: 8 for fp32 input, 4 for fp16 (its
    // encode of 8 weights per word needs the registers; 87 -> 64 per thread)
    constexpr uint32_t kChunk = sizeof(T) == 2 ? 4u : 8u;
    static_assert((64u / kRpp) % kChunk == 0, "passes per chunk");
    const uint32_t cc = (t % kLpr) * 4u * kG, c = c0 + cc;
    const bool full = c + 4u * kG <= cols;
    const bool vec = (reinterpret_cast<uintptr_t>(w) % 16u) == 0 && (static_cast<size_t>(cols) * sizeof(T)) % 16u == 0;
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < 64u / kRpp; i0 += kChunk) {
        uint4 raw[kChunk];
        uint16_t sraw[kChunk];
        uint8_t skip[kChunk];
#pragma unroll
        for (uint32_t j = 0; j < kChunk; ++j) {
            const uint32_t r = r0 + kRpp * (i0 + j) + t / kLpr;
            raw[j] = make_uint4(0u, 0u, 0u, 0u);  // +0.0 in either dtype: code 0
            sraw[j] = 0x3c00u;
            skip[j] = 1;
            if (r < rows) {
                const T* row = w + static_cast<size_t>(r) * cols;
                sraw[j] = scales[r];
                skip[j] = row_skip[r];
                if (full && vec) {
                    raw[j] = __ldcs(reinterpret_cast<const uint4*>(row + c));
                } else {
                    raw[j] = load_raw16_ragged(row, c, cols);
                }
            }
        }
#pragma unroll
        for (uint32_t j = 0; j < kChunk; ++j) {
            const uint32_t rr = kRpp * (i0 + j) + t / kLpr;
            uint32_t packed[kG];
#pragma unroll
            for (uint32_t gq = 0; gq < kG; ++gq) packed[gq] = 0u;
            if (!skip[j]) {
                const float sv = __half2float(__ushort_as_half(sraw[j])), inv = __frcp_rn(sv);
                float4 v[kG];
                raw16_to_float4(raw[j], v);
#pragma unroll
                for (uint32_t gq = 0; gq < kG; ++gq)  // columns >= cols hold +0.0: code 0
                    packed[gq] = encode4<MODE>(v[gq], sv, inv, e, m, bias, cmax);
            }
            if constexpr (kG == 1)
                *reinterpret_cast<uint32_t*>(ts + rr * kTileStride + cc) = packed[0];
            else
                *reinterpret_cast<uint2*>(ts + rr * kTileStride + cc) = make_uint2(packed[0], packed[kG - 1]);
        }
    }
    __syncwarp();
    pack_tile(ts, t, tile, bits, sd);
}

// Exact inverse (prepack.cpp:211-260): every segment's words are cut back
// into the 32 iterations' byte lanes (SWAR), then each iteration's four
// codes go to their two rows with two 16-bit shared stores and the staged
// tile leaves as coalesced 16-byte rows.
template <int W>
__device__ __forceinline__ void unpack_segment(uint32_t (&x)[32], int low, const uint8_t* stream, uint32_t t,
                                               uint32_t tile) {
    constexpr uint32_t kPer = 8u / W, kWords = 4u * W;
    constexpr uint32_t kMask = ((1u << W) - 1u) * 0x01010101u;
    const uint32_t* blk = reinterpret_cast<const uint32_t*>(stream + static_cast<size_t>(tile) * 512u * W);
#pragma unroll
    for (uint32_t j = 0; j < kWords; ++j) {
        const uint32_t word = __ldcs(blk + j * 32u + t);
#pragma unroll
        for (uint32_t g = 0; g < kPer; ++g) x[j * kPer + g] |= ((word >> (8u - W * (g + 1u))) & kMask) << low;
    }
}

__global__ void __launch_bounds__(32 * kPackWarps) unpack_kernel(uint8_t* __restrict__ codes, uint32_t cols_p,
                                                                 uint32_t ntiles, int bits, SplitDescC sd) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * kTileStride];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t tile = blockIdx.x * kPackWarps + warp;
    if (tile >= ntiles) return;
    const uint32_t gc = cols_p / 64u;
    const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
    uint8_t* ts = tile_s[warp];
    uint32_t x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = 0u;
    int low = bits;
    for (int sg = 0; sg < sd.nseg; ++sg) {
        const int w = sd.width[sg];
        low -= w;
        switch (w) {
            case 1: unpack_segment<1>(x, low, sd.stream[sg], t, tile); break;
            case 2: unpack_segment<2>(x, low, sd.stream[sg], t, tile); break;
            case 4: unpack_segment<4>(x, low, sd.stream[sg], t, tile); break;
            default: break;
        }
    }
#pragma unroll
    for (uint32_t it = 0; it < 32u; ++it) {
        const uint32_t s = it >> 3, ch = (it >> 1) & 3u, ph = it & 1u;
        const uint32_t rr = 16u * ch + t / 4u, cc = 16u * s + 8u * ph + 2u * (t % 4u);
        uint32_t a, b;
        asm("prmt.b32 %0, %1, 0, 0x4431;" : "=r"(a) : "r"(x[it]));  // lanes 1, 3 -> row rr
        asm("prmt.b32 %0, %1, 0, 0x4420;" : "=r"(b) : "r"(x[it]));  // lanes 0, 2 -> row rr + 8
        *reinterpret_cast<uint16_t*>(ts + rr * kTileStride + cc) = static_cast<uint16_t>(a);
        *reinterpret_cast<uint16_t*>(ts + (rr + 8u) * kTileStride + cc) = static_cast<uint16_t>(b);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t chunk = i * 32u + t;
        const uint32_t rr = chunk >> 2, cc = (chunk & 3u) * 16u;
        *reinterpret_cast<uint4*>(codes + static_cast<size_t>(r0 + rr) * cols_p + c0 + cc) =
            *reinterpret_cast<const uint4*>(ts + rr * kTileStride + cc);
    }
}

// The two-segment splits ([2,4] FP6, [4,1] FP5) with persistent warps that
// keep the next tile's packed words in flight (registers) while they unpack
// the current one, as prepack_kernel does for the forward direction.
template <int W>
__device__ __forceinline__ void unpack_words(const uint32_t (&wd)[4 * W], uint32_t (&x)[32], int low) {
    constexpr uint32_t kPer = 8u / W;
    constexpr uint32_t kMask = ((1u << W) - 1u) * 0x01010101u;
#pragma unroll
    for (uint32_t j = 0; j < 4u * W; ++j)
#pragma unroll
        for (uint32_t g = 0; g < kPer; ++g) x[j * kPer + g] |= ((wd[j] >> (8u - W * (g + 1u))) & kMask) << low;
}

template <int W0, int W1>
__global__ void __launch_bounds__(32 * kPackWarps) unpack2_kernel(uint8_t* __restrict__ codes, uint32_t cols_p,
                                                                  uint32_t ntiles, const uint8_t* __restrict__ s0,
                                                                  const uint8_t* __restrict__ s1) {
    __shared__ __align__(16) uint8_t tile_s[kPackWarps][64 * kTileStride];
    const uint32_t warp = threadIdx.x >> 5, t = threadIdx.x & 31u;
    const uint32_t nw = gridDim.x * kPackWarps;
    const uint32_t gc = cols_p / 64u;
    uint8_t* ts = tile_s[warp];
    auto load = [&](uint32_t tile, uint32_t (&a)[4 * W0], uint32_t (&b)[4 * W1]) {
        const uint32_t* pa = reinterpret_cast<const uint32_t*>(s0 + static_cast<size_t>(tile) * 512u * W0);
        const uint32_t* pb = reinterpret_cast<const uint32_t*>(s1 + static_cast<size_t>(tile) * 512u * W1);
#pragma unroll
        for (uint32_t j = 0; j < 4u * W0; ++j) a[j] = __ldcs(pa + j * 32u + t);
#pragma unroll
        for (uint32_t j = 0; j < 4u * W1; ++j) b[j] = __ldcs(pb + j * 32u + t);
    };
    uint32_t tile = blockIdx.x * kPackWarps + warp;
    uint32_t ca[4 * W0], cb[4 * W1];
    if (tile < ntiles) load(tile, ca, cb);
    for (; tile < ntiles; tile += nw) {
        uint32_t x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = 0u;
        unpack_words<W0>(ca, x, W1);  // segment 0 holds the high bits
        unpack_words<W1>(cb, x, 0);
        if (tile + nw < ntiles) load(tile + nw, ca, cb);  // next tile in flight
        const uint32_t r0 = (tile / gc) * 64u, c0 = (tile % gc) * 64u;
#pragma unroll
        for (uint32_t it = 0; it < 32u; ++it) {
            const uint32_t sl = it >> 3, ch = (it >> 1) & 3u, ph = it & 1u;
            const uint32_t rr = 16u * ch + t / 4u, cc = 16u * sl + 8u * ph + 2u * (t % 4u);
            uint32_t a, b;
            asm("prmt.b32 %0, %1, 0, 0x4431;" : "=r"(a) : "r"(x[it]));  // lanes 1, 3 -> row rr
            asm("prmt.b32 %0, %1, 0, 0x4420;" : "=r"(b) : "r"(x[it]));  // lanes 0, 2 -> row rr + 8
            *reinterpret_cast<uint16_t*>(ts + rr * kTileStride + cc) = static_cast<uint16_t>(a);
            *reinterpret_cast<uint16_t*>(ts + (rr + 8u) * kTileStride + cc) = static_cast<uint16_t>(b);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t chunk = i * 32u + t;
            const uint32_t rr = chunk >> 2, cc = (chunk & 3u) * 16u;
            *reinterpret_cast<uint4*>(codes + static_cast<size_t>(r0 + rr) * cols_p + c0 + cc) =
                *reinterpret_cast<const uint4*>(ts + rr * kTileStride + cc);
        }
        __syncwarp();  // ts is rewritten next iteration
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
    // row stride 72 halves (144 B): the 8 rows one fragment store touches
    // land 4 banks apart (64 would put them all on the same 4 banks)
    constexpr uint32_t kStr = 72u;
    __shared__ __align__(16) uint16_t tile_s[64 * kStr];
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
            *reinterpret_cast<uint32_t*>(&tile_s[rr * kStr + cc]) = r1[j];
            code_rc(t, k0 + 2u, rr, cc);
            *reinterpret_cast<uint32_t*>(&tile_s[rr * kStr + cc]) = r2[j];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 64u * 8u; i += 64u) {  // 64 rows x 8 uint4
        const uint32_t rr = i >> 3, cc = (i & 7u) * 8u;
        *reinterpret_cast<uint4*>(out + static_cast<size_t>(tr * 64u + rr) * cols_p + tc * 64u + cc) =
            *reinterpret_cast<const uint4*>(&tile_s[rr * kStr + cc]);
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

static int enc_mode(int e, int m) {
    if (e == 3 && m == 2) return kEncHwE3M2;
    if (e == 2 && m == 3) return kEncHwE2M3;
    return e == 2 && m == 2 ? kEncHwE2M2 : kEncGeneric;
}

template <typename T, int MODE>
static void launch_quantize_t(const void* w, uint32_t rows, uint32_t cols, uint32_t rows_p, uint32_t cols_p, int e,
                              int m, double maxrep, uint8_t* codes, uint16_t* scales, unsigned long long* status,
                              uint8_t* row_skip, cudaStream_t st) {
    const size_t bytes = static_cast<size_t>(cols) * sizeof(T);
    // whole rows in shared memory when they fit and are 16-byte aligned (the
    // padding rows past `rows` stay with the two-pass kernel below)
    if (codes != nullptr && row_skip == nullptr && bytes % 16 == 0 && bytes <= kStageMax &&
        reinterpret_cast<uintptr_t>(w) % 16 == 0 && cols % 4 == 0) {
        auto kern = quantize_staged_kernel<T, MODE>;
        if (ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(kStageMax)) == cudaSuccess) {
            kern<<<rows, 256, bytes, st>>>(static_cast<const T*>(w), cols, cols_p, e, m, maxrep, codes, scales,
                                           status);
            if (rows_p > rows)  // padding rows: codes 0, scale 1.0
                quantize_kernel<T, MODE><<<rows_p - rows, 256, 0, st>>>(static_cast<const T*>(w), 0, cols, cols_p, e,
                                                                        m, maxrep, codes + static_cast<size_t>(rows) *
                                                                                               cols_p,
                                                                        scales + rows, status, row_skip);
            return;
        }
        (void)cudaGetLastError();
    }
    quantize_kernel<T, MODE><<<rows_p, 256, 0, st>>>(static_cast<const T*>(w), rows, cols, cols_p, e, m, maxrep, codes,
                                                     scales, status, row_skip);
}

template <typename T>
static void launch_quantize_m(const void* w, uint32_t rows, uint32_t cols, uint32_t rows_p, uint32_t cols_p, int e,
                              int m, double maxrep, uint8_t* codes, uint16_t* scales, unsigned long long* status,
                              uint8_t* row_skip, cudaStream_t st) {
    // the mode only matters for the encode (codes != nullptr)
    switch (codes == nullptr ? kEncGeneric : enc_mode(e, m)) {
        case kEncHwE3M2:
            return launch_quantize_t<T, kEncHwE3M2>(w, rows, cols, rows_p, cols_p, e, m, maxrep, codes, scales, status,
                                                    row_skip, st);
        case kEncHwE2M3:
            return launch_quantize_t<T, kEncHwE2M3>(w, rows, cols, rows_p, cols_p, e, m, maxrep, codes, scales, status,
                                                    row_skip, st);
        case kEncHwE2M2:
            return launch_quantize_t<T, kEncHwE2M2>(w, rows, cols, rows_p, cols_p, e, m, maxrep, codes, scales, status,
                                                    row_skip, st);
        default:
            return launch_quantize_t<T, kEncGeneric>(w, rows, cols, rows_p, cols_p, e, m, maxrep, codes, scales,
                                                     status, row_skip, st);
    }
}

cudaError_t launch_quantize(const void* w, int w_dtype, uint32_t rows, uint32_t cols, uint32_t rows_p,
                            uint32_t cols_p, int e, int m, double maxrep, uint8_t* codes,
                            uint16_t* scales, unsigned long long* status, cudaStream_t st) {
    if (w_dtype == 0)
        launch_quantize_m<float>(w, rows, cols, rows_p, cols_p, e, m, maxrep, codes, scales, status, nullptr, st);
    else
        launch_quantize_m<uint16_t>(w, rows, cols, rows_p, cols_p, e, m, maxrep, codes, scales, status, nullptr, st);
    return cudaGetLastError();
}

template <typename T>
static void launch_qpack(const void* w, uint32_t rows, uint32_t cols, uint32_t cols_p, uint32_t ntiles, int e, int m,
                         double maxrep, const uint16_t* scales, const uint8_t* row_skip, int bits, const SplitDesc& sd,
                         cudaStream_t st) {
    const uint32_t grid = (ntiles + kPackWarps - 1) / kPackWarps;
    const T* wt = static_cast<const T*>(w);
    switch (enc_mode(e, m)) {
        case kEncHwE3M2:
            quantize_pack_kernel<T, kEncHwE3M2><<<grid, 32 * kPackWarps, 0, st>>>(wt, rows, cols, cols_p, ntiles, e, m,
                                                                                 maxrep, scales, row_skip, bits, sd);
            break;
        case kEncHwE2M3:
            quantize_pack_kernel<T, kEncHwE2M3><<<grid, 32 * kPackWarps, 0, st>>>(wt, rows, cols, cols_p, ntiles, e, m,
                                                                                 maxrep, scales, row_skip, bits, sd);
            break;
        case kEncHwE2M2:
            quantize_pack_kernel<T, kEncHwE2M2><<<grid, 32 * kPackWarps, 0, st>>>(wt, rows, cols, cols_p, ntiles, e, m,
                                                                                 maxrep, scales, row_skip, bits, sd);
            break;
        default:
            quantize_pack_kernel<T, kEncGeneric><<<grid, 32 * kPackWarps, 0, st>>>(wt, rows, cols, cols_p, ntiles, e, m,
                                                                                  maxrep, scales, row_skip, bits, sd);
    }
}

cudaError_t launch_quantize_pack(const void* w, int w_dtype, uint32_t rows, uint32_t cols, uint32_t rows_p,
                                 uint32_t cols_p, int e, int m, double maxrep, uint16_t* scales,
                                 unsigned long long* status, uint8_t* row_skip, int nseg, const int* widths,
                                 uint8_t* const* streams, cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    const int bits = 1 + e + m;
    const SplitDesc sd = make_sd(nseg, widths, streams);
    if (w_dtype == 0) {
        launch_quantize_m<float>(w, rows, cols, rows_p, cols_p, e, m, maxrep, nullptr, scales, status, row_skip, st);
        launch_qpack<float>(w, rows, cols, cols_p, ntiles, e, m, maxrep, scales, row_skip, bits, sd, st);
    } else {
        launch_quantize_m<uint16_t>(w, rows, cols, rows_p, cols_p, e, m, maxrep, nullptr, scales, status, row_skip, st);
        launch_qpack<uint16_t>(w, rows, cols, cols_p, ntiles, e, m, maxrep, scales, row_skip, bits, sd, st);
    }
    return cudaGetLastError();
}

// persistent CTAs per SM for the pack / unpack kernels: 11 x 20 KB of
// staging fills the SM's shared memory (measured 8 -> 11: prepack 59.8 ->
// 57.1 us, unpack 56.7 -> 53.6 us at 8192 x 22016)
constexpr uint32_t kPackCtasPerSm = 11;

cudaError_t launch_prepack(const uint8_t* codes, uint32_t rows_p, uint32_t cols_p, int bits, int nseg,
                           const int* widths, uint8_t* const* streams, cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    if (ntiles == 0) return cudaSuccess;
    const uint32_t blocks = std::min<uint32_t>((ntiles + kPackWarps - 1) / kPackWarps, 148u * kPackCtasPerSm);
    prepack_kernel<<<blocks, 32 * kPackWarps, 0, st>>>(codes, cols_p, ntiles, bits, make_sd(nseg, widths, streams));
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint8_t* const* streams, uint32_t rows_p, uint32_t cols_p, int bits, int nseg,
                          const int* widths, uint8_t* codes, cudaStream_t st) {
    const uint32_t ntiles = (rows_p / 64u) * (cols_p / 64u);
    if (ntiles == 0) return cudaSuccess;
    const uint32_t blocks = std::min<uint32_t>((ntiles + kPackWarps - 1) / kPackWarps, 148u * kPackCtasPerSm);
    if (nseg == 2 && widths[0] == 2 && widths[1] == 4) {
        unpack2_kernel<2, 4><<<blocks, 32 * kPackWarps, 0, st>>>(codes, cols_p, ntiles, streams[0], streams[1]);
    } else if (nseg == 2 && widths[0] == 4 && widths[1] == 1) {
        unpack2_kernel<4, 1><<<blocks, 32 * kPackWarps, 0, st>>>(codes, cols_p, ntiles, streams[0], streams[1]);
    } else {
        unpack_kernel<<<(ntiles + kPackWarps - 1) / kPackWarps, 32 * kPackWarps, 0, st>>>(
            codes, cols_p, ntiles, bits, make_sdc(nseg, widths, streams));
    }
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
