// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (/root/reference/proj), compiled together with the reference's own
// sources into oracle/_ref/libfpxref.so by oracle/Makefile.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used to pin the C restatement
// (oracle/fpx_oracle.c), to generate tests/golden/, and as the CPU baseline
// arm of bench.py.  No reference source is copied into this repository; this
// file only marshals plain buffers into the reference's value types and calls
// its public API (codec.hpp:66, prepack.hpp:84-86, gemm.hpp:27-32).
//
// Status: 0 ok, else 1 + (int)fpx::ErrorCode; ref_last_error() has the text.
#include <cstdint>
#include <cstring>
#include <string>

#include "fpx/codec.hpp"
#include "fpx/error.hpp"
#include "fpx/format.hpp"
#include "fpx/gemm.hpp"
#include "fpx/half.hpp"
#include "fpx/prepack.hpp"

namespace {
thread_local std::string g_err;

int fail(const fpx::Error& e) {
    g_err = e.formatted();
    return 1 + static_cast<int>(e.code());
}

fpx::QuantizedMatrix make_q(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p,
                            uint32_t cols_p, uint32_t orig_rows, uint32_t orig_cols, int e,
                            int m) {
    fpx::QuantizedMatrix q;
    q.format = fpx::FpxFormat::make(e, m);
    q.rows = rows_p;
    q.cols = cols_p;
    q.orig_rows = orig_rows;
    q.orig_cols = orig_cols;
    q.codes.assign(codes, codes + size_t(rows_p) * cols_p);
    q.scales.assign(scales, scales + rows_p);
    return q;
}

fpx::ScalarMatrix make_b(const uint16_t* b, uint32_t b_rows, uint32_t n) {
    fpx::ScalarMatrix m = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp16, fpx::Layout::ColMajor, b_rows, n);
    std::memcpy(m.f16.data(), b, size_t(b_rows) * n * 2);
    return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_quantize(const float* w, uint32_t rows, uint32_t cols, int e, int m, uint8_t* codes,
                 uint16_t* scales) {
    try {
        fpx::ScalarMatrix s = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp32, fpx::Layout::RowMajor, rows, cols);
        std::memcpy(s.f32.data(), w, size_t(rows) * cols * 4);
        fpx::QuantizedMatrix q = fpx::quantize_matrix(s, fpx::FpxFormat::make(e, m));
        std::memcpy(codes, q.codes.data(), q.codes.size());
        std::memcpy(scales, q.scales.data(), q.scales.size() * 2);
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

// streams[i] must hold rows_p*cols_p*widths[i]/8 bytes (split = preset).
int ref_pack(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
             uint32_t orig_rows, uint32_t orig_cols, int e, int m, uint8_t* const* streams) {
    try {
        fpx::PackedWeights p = fpx::pack(make_q(codes, scales, rows_p, cols_p, orig_rows, orig_cols, e, m));
        for (size_t i = 0; i < p.streams.size(); ++i)
            std::memcpy(streams[i], p.streams[i].data(), p.streams[i].size());
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

int ref_unpack(uint8_t const* const* streams, const uint16_t* scales, uint32_t rows_p,
               uint32_t cols_p, int e, int m, uint8_t* codes) {
    try {
        fpx::PackedWeights p;
        p.format = fpx::FpxFormat::make(e, m);
        p.split = fpx::SplitScheme::for_format(p.format);
        p.rows = p.orig_rows = rows_p;
        p.cols = p.orig_cols = cols_p;
        p.scales.assign(scales, scales + rows_p);
        for (int w : p.split.widths) {
            size_t nb = size_t(rows_p) * cols_p * w / 8;
            p.streams.emplace_back(streams[p.streams.size()], streams[p.streams.size()] + nb);
        }
        fpx::QuantizedMatrix q = fpx::unpack(p);
        std::memcpy(codes, q.codes.data(), q.codes.size());
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

int ref_dequantize(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
                   int e, int m, uint16_t* out) {
    try {
        fpx::ScalarMatrix w = fpx::dequantize_reference(make_q(codes, scales, rows_p, cols_p, rows_p, cols_p, e, m));
        std::memcpy(out, w.f16.data(), w.f16.size() * 2);
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

uint16_t ref_float_to_half(float f) { return fpx::float_to_half(f); }
float ref_half_to_float(uint16_t h) { return fpx::half_to_float(h); }
uint16_t ref_half_mul(uint16_t a, uint16_t b) { return fpx::half_mul(a, b); }
float ref_decode(uint32_t code, int e, int m) { return fpx::decode_scalar(code, fpx::FpxFormat::make(e, m)); }
uint32_t ref_encode(double v, int e, int m) { return fpx::encode_scalar(v, fpx::FpxFormat::make(e, m)); }

uint16_t ref_effective_scale(uint16_t s, int e, int m) {
    return fpx::effective_scale(s, fpx::FpxFormat::make(e, m));
}

// Packed-path GEMM through the reference's own public API: quantized codes
// are packed with fpx::pack (once, outside any timing done by the caller of
// ref_gemm_packed_prepared) -- see ref_prepare / ref_release below.
struct RefPrepared {
    fpx::PackedWeights p;
    fpx::QuantizedMatrix q;
};

void* ref_prepare(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
                  uint32_t orig_rows, uint32_t orig_cols, int e, int m) {
    try {
        auto* r = new RefPrepared;
        r->q = make_q(codes, scales, rows_p, cols_p, orig_rows, orig_cols, e, m);
        r->p = fpx::pack(r->q);
        return r;
    } catch (const fpx::Error& err) {
        fail(err);
        return nullptr;
    }
}

void ref_release(void* h) { delete static_cast<RefPrepared*>(h); }

// C: fp32 col-major rows_p x n.
int ref_gemm_packed(void* h, const uint16_t* b, uint32_t b_rows, uint32_t n, float* c) {
    try {
        auto* r = static_cast<RefPrepared*>(h);
        fpx::ScalarMatrix out = fpx::gemm_packed(r->p, make_b(b, b_rows, n));
        std::memcpy(c, out.f32.data(), out.f32.size() * 4);
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

// gemm_reference straight from codes (no pack): the parity tests' oracle C
// for full-size problems.  C: fp32 col-major rows_p x n.
int ref_gemm_reference_codes(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
                             uint32_t orig_rows, uint32_t orig_cols, int e, int m, const uint16_t* b, uint32_t b_rows,
                             uint32_t n, float* c) {
    try {
        fpx::ScalarMatrix out = fpx::gemm_reference(make_q(codes, scales, rows_p, cols_p, orig_rows, orig_cols, e, m),
                                                    make_b(b, b_rows, n));
        std::memcpy(c, out.f32.data(), out.f32.size() * 4);
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

int ref_gemm_reference(void* h, const uint16_t* b, uint32_t b_rows, uint32_t n, float* c) {
    try {
        auto* r = static_cast<RefPrepared*>(h);
        fpx::ScalarMatrix out = fpx::gemm_reference(r->q, make_b(b, b_rows, n));
        std::memcpy(c, out.f32.data(), out.f32.size() * 4);
        return 0;
    } catch (const fpx::Error& err) {
        return fail(err);
    }
}

}  // extern "C"
