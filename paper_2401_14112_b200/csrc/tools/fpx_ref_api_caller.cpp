// fpx_ref_api_caller.cpp -- a caller written ONLY against the reference
// library's public headers and names (/root/reference/proj/include/fpx/:
// format.hpp, error.hpp, half.hpp, codec.hpp, prepack.hpp, gemm.hpp, io.hpp),
// compiled unchanged with -I include (include/fpx/*.hpp) and linked against
// libfpx_b200.so.  It is the drop-in check of SURVEY §8b: every call below is
// a reference API call, served by the sm_100a kernels.
//
// Usage: fpx_ref_api_caller [out_dir]
//   Runs SPEC.md's scalar KATs, error behaviour and contracts (acceptance
//   criteria 2 and 3: unpack(pack(q)) == q, gemm_packed == gemm_reference
//   bit for bit; dequantize_reference == the packed path's W), then, with
//   out_dir, writes a fixed problem's inputs and outputs as raw little-endian
//   files for tests/test_gpu_parity.py to compare with the reference itself.
// Exit 0 = all checks passed; 1 = a check failed; 3 = device/runtime error.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#include "fpx/codec.hpp"
#include "fpx/error.hpp"
#include "fpx/format.hpp"
#include "fpx/gemm.hpp"
#include "fpx/half.hpp"
#include "fpx/io.hpp"
#include "fpx/prepack.hpp"

namespace {

int g_fail = 0;

void expect(bool ok, const std::string& what) {
    if (!ok) {
        std::printf("FAIL %s\n", what.c_str());
        ++g_fail;
    }
}

template <typename F>
void expect_error(fpx::ErrorCode code, F&& fn, const std::string& what) {
    try {
        fn();
        expect(false, what + ": no error");
    } catch (const fpx::Error& e) {
        expect(e.code() == code, what + ": got " + e.formatted());
    }
}

template <typename T>
void dump(const std::string& dir, const char* name, const std::vector<T>& v) {
    std::ofstream f(dir + "/" + name, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const fpx::FpxFormat e3m2 = fpx::FpxFormat::e3m2();
        // ---- format.hpp / half.hpp
        expect(e3m2.bias() == 3 && e3m2.total_bits() == 6 && e3m2.max_representable() == 28.0f, "e3m2 descriptor");
        expect(fpx::FpxFormat::parse("e2m3") == fpx::FpxFormat::e2m3(), "parse e2m3");
        expect(!fpx::FpxFormat::parse("e9m9").has_value(), "parse rejects e9m9");
        expect(fpx::SplitScheme::for_format(e3m2).widths == std::vector<int>({2, 4}), "e3m2 split [2,4]");
        expect(fpx::SplitScheme::for_format(fpx::FpxFormat::e2m2()).widths == std::vector<int>({4, 1}), "e2m2 split [4,1]");
        expect(e3m2.ulp_at(1.0) == 0.25f && e3m2.ulp_at(0.01) == 0.0625f && e3m2.ulp_at(100.0) == 4.0f, "ulp_at");
        expect(fpx::float_to_half(1.0f) == 0x3C00 && fpx::half_to_float(0x3000) == 0.125f, "half conversions");
        expect(fpx::half_mul(0x3C00, 0x4000) == 0x4000 && fpx::half_is_nan(0x7e00) && !fpx::half_is_finite(0x7c00),
               "half_mul / classification");
        expect_error(fpx::ErrorCode::InvalidFormat, [] { fpx::FpxFormat::make(6, 3); }, "make(6,3)");
        // ---- codec.hpp scalar KATs (with SURVEY §4.3's errata:
        // the S|EEE|MM code 0b011100 is E=7 -> 16.0; 1.0 is 0b001100)
        expect(fpx::decode_scalar(0b000000, e3m2) == 0.0f, "decode 0");
        expect(fpx::decode_scalar(0b011100, e3m2) == 16.0f, "decode 0b011100");
        expect(fpx::decode_scalar(0b001100, e3m2) == 1.0f, "decode 0b001100");
        expect(fpx::decode_scalar(0b011111, e3m2) == 28.0f, "decode max");
        expect(fpx::decode_scalar(0b000001, e3m2) == 0.0625f, "decode min subnormal");
        expect(fpx::encode_scalar(1.0, e3m2) == 0b001100u, "encode 1.0");
        expect(fpx::encode_scalar(1000.0, e3m2) == 0b011111u, "encode saturates");
        expect(fpx::encode_scalar(-0.0, e3m2) == 0b100000u, "encode -0");
        for (const fpx::FpxFormat f : {e3m2, fpx::FpxFormat::e2m3(), fpx::FpxFormat::e2m2(), fpx::FpxFormat::e2m1()})
            for (uint32_t c = 0; c < f.code_count(); ++c)
                expect(fpx::encode_scalar(fpx::decode_scalar(c, f), f) == c, "round trip " + f.name() + " code " + std::to_string(c));
        expect_error(fpx::ErrorCode::InvalidCode, [&] { fpx::decode_scalar(64, e3m2); }, "decode 64");
        expect_error(fpx::ErrorCode::InvalidValue, [&] { fpx::encode_scalar(std::nan(""), e3m2); }, "encode NaN");
        expect(fpx::effective_scale(0x3C00, e3m2) == fpx::float_to_half(4096.0f), "effective_scale e3m2");

        // ---- matrices: a ragged 200 x 330 problem (padded to 256 x 384), N = 24
        const uint32_t rows = 200, cols = 330, n = 24;
        std::mt19937 rng(2401);
        std::normal_distribution<float> nd(0.0f, 0.02f), na(0.0f, 1.0f);
        fpx::ScalarMatrix w = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp32, fpx::Layout::RowMajor, rows, cols);
        for (float& v : w.f32) v = nd(rng);
        for (uint32_t c = 0; c < cols; ++c) w.f32[5 * cols + c] = 0.0f;  // an all-zero row: scale 1.0
        fpx::ScalarMatrix b = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp16, fpx::Layout::ColMajor, cols, n);
        for (uint16_t& v : b.f16) v = fpx::float_to_half(na(rng));

        const fpx::QuantizedMatrix q = fpx::quantize_matrix(w, e3m2);
        expect(q.rows == 256 && q.cols == 384 && q.orig_rows == rows && q.orig_cols == cols, "padded dims");
        expect(q.scales[5] == 0x3C00, "zero row scale 1.0");
        const fpx::PackedWeights p = fpx::pack(q);
        expect(p.streams.size() == 2 && p.streams[0].size() == 256u * 384u / 4u && p.streams[1].size() == 256u * 384u / 2u,
               "stream size law");
        expect(fpx::unpack(p) == q, "unpack(pack(q)) == q (acceptance 2)");
        const fpx::ScalarMatrix wq = fpx::dequantize_reference(q);
        expect(wq.dtype == fpx::Dtype::Fp16 && wq.rows == q.rows && wq.cols == q.cols, "dequantize_reference shape");
        const fpx::ScalarMatrix c_packed = fpx::gemm_packed(p, b);
        const fpx::ScalarMatrix c_ref = fpx::gemm_reference(q, b);
        expect(c_packed.rows == q.rows && c_packed.cols == n && c_packed.layout == fpx::Layout::ColMajor, "C shape");
        expect(c_packed.f32 == c_ref.f32, "gemm_packed == gemm_reference bit for bit (acceptance 3)");
        // C against an fp64 product of the bit-exact W (north-star tolerance per output vector)
        double worst = 0.0;
        for (uint32_t j = 0; j < n; ++j) {
            double err = 0.0, nrm = 0.0;
            for (uint32_t r = 0; r < q.rows; ++r) {
                double acc = 0.0;
                for (uint32_t k = 0; k < cols; ++k)
                    acc += double(fpx::half_to_float(wq.f16[size_t(r) * q.cols + k])) *
                           double(fpx::half_to_float(b.f16[size_t(j) * cols + k]));
                err = std::max(err, std::fabs(acc - double(c_packed.f32[size_t(j) * q.rows + r])));
                nrm = std::max(nrm, std::fabs(acc));
            }
            worst = std::max(worst, nrm > 0 ? err / nrm : err);
        }
        expect(worst <= 1e-2, "gemm within 1e-2 ||C[:,n]||inf (got " + std::to_string(worst) + ")");
        // ---- error behaviour (gemm.cpp:21-29, codec.cpp:105-110)
        expect_error(fpx::ErrorCode::ShapeMismatch,
                     [&] { fpx::gemm_packed(p, fpx::ScalarMatrix::zeros(fpx::Dtype::Fp16, fpx::Layout::ColMajor, 100, 2)); },
                     "gemm K mismatch");
        fpx::ScalarMatrix wnan = w;
        wnan.f32[7 * cols + 3] = std::nan("");
        expect_error(fpx::ErrorCode::InvalidValue, [&] { fpx::quantize_matrix(wnan, e3m2); }, "quantize NaN row");
        fpx::QuantizedMatrix qbad = q;
        qbad.codes[17] = 0x40;
        expect_error(fpx::ErrorCode::InvalidCode, [&] { fpx::dequantize_reference(qbad); }, "dequantize invalid code");
        // ---- io.hpp round trip
        expect(fpx::deserialize_packed(fpx::serialize_packed(p)) == p, "PackFile round trip");
        expect(std::memcmp(fpx::kPackMagic, "FPXPACK1", 8) == 0 && fpx::kPackVersion == 1, "io constants");

        if (argc > 1) {
            const std::string dir = argv[1];
            dump(dir, "w_f32.bin", w.f32);
            dump(dir, "b_f16.bin", b.f16);
            dump(dir, "codes.bin", q.codes);
            dump(dir, "scales.bin", q.scales);
            dump(dir, "stream0.bin", p.streams[0]);
            dump(dir, "stream1.bin", p.streams[1]);
            dump(dir, "wq_f16.bin", wq.f16);
            dump(dir, "c_f32.bin", c_packed.f32);
        }
    } catch (const fpx::Error& e) {
        std::printf("unexpected %s\n", e.formatted().c_str());
        return 1;
    } catch (const std::exception& e) {
        std::printf("%s\n", e.what());
        return 3;
    }
    std::printf(g_fail ? "ref-api caller: %d check(s) failed\n" : "ref-api caller: all checks passed\n", g_fail);
    return g_fail ? 1 : 0;
}
