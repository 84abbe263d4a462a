// fpx_cpp_selftest -- exercises the C++ drop-in (include/fpx_b200.hpp) the way
// a caller of the reference library would: quantize -> pack -> gemm_packed,
// plus unpack / dequantize, checking shapes, the round trip and C against a
// host fp64 dot product of the device-dequantised weights.
// Exit: 0 ok, 1 mismatch, 3 fpx::Error / DeviceError (message on stdout).
#include <cmath>
#include <cstdio>
#include <random>

#include "fpx_b200.hpp"

static double h2d(uint16_t h) {
    const int e = (h >> 10) & 31, m = h & 1023;
    const double v = e == 0 ? std::ldexp(double(m), -24) : std::ldexp(double(1024 + m), e - 25);
    return (h & 0x8000) ? -v : v;
}

int main() {
    try {
        std::mt19937 rng(7);
        std::normal_distribution<float> nd(0.0f, 0.02f);
        const uint32_t rows = 200, cols = 300, n = 5;
        fpx::ScalarMatrix w = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp32, fpx::Layout::RowMajor, rows, cols);
        for (float& x : w.f32) x = nd(rng);
        const fpx::QuantizedMatrix q = fpx::quantize_matrix(w, fpx::FpxFormat::e3m2());
        const fpx::PackedWeights p = fpx::pack(q);
        if (p.rows != 256 || p.cols != 320 || p.streams.size() != 2 || p.streams[0].size() != 256 * 320 * 2 / 8) {
            std::printf("bad packed shape\n");
            return 1;
        }
        if (!(fpx::unpack(p) == q)) {
            std::printf("unpack(pack(q)) != q\n");
            return 1;
        }
        const fpx::ScalarMatrix wd = fpx::dequantize(p);
        fpx::ScalarMatrix b = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp32, fpx::Layout::ColMajor, cols, n);
        std::normal_distribution<float> na(0.0f, 1.0f);
        for (float& x : b.f32) x = na(rng);
        const fpx::ScalarMatrix c = fpx::gemm_packed(p, fpx::to_fp16(b));
        const fpx::ScalarMatrix b16 = fpx::to_fp16(b);
        double worst = 0.0;
        for (uint32_t j = 0; j < n; ++j) {
            double nrm = 0.0, err = 0.0;
            for (uint32_t r = 0; r < p.rows; ++r) {
                double ref = 0.0;
                for (uint32_t k = 0; k < cols; ++k) ref += h2d(wd.f16[size_t(r) * p.cols + k]) * h2d(b16.f16[size_t(j) * cols + k]);
                nrm = std::fmax(nrm, std::fabs(ref));
                err = std::fmax(err, std::fabs(ref - c.f32[size_t(j) * p.rows + r]));
            }
            worst = std::fmax(worst, err / nrm);
        }
        std::printf("fpx_cpp_selftest: rows %u cols %u n %u max rel err %.3g\n", rows, cols, n, worst);
        try {
            fpx::ScalarMatrix bad = fpx::ScalarMatrix::zeros(fpx::Dtype::Fp16, fpx::Layout::ColMajor, 100, 2);
            fpx::gemm_packed(p, bad);
            std::printf("shape error not raised\n");
            return 1;
        } catch (const fpx::Error& e) {
            std::printf("expected: %s\n", e.formatted().c_str());
        }
        return worst < 1e-3 ? 0 : 1;
    } catch (const fpx::Error& e) {
        std::printf("%s\n", e.formatted().c_str());
        return 3;
    } catch (const fpx::DeviceError& e) {
        std::printf("%s\n", e.what());
        return 3;
    }
}
