// fpx_sanitize_driver.cpp -- runs every device entry point of the C-ABI once
// at small shapes, for compute-sanitizer (memcheck / synccheck / racecheck)
// in tests/test_gpu_parity.py.  No torch, no Python: the sanitizer sees only
// libfpx_b200.so's kernels.  Exit 0 = every call returned FPX_OK and the
// outputs passed their self-checks, 1 otherwise.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "fpx_c.h"

#define CK(call)                                                                   \
    do {                                                                           \
        const int st_ = (call);                                                    \
        if (st_ != 0) {                                                            \
            std::printf("FAIL %s -> %d %s\n", #call, st_, fpx_last_error());       \
            return 1;                                                              \
        }                                                                          \
    } while (0)
#define CU(call)                                                                   \
    do {                                                                           \
        const cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) {                                                   \
            std::printf("FAIL %s -> %s\n", #call, cudaGetErrorString(e_));         \
            return 1;                                                              \
        }                                                                          \
    } while (0)

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(T) + 16) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, n * sizeof(T) + 16);
    return static_cast<T*>(p);
}

int main() {
    const uint32_t rows = 250, cols = 500, rp = 256, cp = 512;
    std::mt19937 rng(7);
    std::normal_distribution<float> nd(0.0f, 0.02f);
    std::vector<float> w(size_t(rows) * cols);
    for (float& v : w) v = nd(rng);
    float* d_w = dalloc<float>(w.size());
    CU(cudaMemcpy(d_w, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
    uint8_t* codes = dalloc<uint8_t>(size_t(rp) * cp);
    uint16_t* scales = dalloc<uint16_t>(rp);
    cudaStream_t s = nullptr;
    CU(cudaStreamCreate(&s));
    fpx_stream_t fs = reinterpret_cast<fpx_stream_t>(s);

    // K0 quantize, K1 prepack / unpack, K3 dequantize (packed + codes)
    CK(fpx_quantize(d_w, FPX_FP32, rows, cols, 3, 2, codes, scales, nullptr, fs));
    uint8_t* st[2] = {dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 2)), dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 4))};
    CK(fpx_prepack(codes, scales, rp, cp, 3, 2, nullptr, 0, st, fs));
    uint8_t* codes2 = dalloc<uint8_t>(size_t(rp) * cp);
    CK(fpx_unpack(st, rp, cp, 3, 2, nullptr, 0, codes2, fs));
    uint16_t* w16a = dalloc<uint16_t>(size_t(rp) * cp);
    uint16_t* w16b = dalloc<uint16_t>(size_t(rp) * cp);
    CK(fpx_dequantize(st, 2, nullptr, scales, rp, cp, 3, 2, w16a, fs));
    CK(fpx_dequantize_codes(codes, scales, rp, cp, 3, 2, w16b, nullptr, fs));
    // fused quantize + pack
    uint8_t* st2[2] = {dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 2)), dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 4))};
    uint16_t* scales2 = dalloc<uint16_t>(rp);
    CK(fpx_quantize_pack(d_w, FPX_FP32, rows, cols, 3, 2, nullptr, 0, st2, scales2, nullptr, fs));
    // e2m2 [4,1] and a LUT-path format (e4m3, [4,4])
    uint8_t* c5 = dalloc<uint8_t>(size_t(rp) * cp);
    uint16_t* s5 = dalloc<uint16_t>(rp);
    CK(fpx_quantize(d_w, FPX_FP32, rows, cols, 2, 2, c5, s5, nullptr, fs));
    uint8_t* st5[2] = {dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 4)), dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 1))};
    CK(fpx_prepack(c5, s5, rp, cp, 2, 2, nullptr, 0, st5, fs));
    uint8_t* c8 = dalloc<uint8_t>(size_t(rp) * cp);
    uint16_t* s8 = dalloc<uint16_t>(rp);
    CK(fpx_quantize(d_w, FPX_FP32, rows, cols, 4, 3, c8, s8, nullptr, fs));
    uint8_t* st8[2] = {dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 4)), dalloc<uint8_t>(fpx_stream_bytes(rp, cp, 4))};
    CK(fpx_prepack(c8, s8, rp, cp, 4, 3, nullptr, 0, st8, fs));
    CK(fpx_dequantize(st8, 2, nullptr, s8, rp, cp, 4, 3, w16b, fs));

    // K2: decode kernel (N <= 128) at several widths and splits, the
    // single-issuer kernel (N > 128), ragged K (staged), fused epilogue.
    const uint32_t nmax = 200;
    std::vector<uint16_t> act(size_t(nmax) * cp);
    std::uniform_int_distribution<uint32_t> ub(0, 0xffffu);
    for (auto& v : act) {  // fp16 patterns of magnitude [2^-3, 2^1): sign | exponent 12..15 | mantissa
        const uint32_t r = ub(rng);
        v = static_cast<uint16_t>((r & 0x8000u) | ((12u + (r >> 10) % 4u) << 10) | (r & 0x3ffu));
    }
    uint16_t* d_act = dalloc<uint16_t>(act.size());
    CU(cudaMemcpy(d_act, act.data(), act.size() * 2, cudaMemcpyHostToDevice));
    float* c = dalloc<float>(size_t(nmax) * rp);
    const size_t ws_bytes = 64u << 20;
    void* ws = dalloc<uint8_t>(ws_bytes);
    for (uint32_t n : {1u, 16u, 32u, 64u, 128u, 200u})
        for (int split : {1, 3}) {
            CK(fpx_linear(st, 2, scales, rp, cp, 3, 2, d_act, cp, n, c, rp, split, ws, ws_bytes, fs));
            CK(fpx_linear(st5, 2, s5, rp, cp, 2, 2, d_act, cp, n, c, rp, split, ws, ws_bytes, fs));
        }
    CK(fpx_linear(st, 2, scales, rp, cp, 3, 2, d_act, cols, 24, c, rp, 0, ws, ws_bytes, fs));  // K_act < K_p
    float* bias = dalloc<float>(rp);
    uint16_t* resid = dalloc<uint16_t>(size_t(16) * rp);
    fpx_epilogue epi{FPX_FP16, bias, FPX_ACT_SILU, resid};
    CK(fpx_linear_ex(st, 2, scales, rp, cp, 3, 2, d_act, cp, 16, c, rp, 2, &epi, ws, ws_bytes, fs));
    CK(fpx_linear_workspace_reset(ws, ws_bytes, fs));

    // multi-GPU helpers on one device: 1-rank sharded call, gather permute
    const size_t sws = fpx_linear_sharded_workspace_size(rp, cp, cp, 8, 1, 0);
    void* sw = dalloc<uint8_t>(sws);
    CK(fpx_linear_sharded(st, 2, scales, rp, cp, 3, 2, d_act, cp, 8, c, rp, 0, 0, 1, nullptr, sw, sws, fs));
    uint32_t h_row0[2] = {0, 128}, h_nrows[2] = {128, 128};
    uint32_t* row0 = dalloc<uint32_t>(2);
    uint32_t* nrows = dalloc<uint32_t>(2);
    CU(cudaMemcpy(row0, h_row0, 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(nrows, h_nrows, 8, cudaMemcpyHostToDevice));
    float* gathered = dalloc<float>(size_t(2) * 8 * 128);
    CK(fpx_gather_permute(gathered, row0, nrows, 2, 128, 8, c, rp, fs));
    CU(cudaStreamSynchronize(s));

    // self-checks: unpack == codes, the two de-quantisers agree
    std::vector<uint8_t> h1(size_t(rp) * cp), h2(h1.size());
    CU(cudaMemcpy(h1.data(), codes, h1.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(h2.data(), codes2, h2.size(), cudaMemcpyDeviceToHost));
    if (h1 != h2) {
        std::printf("FAIL unpack(pack(q)) != q\n");
        return 1;
    }
    CK(fpx_dequantize(st, 2, nullptr, scales, rp, cp, 3, 2, w16a, fs));
    CK(fpx_dequantize_codes(codes, scales, rp, cp, 3, 2, w16b, nullptr, fs));
    std::vector<uint16_t> a(size_t(rp) * cp), b(a.size());
    CU(cudaMemcpy(a.data(), w16a, a.size() * 2, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(b.data(), w16b, b.size() * 2, cudaMemcpyDeviceToHost));
    if (a != b) {
        std::printf("FAIL dequantize(packed) != dequantize_codes\n");
        return 1;
    }
    std::printf("sanitize driver ok\n");
    return 0;
}
