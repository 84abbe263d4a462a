// Micro-benchmark (bring-up only, not part of the product): semantics and
// throughput of the sm_100a FP6 -> f16x2 converts vs the SWAR ALU path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f2fp_bench f2fp_bench.cu
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t cvt_e3m2x2(uint16_t v) {
    uint32_t d;
    asm("cvt.rn.f16x2.e3m2x2 %0, %1;" : "=r"(d) : "h"(v));
    return d;
}
__device__ __forceinline__ uint32_t cvt_e2m3x2(uint16_t v) {
    uint32_t d;
    asm("cvt.rn.f16x2.e2m3x2 %0, %1;" : "=r"(d) : "h"(v));
    return d;
}

__global__ void sem_kernel(uint32_t* out3, uint32_t* out2) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 65536) {
        out3[i] = cvt_e3m2x2(static_cast<uint16_t>(i));
        out2[i] = cvt_e2m3x2(static_cast<uint16_t>(i));
    }
}

// Throughput: each thread converts many independent words.
__global__ void tput_cvt(const uint32_t* in, uint32_t* out, int iters) {
    uint32_t x0 = in[threadIdx.x], x1 = in[threadIdx.x + 1], x2 = in[threadIdx.x + 2], x3 = in[threadIdx.x + 3];
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc0 ^= cvt_e3m2x2(static_cast<uint16_t>(x0 >> u));
            acc1 ^= cvt_e3m2x2(static_cast<uint16_t>(x1 >> u));
            acc2 ^= cvt_e3m2x2(static_cast<uint16_t>(x2 >> u));
            acc3 ^= cvt_e3m2x2(static_cast<uint16_t>(x3 >> u));
        }
        x0 += 0x01010101u, x1 += 0x03030303u, x2 += 0x05050505u, x3 += 0x07070707u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
}

// Same loop with the ALU ops of the shifted source only (baseline overhead).
__global__ void tput_lop(const uint32_t* in, uint32_t* out, int iters) {
    uint32_t x0 = in[threadIdx.x], x1 = in[threadIdx.x + 1], x2 = in[threadIdx.x + 2], x3 = in[threadIdx.x + 3];
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc0 ^= (x0 >> u) & 0x3f3f;
            acc1 ^= (x1 >> u) & 0x3f3f;
            acc2 ^= (x2 >> u) & 0x3f3f;
            acc3 ^= (x3 >> u) & 0x3f3f;
        }
        x0 += 0x01010101u, x1 += 0x03030303u, x2 += 0x05050505u, x3 += 0x07070707u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
}

static float h2f(uint16_t h) {
    __half x;
    memcpy(&x, &h, 2);
    return __half2float(x);
}

static double decode(uint32_t c, int e, int m) {
    int bias = (1 << (e - 1)) - 1;
    uint32_t s = (c >> (e + m)) & 1, ef = (c >> m) & ((1 << e) - 1), mf = c & ((1 << m) - 1);
    double v = ef == 0 ? ldexp(double(mf), 1 - bias - m) : ldexp(double((1 << m) | mf), int(ef) - bias - m);
    return s ? -v : v;
}

int main() {
    uint32_t *d3, *d2;
    cudaMalloc(&d3, 65536 * 4);
    cudaMalloc(&d2, 65536 * 4);
    sem_kernel<<<256, 256>>>(d3, d2);
    std::vector<uint32_t> h3(65536), h2(65536);
    cudaMemcpy(h3.data(), d3, 65536 * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), d2, 65536 * 4, cudaMemcpyDeviceToHost);
    int bad3 = 0, bad2 = 0, bad3_clean = 0, bad2_clean = 0;
    for (uint32_t i = 0; i < 65536; ++i) {
        const uint32_t lo = i & 0x3f, hi = (i >> 8) & 0x3f;
        const bool clean = (i & 0xc0c0) == 0;
        const double e_lo3 = decode(lo, 3, 2), e_hi3 = decode(hi, 3, 2);
        const double e_lo2 = decode(lo, 2, 3), e_hi2 = decode(hi, 2, 3);
        const bool ok3 = h2f(h3[i] & 0xffff) == e_lo3 && h2f(h3[i] >> 16) == e_hi3 &&
                         (std::signbit(h2f(h3[i] & 0xffff)) == std::signbit(e_lo3));
        const bool ok2 = h2f(h2[i] & 0xffff) == e_lo2 && h2f(h2[i] >> 16) == e_hi2;
        if (!ok3) { bad3++; if (clean) bad3_clean++; }
        if (!ok2) { bad2++; if (clean) bad2_clean++; }
        if (i == 0x0c0c || i == 0x2c2c || i == 0xcc0c)
            printf("in %04x -> e3m2 %08x (%g %g)  e2m3 %08x\n", i, h3[i], h2f(h3[i] & 0xffff), h2f(h3[i] >> 16), h2[i]);
    }
    printf("e3m2x2: mismatches %d (clean-top-bits inputs: %d)\n", bad3, bad3_clean);
    printf("e2m3x2: mismatches %d (clean-top-bits inputs: %d)\n", bad2, bad2_clean);

    uint32_t *in, *out;
    cudaMalloc(&in, 4096 * 4);
    cudaMemset(in, 0x5a, 4096 * 4);
    cudaMalloc(&out, 148 * 4 * 1024 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        for (int which = 0; which < 2; ++which) {
            cudaEventRecord(a);
            if (which == 0) tput_cvt<<<148 * 4, 512>>>(in, out, iters);
            else tput_lop<<<148 * 4, 512>>>(in, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double ops = 148.0 * 4 * 512 * iters * 32;  // converts (or and-shift pairs)
            printf("%s: %.3f ms, %.1f Gop/s, %.2f ops/clk/SM @1.9GHz\n", which ? "shift+and" : "cvt e3m2x2", ms,
                   ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.9e9);
        }
    }
    return 0;
}
