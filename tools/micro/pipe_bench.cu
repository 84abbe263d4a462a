// Micro-benchmark (bring-up only): which issue pipe does each instruction of
// the de-quantisation inner loop use, and at what rate?  Each kernel runs 8
// independent dependency chains per thread of one instruction mix over a
// full-occupancy grid; rate = thread-instructions / SM / clock (SM clock
// measured with clock64 inside the kernel).  Mixes that share a pipe add
// their times; mixes on different pipes overlap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t f2fp(uint32_t x) {
    uint32_t d;
    asm volatile("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.rn.f16x2.e3m2x2 %0, l;\n\t}" : "=r"(d) : "r"(x));
    return d;
}
__device__ __forceinline__ uint32_t f2fp_hi(uint32_t x) {
    uint32_t d;
    asm volatile("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.rn.f16x2.e3m2x2 %0, h;\n\t}" : "=r"(d) : "r"(x));
    return d;
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0xe8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t shf(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("shf.r.wrap.b32 %0, %1, %2, 3;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("prmt.b32 %0, %1, %2, 0x2031;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, 4, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ uint32_t imadhi(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// mix: bit0 F2FP, bit1 LOP3, bit2 SHF, bit3 PRMT, bit4 HMUL2, bit5 IMAD, bit6 IMAD.HI
template <int MIX>
__global__ void pipe_kernel(const uint32_t* in, uint32_t* out, int iters, unsigned long long* clk) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = in[(threadIdx.x + i) & 1023];
    const uint32_t k = in[1000];
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MIX & 1) v[i] = f2fp(v[i]);
            if (MIX & 2) v[i] = lop3(v[i], k, v[(i + 1) & 7]);
            if (MIX & 4) v[i] = shf(v[i], k);
            if (MIX & 8) v[i] = prmt(v[i], k);
            if (MIX & 16) v[i] = hmul2(v[i], k);
            if (MIX & 32) v[i] = imad(v[i], k);
            if (MIX & 64) v[i] = imadhi(v[i], k | 0x40000000u);
        }
    }
    unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

template <int MIX>
void run(const char* name, const uint32_t* in, uint32_t* out, unsigned long long* clk) {
    const int iters = 4000, ctas = 148 * 4, threads = 512;
    pipe_kernel<MIX><<<ctas, threads>>>(in, out, iters, clk);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    pipe_kernel<MIX><<<ctas, threads>>>(in, out, iters, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const int nops = __builtin_popcount(MIX);
    const double thread_insts = double(ctas) * threads * iters * 8 * nops;
    const double ghz = double(c) / (ms * 1e6);  // one CTA's clock span over the launch time (approx.)
    const double per_sm_clk = thread_insts / 148 / (ms * 1e-3 * ghz * 1e9);
    printf("%-22s %7.3f ms  clk~%.2f GHz  %6.1f thread-inst/clk/SM (%5.2f warp-inst/clk/SM) = %5.1f per instr kind\n",
           name, ms, ghz, per_sm_clk, per_sm_clk / 32, per_sm_clk / nops);
}

int main() {
    uint32_t *in, *out;
    unsigned long long* clk;
    cudaMalloc(&in, 4096 * 4);
    cudaMemset(in, 0x1b, 4096 * 4);
    cudaMalloc(&out, 148 * 4 * 512 * 4);
    cudaMalloc(&clk, 8);
    run<1>("F2FP", in, out, clk);
    run<2>("LOP3", in, out, clk);
    run<4>("SHF", in, out, clk);
    run<8>("PRMT", in, out, clk);
    run<16>("HMUL2", in, out, clk);
    run<32>("IMAD", in, out, clk);
    run<1 | 2>("F2FP+LOP3", in, out, clk);
    run<1 | 16>("F2FP+HMUL2", in, out, clk);
    run<1 | 32>("F2FP+IMAD", in, out, clk);
    run<2 | 16>("LOP3+HMUL2", in, out, clk);
    run<2 | 32>("LOP3+IMAD", in, out, clk);
    run<1 | 2 | 16>("F2FP+LOP3+HMUL2", in, out, clk);
    run<1 | 8 | 16>("F2FP+PRMT+HMUL2", in, out, clk);
    run<2 | 4 | 8>("LOP3+SHF+PRMT", in, out, clk);
    run<64>("IMAD.HI", in, out, clk);
    run<2 | 64>("LOP3+IMAD.HI", in, out, clk);
    run<1 | 64>("F2FP+IMAD.HI", in, out, clk);
    run<1 | 2 | 16 | 32>("F2FP+LOP3+HMUL2+IMAD", in, out, clk);
    run<1 | 2 | 16 | 64>("F2FP+LOP3+HMUL2+IMADHI", in, out, clk);
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
