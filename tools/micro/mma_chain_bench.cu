// Micro-benchmark (bring-up only): throughput of tcgen05.mma kind::f16 with A
// from TMEM (M=128, K=16) as a function of N and of how many INDEPENDENT
// accumulators the issue stream rotates over.  MMAs into the same
// accumulator are a dependency chain; rounds of 8 MMAs, commit per round,
// 2 rounds in flight.  One CTA per SM on all 148 SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o mma_chain_bench mma_chain_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

template <int N, int NACC>
__global__ void __launch_bounds__(64, 1) bench(unsigned long long* out, int rounds) {
    __shared__ __align__(1024) uint8_t bsm[32768];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        constexpr uint32_t idesc = umma_idesc_f16(128, N);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        unsigned long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (r >= 2) mbar_wait(&bar[r & 1], ((r >> 1) - 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma_f16_ts(tmem + 64 + (k % NACC) * N, tmem + (k & 3) * 8, bdesc + 2 * (k & 3), idesc, 1u);
                umma_commit(&bar[r & 1]);
            }
            __syncwarp();
        }
        mbar_wait(&bar[(rounds - 2) & 1], ((rounds - 2) >> 1) & 1);
        mbar_wait(&bar[(rounds - 1) & 1], ((rounds - 1) >> 1) & 1);
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, int NACC>
void run(unsigned long long* d) {
    unsigned long long h[148];
    const int rounds = 2000;
    bench<N, NACC><<<148, 64>>>(d, rounds);
    if (cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        return;
    }
    double c = 0;
    for (int b = 0; b < 148; ++b) c += h[b];
    c /= 148;
    printf("N=%3d accumulators=%d : %6.1f cycles/MMA  (%5.1f MAC/clk/SM x1e3)\n", N, NACC, c / rounds / 8,
           128.0 * N * 16 / (c / rounds / 8) / 1e3);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<16, 1>(d);
    run<16, 2>(d);
    run<16, 4>(d);
    run<16, 8>(d);
    run<32, 1>(d);
    run<32, 2>(d);
    run<32, 4>(d);
    run<32, 8>(d);
    run<64, 1>(d);
    run<64, 4>(d);
    run<128, 1>(d);
    run<128, 2>(d);
    run<256, 1>(d);
    return 0;
}
