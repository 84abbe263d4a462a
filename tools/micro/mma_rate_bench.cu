// Micro-benchmark (bring-up only): sustained tcgen05.mma kind::f16 rate for
// small N, A from TMEM (TS) vs A from shared memory (SS), M = 64 / 128,
// with R MMAs per commit and up to 4 commit groups in flight.  One CTA per
// SM on all 148 SMs; cycles per MMA averaged over CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o mma_rate_bench mma_rate_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

template <int M, int N, bool TS, int R, int NACC = 1, int INF = 4>
__global__ void __launch_bounds__(64, 1) bench(unsigned long long* out, int rounds) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* bsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[16];
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) {
        for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        constexpr uint32_t idesc = umma_idesc_f16(M, N);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        const uint64_t adesc = umma_desc_sw128_kmajor(smem_u32(bsm + 32768));
        unsigned long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (r >= INF) mbar_wait(&bar[r % INF], ((r / INF) - 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    if constexpr (TS)
                        umma_f16_ts(tmem + 256 + (k % NACC) * N, tmem + (k & 3) * 8, bdesc + 2 * (k & 3), idesc, 1u);
                    else
                        umma_f16_ss(tmem + 256 + (k % NACC) * N, adesc + 2 * (k & 3), bdesc + 2 * (k & 3), idesc, 1u);
                }
                umma_commit(&bar[r % INF]);
            }
            __syncwarp();
        }
        for (int r = rounds - INF; r < rounds; ++r) mbar_wait(&bar[r % INF], (r / INF) & 1);
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int M, int N, bool TS, int R, int NACC = 1, int INF = 4>
void run(unsigned long long* d) {
    unsigned long long h[148];
    const int rounds = 512;
    cudaFuncSetAttribute(bench<M, N, TS, R, NACC, INF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50176);
    bench<M, N, TS, R, NACC, INF><<<148, 64, 50176>>>(d, rounds);
    if (cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        exit(1);
    }
    double c = 0;
    for (int b = 0; b < 148; ++b) c += h[b];
    c /= 148;
    const double per = c / rounds / R;
    printf("%s M=%3d N=%3d R=%2d acc=%d inflight=%2d : %6.1f cycles/MMA  -> %5.1f weights(MxK)/clk/SM\n", TS ? "TS" : "SS", M, N, R, NACC, INF, per,
           M * 16.0 / per);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<128, 16, true, 8, 1, 2>(d);
    run<128, 16, true, 8, 1, 4>(d);
    run<128, 16, true, 8, 1, 8>(d);
    run<128, 16, true, 8, 1, 16>(d);
    run<128, 16, true, 24, 1, 4>(d);
    run<128, 16, true, 24, 1, 8>(d);
    run<128, 16, true, 64, 1, 4>(d);
    run<128, 16, true, 64, 1, 8>(d);
    return 0;
}
