// Micro-benchmark (bring-up only): separates tcgen05.mma throughput from
// tcgen05.commit cost and commit->mbarrier latency (TS, M=128, N=16, K=16).
//   (a) T MMAs, one commit at the end          -> MMA throughput
//   (b) T MMAs, a commit every R (never waited) -> added cost of a commit
//   (c) R MMAs + commit, wait, repeated         -> round latency
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o mma_commit_bench mma_commit_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

__global__ void __launch_bounds__(64, 1) bench(unsigned long long* out, int mode, int T, int R) {
    __shared__ __align__(1024) uint8_t bsm[16384];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        constexpr uint32_t idesc = umma_idesc_f16(128, 16);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        unsigned long long t0 = clock64();
        if (mode == 0 || mode == 1) {
            for (int i = 0; i < T; i += 4) {
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_f16_ts(tmem + 256 + ((i >> 2) & 7) * 16, tmem + k * 8, bdesc + 2 * k, idesc, 1u);
                    if (mode == 1 && ((i + 4) % R) == 0) umma_commit(&bar[1]);
                }
                __syncwarp();
            }
            if (threadIdx.x == 0) umma_commit(&bar[0]);
            __syncwarp();
            mbar_wait(&bar[0], 0);
        } else {
            uint32_t ph = 0;
            for (int i = 0; i < T; i += R, ph ^= 1) {
                if (threadIdx.x == 0) {
                    for (int k = 0; k < R; ++k)
                        umma_f16_ts(tmem + 256, tmem + (k & 3) * 8, bdesc + 2 * (k & 3), idesc, 1u);
                    umma_commit(&bar[0]);
                }
                __syncwarp();
                mbar_wait(&bar[0], ph);
            }
        }
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

void run(unsigned long long* d, int mode, int T, int R) {
    unsigned long long h[148];
    bench<<<148, 64>>>(d, mode, T, R);
    if (cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        exit(1);
    }
    double c = 0;
    for (int b = 0; b < 148; ++b) c += h[b];
    c /= 148;
    const char* names[] = {"(a) no commits      ", "(b) commit every R  ", "(c) R + commit + wait"};
    printf("%s T=%5d R=%3d : %8.0f cycles total, %6.1f cycles/MMA, %7.1f cycles/round\n", names[mode], T, R, c, c / T,
           c / T * R);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run(d, 0, 4096, 4);
    run(d, 0, 16384, 4);
    for (int R : {4, 8, 16, 32}) run(d, 1, 4096, R);
    for (int R : {1, 4, 8, 16, 32, 64}) run(d, 2, 2048, R);
    return 0;
}
