// Micro-benchmark (bring-up only): does tcgen05.st traffic from many warps
// slow down tcgen05.mma issue/execution (A from TMEM, M=128, N=16) on the
// same SM?  One CTA per SM, 148 CTAs.
//   warp 0      : MMA issuer, R rounds of 8 MMAs + commit (waits the round two back)
//   warps 1..16 : optional tcgen05.st 16x128b.x8 x2 + wait::st loops into
//                 disjoint TMEM columns (the de-quantisers' store pattern)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o tmem_contention_bench tmem_contention_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

__global__ void __launch_bounds__(17 * 32, 1) bench(unsigned long long* out, int rounds, int mode, int st_iters) {
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
    unsigned long long t0 = clock64();
    if (warp == 0 && (mode & 1)) {
        constexpr uint32_t idesc = umma_idesc_f16(128, 16);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        for (int r = 0; r < rounds; ++r) {
            if (r >= 2) mbar_wait(&bar[r & 1], ((r >> 1) - 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma_f16_ts(tmem + 256 + (r & 3) * 16, tmem + k * 8, bdesc + 2 * (k & 3), idesc, k ? 1u : 0u);
                umma_commit(&bar[r & 1]);
            }
            __syncwarp();
        }
        if (rounds >= 2) {
            mbar_wait(&bar[(rounds - 2) & 1], ((rounds - 2) >> 1) & 1);
            mbar_wait(&bar[(rounds - 1) & 1], ((rounds - 1) >> 1) & 1);
        }
        if (threadIdx.x == 0) out[blockIdx.x * 2 + 0] = clock64() - t0;
    } else if (warp >= 1 && (mode & 2)) {
        const uint32_t q = warp & 3u;
        const uint32_t col = 64 + ((warp - 1) / 4) * 32;  // 4 groups x 32 columns at 64..191
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0x3c003c00u + i;
        for (int it = 0; it < st_iters; ++it) {
            tmem_st_16x128b_x8(tmem + ((32 * q) << 16) + col, v);
            tmem_st_16x128b_x8(tmem + ((32 * q) << 16) + col + (16u << 16), v);
            tmem_st_wait();
            v[0] += 1;
        }
        if ((threadIdx.x & 31) == 0 && warp == 1) out[blockIdx.x * 2 + 1] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 2 * 8);
    unsigned long long h[296];
    const int rounds = 4000, st_iters = 4000;
    const char* names[] = {"", "MMA alone", "STTM alone", "MMA + STTM"};
    for (int mode = 1; mode <= 3; ++mode) {
        cudaMemset(d, 0, sizeof(h));
        bench<<<148, 17 * 32>>>(d, rounds, mode, st_iters);
        if (cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
        double mma = 0, st = 0;
        for (int b = 0; b < 148; ++b) mma += h[2 * b], st += h[2 * b + 1];
        mma /= 148, st /= 148;
        printf("%-12s: MMA %7.1f cycles/round of 8 (%5.1f /MMA) | STTM pair+wait %7.1f cycles/iter per warp\n",
               names[mode], mma / rounds, mma / rounds / 8, st / st_iters);
    }
    return 0;
}
