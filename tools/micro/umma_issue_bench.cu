// Micro-benchmark (bring-up only): issue cost of tcgen05.mma (A from TMEM,
// M=128, kind::f16) and tcgen05.commit + mbarrier round trip on one SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o umma_issue_bench umma_issue_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

template <int N>
__global__ void bench(unsigned long long* out, int rounds, int mmas_per_round, int mode) {
    __shared__ __align__(1024) uint8_t bsm[16384];
    __shared__ uint64_t bar, bar2, bar3;
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        mbar_init(&bar3, 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1) {
        constexpr uint32_t idesc = umma_idesc_f16(128, N);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        uint32_t phase = 0;
        unsigned long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (elect_one()) {
                for (int k = 0; k < mmas_per_round; ++k)
                    umma_f16_ts(tmem + 256, tmem + (k & 7) * 8, bdesc + (k & 3) * 2, idesc, 1u);
                if (mode == 1) umma_commit(&bar2);
                if (mode == 2) umma_commit(&bar);
            }
            __syncwarp();
            if (mode == 2) {
                mbar_wait(&bar, phase);
                phase ^= 1;
                tc_fence_after();
            }
        }
        unsigned long long t1 = clock64();
        if (elect_one()) umma_commit(&bar3);  // drain everything issued
        __syncwarp();
        mbar_wait(&bar3, 0);
        if (threadIdx.x == 32) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const char* names[] = {"issue only", "issue+commit", "issue+commit+wait"};
    for (int mode = 0; mode < 3; ++mode)
        for (int m : {1, 4, 8, 16}) {
            const int rounds = 2000;
            bench<16><<<1, 64>>>(d, rounds, m, mode);
            unsigned long long c = 0;
            cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                printf("err %s\n", cudaGetErrorString(e));
                return 1;
            }
            fflush(stdout);
            printf("N=16 %-18s mmas/round=%2d : %7.1f cycles/round, %6.1f cycles/mma\n", names[mode], m,
                   double(c) / rounds, double(c) / rounds / m);
        }
    for (int m : {8}) {
        bench<32><<<1, 64>>>(d, 2000, m, 2);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("N=32 issue+commit+wait mmas/round=%d : %.1f cycles/round\n", m, double(c) / 2000);
        bench<128><<<1, 64>>>(d, 2000, m, 2);
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("N=128 issue+commit+wait mmas/round=%d : %.1f cycles/round\n", m, double(c) / 2000);
    }
    return 0;
}
