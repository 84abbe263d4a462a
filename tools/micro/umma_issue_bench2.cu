// Micro-benchmark (bring-up only): where does the fixed per-round cost of
// issuing a batch of tcgen05.mma come from?  Variants of the issue loop.
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

// all lanes execute; one asm block elects a lane and issues R MMAs predicated
template <int R>
FPX_DEV void issue_pred(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, 1, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(a + k * 8), "l"(b + 2 * (k & 3)), "r"(idesc)
            : "memory");
    }
}

template <int R>
__global__ void bench(unsigned long long* out, int rounds, int variant) {
    __shared__ __align__(1024) uint8_t bsm[16384];
    __shared__ uint64_t bar3;
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) {
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
        constexpr uint32_t idesc = umma_idesc_f16(128, 16);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        unsigned long long t0 = clock64();
        if (variant == 0) {  // elect + branch
            for (int r = 0; r < rounds; ++r) {
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < R; ++k) umma_f16_ts(tmem + 256, tmem + k * 8, bdesc + 2 * (k & 3), idesc, 1u);
                }
                __syncwarp();
            }
        } else if (variant == 1) {  // predicated inside asm, warp stays converged
            for (int r = 0; r < rounds; ++r) issue_pred<R>(tmem + 256, tmem, bdesc, idesc);
        } else if (variant == 2) {  // lane 0 only, whole loop divergent
            if (lane == 0)
                for (int r = 0; r < rounds; ++r) {
#pragma unroll
                    for (int k = 0; k < R; ++k) umma_f16_ts(tmem + 256, tmem + k * 8, bdesc + 2 * (k & 3), idesc, 1u);
                }
            __syncwarp();
        } else {  // elect once outside the loop
            if (elect_one()) {
                for (int r = 0; r < rounds; ++r) {
#pragma unroll
                    for (int k = 0; k < R; ++k) umma_f16_ts(tmem + 256, tmem + k * 8, bdesc + 2 * (k & 3), idesc, 1u);
                }
            }
            __syncwarp();
        }
        unsigned long long t1 = clock64();
        if (elect_one()) umma_commit(&bar3);
        __syncwarp();
        mbar_wait(&bar3, 0);
        if (threadIdx.x == 32) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int R>
void run(unsigned long long* d) {
    const char* names[] = {"elect+branch", "pred-in-asm", "lane0-loop", "elect-outside"};
    for (int v = 0; v < 4; ++v) {
        const int rounds = 2000;
        bench<R><<<1, 64>>>(d, rounds, v);
        unsigned long long c = 0;
        if (cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
            printf("error\n");
            return;
        }
        printf("R=%2d %-14s %7.1f cycles/round %6.1f cycles/mma\n", R, names[v], double(c) / rounds,
               double(c) / rounds / R);
        fflush(stdout);
    }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    run<1>(d);
    run<4>(d);
    run<8>(d);
    run<16>(d);
    return 0;
}
