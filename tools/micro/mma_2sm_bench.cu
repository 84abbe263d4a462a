// Micro-benchmark (bring-up only): is the ~44-cycle per-instruction cost of
// a small-N kind::f16 tcgen05.mma paid per instruction or per SM?  Compares
// cta_group::1 (M=128 per SM) with cta_group::2 (M=256 across an SM pair:
// one instruction issued by the pair's leader covers 2 x 128 rows).
// A from TMEM (TS), N=32, K=16, R MMAs per commit, 4 commit groups in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o mma_2sm_bench mma_2sm_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

template <int CG, int N, int R>
__global__ void __launch_bounds__(64, 1) bench(unsigned long long* out, int rounds) {
    __shared__ __align__(1024) uint8_t bsm[16384];
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    if (threadIdx.x == 32) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
    fence_proxy_async();
    if (warp == 0) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            tmem_alloc<512>(&tslot);
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    unsigned long long cyc = 0;
    if (warp == 0 && rank == 0) {
        constexpr uint32_t idesc = umma_idesc_f16(128 * CG, N);
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        unsigned long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (r >= 4) mbar_wait(&bar[r & 3], ((r >> 2) - 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const uint32_t a = tmem + (k & 3) * 8, d = tmem + 256;
                    const uint64_t b = bdesc + 2 * (k & 3);
                    if constexpr (CG == 2) {
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                            "r"(a), "l"(b), "r"(idesc), "r"(1u)
                            : "memory");
                    } else {
                        umma_f16_ts(d, a, b, idesc, 1u);
                    }
                }
                if constexpr (CG == 2) {
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            smem_u32(&bar[r & 3]))
                        : "memory");
                } else {
                    umma_commit(&bar[r & 3]);
                }
            }
            __syncwarp();
        }
        for (int r = rounds - 4; r < rounds; ++r) mbar_wait(&bar[r & 3], (r >> 2) & 1);
        cyc = clock64() - t0;
        if (threadIdx.x == 0) out[blockIdx.x] = cyc;
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    if (warp == 0) {
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else
            tmem_dealloc<512>(tmem);
    }
}

template <int CG, int N, int R>
void run(unsigned long long* d) {
    const int rounds = 512;
    cudaMemset(d, 0, 148 * 8);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(64);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, bench<CG, N, R>, d, rounds);
    unsigned long long h[148];
    if (e != cudaSuccess || cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        exit(1);
    }
    double c = 0;
    int cnt = 0;
    for (int b = 0; b < 148; ++b)
        if (h[b]) c += h[b], ++cnt;
    c /= cnt;
    const double per = c / rounds / R;
    printf("cta_group::%d M=%3d N=%3d R=%2d : %6.1f cycles/instr, %5.1f weights(MxK)/clk per SM (%d issuing CTAs)\n", CG,
           128 * CG, N, R, per, 128.0 * 16 / per, cnt);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<1, 32, 32>(d);
    run<2, 32, 32>(d);
    run<1, 32, 8>(d);
    run<2, 32, 8>(d);
    run<2, 64, 32>(d);
    run<2, 256, 32>(d);
    return 0;
}
