// Micro-benchmark (bring-up only): back-to-back launch cost (CUDA graph of
// 30 launches) of an EMPTY persistent kernel shaped like the decode kernel
// (148 CTAs x 736 threads, ~200 KB dynamic smem, TMEM alloc/dealloc,
// mbarrier init), vs a trivial kernel, vs with a 20 us busy loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o launch_bench launch_bench.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

__global__ void trivial(int* p) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p == nullptr) printf("x");
}

template <bool kTmem>
__global__ void __launch_bounds__(736, 1) shaped(unsigned long long spin_ns) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 200 * 1024);
    const uint32_t warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 60; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (kTmem && warp == 22) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (spin_ns && threadIdx.x == 0) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        unsigned long long t = t0;
        while (t - t0 < spin_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    }
    tc_fence_before();
    __syncthreads();
    if (kTmem && warp == 22) {
        tc_fence_after();
        tmem_dealloc<512>(tslot);
    }
}

template <typename F>
float graph_us(F launch, int n = 30) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    launch(s);
    cudaStreamSynchronize(s);
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) launch(s);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000 / n;
}

int main() {
    const int smem = 200 * 1024 + 60 * 8;
    cudaFuncSetAttribute(shaped<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(shaped<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    printf("trivial 148x32             : %6.2f us/launch\n", graph_us([](cudaStream_t s) { trivial<<<148, 32, 0, s>>>(nullptr); }));
    printf("shaped, no TMEM, empty     : %6.2f us/launch\n",
           graph_us([&](cudaStream_t s) { shaped<false><<<148, 736, smem, s>>>(0); }));
    printf("shaped, TMEM, empty        : %6.2f us/launch\n",
           graph_us([&](cudaStream_t s) { shaped<true><<<148, 736, smem, s>>>(0); }));
    printf("shaped, TMEM, 20 us spin   : %6.2f us/launch\n",
           graph_us([&](cudaStream_t s) { shaped<true><<<148, 736, smem, s>>>(20000); }));
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
