// Micro-benchmark (bring-up only): per-operation cost of the pipeline sync
// primitives in a single thread (cycles per op, 4096 iterations).
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

template <int op>
__global__ void bench(unsigned long long* out, unsigned long long* gbuf) {
    __shared__ uint64_t bars[64];
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<32>(&tslot);
    if (threadIdx.x == 32) {
        for (int i = 0; i < 64; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int iters = 4096;
    if (warp == 1 && elect_one()) {
        // complete phase 0 of every barrier for the "wait on completed" test
        if (op == 0) for (int i = 0; i < 64; ++i) mbar_arrive(&bars[i]);
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            uint64_t* b = &bars[i & 63];
            if constexpr (op == 0) mbar_wait(b, 0);                  // wait, already complete
            if constexpr (op == 1) mbar_arrive(b);                   // plain arrive
            if constexpr (op == 2) mbar_arrive_expect_tx(b, 0);      // arrive.expect_tx(0)
            if constexpr (op == 3) umma_commit(b);                   // tcgen05.commit (nothing pending)
            if constexpr (op == 4) tc_fence_after();                 // tcgen05.fence::after_thread_sync
            if constexpr (op == 5) gbuf[i & 1023] = clock64();       // trace store
            if constexpr (op == 6) { mbar_arrive(b); mbar_wait(b, (i >> 6) & 1); }  // arrive + wait own phase
            if constexpr (op == 7) asm volatile("" ::"l"(b));        // empty loop
        }
        unsigned long long t1 = clock64();
        out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<32>(tslot);
}

int main() {
    unsigned long long *d, *g;
    cudaMalloc(&d, 8);
    cudaMalloc(&g, 8 * 1024);
    const char* names[] = {"try_wait(complete)", "mbarrier.arrive", "arrive.expect_tx(0)", "tcgen05.commit",
                           "tcgen05.fence::after", "clock64+STG", "arrive+wait(own)", "empty loop"};
    void (*kernels[])(unsigned long long*, unsigned long long*) = {bench<0>, bench<1>, bench<2>, bench<3>,
                                                                  bench<4>, bench<5>, bench<6>, bench<7>};
    for (int op = 0; op < 8; ++op) {
        kernels[op]<<<1, 64>>>(d, g);
        unsigned long long c = 0;
        if (cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
            printf("error at op %d\n", op);
            return 1;
        }
        printf("%-22s %6.1f cycles/op\n", names[op], double(c) / 4096);
        fflush(stdout);
    }
    return 0;
}
