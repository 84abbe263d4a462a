// Host->device copy of one decode step's activations (2.77 MB): copy engine
// on 1 / 2 / 4 streams vs a zero-copy kernel reading mapped pinned memory.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        dst[i] = src[i];
    }
}

int main() {
    const size_t nb = 2774016;
    void *h, *hm, *d;
    cudaHostAlloc(&h, nb, cudaHostAllocDefault);
    cudaHostAlloc(&hm, nb, cudaHostAllocMapped);
    cudaMalloc(&d, nb);
    memset(h, 1, nb);
    memset(hm, 1, nb);
    void* hm_dev;
    cudaHostGetDevicePointer(&hm_dev, hm, 0);
    cudaStream_t s[4];
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, ev[4];
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    auto run = [&](const char* name, auto&& fn) {
        for (int w = 0; w < 3; ++w) fn();
        cudaDeviceSynchronize();
        const int reps = 50;
        cudaEventRecord(e0, s[0]);
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1, s[0]);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-32s %7.1f us  %6.1f GB/s\n", name, ms * 1e3 / reps, nb * reps / (ms * 1e-3) / 1e9);
    };
    auto split = [&](int k, void* src) {
        cudaEventRecord(ev[0], s[0]);
        for (int i = 1; i < k; ++i) cudaStreamWaitEvent(s[i], ev[0]);
        for (int i = 0; i < k; ++i)
            cudaMemcpyAsync((char*)d + nb / k * i, (char*)src + nb / k * i, nb / k, cudaMemcpyHostToDevice, s[i]);
        for (int i = 1; i < k; ++i) cudaEventRecord(ev[i], s[i]), cudaStreamWaitEvent(s[0], ev[i]);
    };
    for (int pass = 0; pass < 2; ++pass) {
        run("CE 1 stream", [&] { split(1, h); });
        run("CE 2 streams", [&] { split(2, h); });
        run("CE 4 streams", [&] { split(4, h); });
        run("CE 1 stream (mapped buffer)", [&] { split(1, hm); });
        for (int g : {16, 32, 64, 148}) {
            char nm[64];
            snprintf(nm, sizeof nm, "zero-copy kernel %3d CTAs", g);
            run(nm, [&] { zc_copy<<<g, 256, 0, s[0]>>>((const uint4*)hm_dev, (uint4*)d, nb / 16); });
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
