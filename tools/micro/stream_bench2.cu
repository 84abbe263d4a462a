// Micro-benchmark (bring-up only): which weight-streaming scheme reaches the
// B200 HBM read roofline for a 135 MB packed FP6 weight (llama-65B FFN)?
// Variants: 1-D TMA bulk copies into an SMEM ring (1 or 2 CTAs/SM, per-CTA
// contiguous slice vs chunk-interleaved across CTAs, with/without L2 cache
// hint, with an L2 bulk prefetch running ahead), vs a plain LDG stream.
// Every variant is timed as 12 back-to-back launches over 3 rotating copies
// (405 MB > L2), so the per-launch figure excludes launch latency effects
// that a single timed launch would include; a single-launch figure is printed too.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o stream_bench2 stream_bench2.cu
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

FPX_DEV void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

FPX_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

struct Args {
    const uint8_t* src;
    size_t total;     // bytes of one copy
    int chunk;        // bytes per stage
    int stages;
    int interleave;   // 0: CTA-contiguous slices, 1: chunk c goes to CTA c % grid
    int hint;         // 0 none, 1 evict_first
    int prefetch;     // chunks of L2 prefetch run-ahead (0 = off)
    unsigned long long* sink;
};

__global__ void __launch_bounds__(64) tma_stream(Args a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[32], empty[32];
    const uint32_t warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.stages; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const size_t nchunks = a.total / a.chunk;
    size_t c_begin, c_step, c_end;
    if (a.interleave) {
        c_begin = blockIdx.x, c_step = gridDim.x, c_end = nchunks;
    } else {
        c_begin = nchunks * blockIdx.x / gridDim.x, c_step = 1, c_end = nchunks * (blockIdx.x + 1) / gridDim.x;
    }
    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol = policy_evict_first();
            int s = 0;
            size_t pf = c_begin;
            for (size_t c = c_begin; c < c_end; c += c_step, ++s) {
                if (a.prefetch) {
                    const size_t lim = c + (size_t)a.prefetch * c_step;
                    for (; pf < c_end && pf <= lim; pf += c_step) bulk_prefetch_l2(a.src + pf * a.chunk, a.chunk);
                }
                const int st = s % a.stages;
                mbar_wait(&empty[st], ((s / a.stages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[st], a.chunk);
                if (a.hint)
                    bulk_g2s(sm + st * a.chunk, a.src + c * a.chunk, a.chunk, &full[st], pol);
                else
                    bulk_g2s_nohint(sm + st * a.chunk, a.src + c * a.chunk, a.chunk, &full[st]);
            }
        }
    } else {
        unsigned long long acc = 0;
        if (elect_one()) {
            int s = 0;
            for (size_t c = c_begin; c < c_end; c += c_step, ++s) {
                const int st = s % a.stages;
                mbar_wait(&full[st], (s / a.stages) & 1);
                acc += sm[st * a.chunk];
                mbar_arrive(&empty[st]);
            }
        }
        if (acc == 0x1234567) a.sink[0] = acc;
    }
}

__global__ void ldg_stream(const uint4* src, size_t n16, unsigned long long* sink) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
#pragma unroll 1
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x1234567) sink[0] = acc;
}

int main() {
    const size_t per = 135266304;
    uint8_t* buf;
    cudaMalloc(&buf, 3 * per);
    cudaMemset(buf, 1, 3 * per);
    unsigned long long* sink;
    cudaMalloc(&sink, 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch) {
        for (int r = 0; r < 3; ++r) launch(r);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        launch(0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float one;
        cudaEventElapsedTime(&one, a, b);
        cudaEventRecord(a);
        for (int r = 1; r <= 12; ++r) launch(r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return std::make_pair(one * 1e3f, ms / 12 * 1e3f);
    };
    for (int cpb : {4, 8}) {
        auto [one, us] = timeit([&](int r) {
            ldg_stream<<<148 * cpb, 512>>>(reinterpret_cast<const uint4*>(buf + (r % 3) * per), per / 16, sink);
        });
        printf("LDG stream %d CTA/SM x512: single %.1f us | b2b %.1f us %.0f GB/s\n", cpb, one, us, per / (us * 1e-6) / 1e9);
    }
    struct Cfg { int chunk, stages, ctas_per_sm, interleave, hint, prefetch; };
    const Cfg cfgs[] = {
        {16384, 12, 1, 0, 1, 0}, {16384, 12, 1, 1, 1, 0}, {16384, 12, 1, 0, 0, 0}, {16384, 12, 1, 1, 0, 0},
        {16384, 6, 2, 0, 1, 0},  {16384, 6, 2, 1, 1, 0},  {8192, 12, 2, 1, 1, 0},  {32768, 6, 1, 1, 1, 0},
        {16384, 12, 1, 1, 1, 4}, {16384, 12, 1, 1, 1, 12}, {16384, 12, 1, 0, 1, 8}, {8192, 24, 1, 1, 1, 0},
        {24576, 8, 1, 1, 1, 0},  {12288, 16, 1, 1, 1, 0}, {16384, 4, 3, 1, 1, 0},
    };
    for (const Cfg& c : cfgs) {
        const int smem = c.chunk * c.stages;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = 148 * c.ctas_per_sm;
        auto [one, us] = timeit([&](int r) {
            Args ar{buf + (r % 3) * per, per / c.chunk * c.chunk, c.chunk, c.stages, c.interleave, c.hint, c.prefetch, sink};
            tma_stream<<<grid, 64, smem>>>(ar);
        });
        printf("TMA chunk %6d x %2d stages, %d CTA/SM, %s, hint %d, prefetch %2d: single %.1f us | b2b %.1f us %.0f GB/s\n",
               c.chunk, c.stages, c.ctas_per_sm, c.interleave ? "interleaved" : "contiguous ", c.hint, c.prefetch, one,
               us, per / (us * 1e-6) / 1e9);
        fflush(stdout);
    }
    cudaError_t e = cudaGetLastError();
    printf("last error: %s\n", cudaGetErrorString(e));
    return 0;
}
