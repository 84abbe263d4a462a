// Micro-benchmark (bring-up only): steady-state HBM READ bandwidth on B200,
// i.e. the ceiling a weight-streaming kernel can approach, measured with a
// stream long enough (2 GiB per launch) that launch ramp and tail vanish,
// and the same readers over 135 MB (one llama-65B FP6 weight) for the
// per-launch overhead.
//   A  1-D TMA bulk copies into an SMEM ring, 1 consumer warp releasing
//      slots at once (CTAs/SM x stages x chunk swept)
//   B  LDG.128 streaming, many warps, 8 independent loads in flight/thread
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o read_bw_bench read_bw_bench.cu
#include <cstdint>
#include <cstdio>
#include <vector>

#include "ptx_sm100.cuh"

using namespace fpxk;

struct TArgs {
    const uint8_t* src;
    size_t total;
    int chunk;
    int stages;
    unsigned long long* sink;
};

__global__ void __launch_bounds__(64) tma_read(TArgs a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[32], empty[32];
    const uint32_t warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.stages; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const size_t nchunks = a.total / a.chunk;
    const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
    const uint64_t pol = policy_evict_first();
    if (warp == 0) {
        if (elect_one()) {
            uint32_t i = 0;
            for (size_t c = c0; c < c1; ++c, ++i) {
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1u;
                if (i >= (uint32_t)a.stages) mbar_wait(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], a.chunk);
                bulk_g2s(sm + (size_t)s * a.chunk, a.src + c * a.chunk, a.chunk, &full[s], pol);
            }
        }
    } else {
        uint32_t i = 0, acc = 0;
        for (size_t c = c0; c < c1; ++c, ++i) {
            const uint32_t s = i % a.stages, ph = (i / a.stages) & 1u;
            mbar_wait(&full[s], ph);
            acc ^= lds32(smem_u32(sm + (size_t)s * a.chunk + 4 * (threadIdx.x & 31)));
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 0x12345679u) atomicAdd(a.sink, 1ull);
    }
}


// The decode kernel's weight pattern: a CTA streams one unit (2 tile-rows x
// a K chunk) of the hi (1 KB/tile) and lo (2 KB/tile) streams; a stage is
// KS k-tiles: 4 bulk copies (hi r0, hi r1, lo r0, lo r1) of KS KB / 2 KS KB.
struct PArgs {
    const uint8_t* hi;
    const uint8_t* lo;
    int kt, tile_rows, split, ks, stages;
    unsigned long long* sink;
    int hb = 1024, lb = 2048;  // stream bytes per 64x64 tile (e3m2: 2-bit hi, 4-bit lo)
    int passes = 1;            // linears streamed back to back inside ONE launch
    size_t pass_stride = 0;    // bytes between the passes' weight copies (3 rotated)
};
__global__ void __launch_bounds__(64) pattern_read(PArgs a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[32], empty[32];
    const uint32_t warp = threadIdx.x >> 5;
    const int stage_bytes = 2 * (a.hb + a.lb) * a.ks;
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.stages; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int units = a.tile_rows / 2 * a.split;
    const int u0 = (int)((long)blockIdx.x * units / gridDim.x), u1 = (int)((long)(blockIdx.x + 1) * units / gridDim.x);
    const uint64_t pol = policy_evict_first();
    if (warp == 0) {
        if (elect_one()) {
            uint32_t i = 0;
            for (int pass = 0; pass < a.passes; ++pass)
            for (int u = u0; u < u1; ++u) {
                const size_t po = (pass % 3) * a.pass_stride;
                const int mt = u / a.split, ch = u % a.split;
                const int k0 = ch * a.kt / a.split, k1 = (ch + 1) * a.kt / a.split;
                for (int k = k0; k + a.ks <= k1; k += a.ks, ++i) {
                    const uint32_t s = i % a.stages, ph = (i / a.stages) & 1u;
                    if (i >= (uint32_t)a.stages) mbar_wait(&empty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[s], stage_bytes);
                    uint8_t* d = sm + (size_t)s * stage_bytes;
                    for (int r = 0; r < 2; ++r) {
                        const size_t t = (size_t)(2 * mt + r) * a.kt + k;
                        bulk_g2s(d + r * a.hb * a.ks, a.hi + po + t * a.hb, a.hb * a.ks, &full[s], pol);
                        bulk_g2s(d + 2 * a.hb * a.ks + r * a.lb * a.ks, a.lo + po + t * a.lb, a.lb * a.ks, &full[s],
                                 pol);
                    }
                }
            }
        }
    } else {
        uint32_t i = 0, acc = 0;
        for (int pass = 0; pass < a.passes; ++pass)
        for (int u = u0; u < u1; ++u) {
            const int ch = u % a.split;
            const int k0 = ch * a.kt / a.split, k1 = (ch + 1) * a.kt / a.split;
            for (int k = k0; k + a.ks <= k1; k += a.ks, ++i) {
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1u;
                mbar_wait(&full[s], ph);
                acc ^= lds32(smem_u32(sm + (size_t)s * stage_bytes + 4 * (threadIdx.x & 31)));
                __syncwarp();
                if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
            }
        }
        if (acc == 0x12345679u) atomicAdd(a.sink, 1ull);
    }
}

__global__ void __launch_bounds__(512) ldg_read(const uint4* __restrict__ src, size_t nvec,
                                                unsigned long long* sink) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    size_t i = tid;
    for (; i + 7 * stride < nvec; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < nvec; i += stride) {
        const uint4 v = __ldcs(src + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345679u) atomicAdd(sink, 1ull);
}

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

int main() {
    const size_t big = size_t(2) << 30, small = 135266304;
    const int copies = 3;  // small runs rotate 3 copies (> L2)
    uint8_t* buf;
    CK(cudaMalloc(&buf, big + copies * small + 4096));
    CK(cudaMemset(buf, 1, big + copies * small + 4096));
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    auto time_it = [&](auto&& launch, int reps) {
        launch(0);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch(r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms * 1e3 / reps;  // us per launch
    };
    struct TC { int cps, stages, chunk; };
    std::vector<TC> tcs = {{1, 12, 16384}, {1, 6, 32768}, {1, 24, 8192}, {1, 13, 12288}, {1, 4, 49152},
                           {2, 6, 16384}, {2, 12, 8192}, {3, 4, 16384}, {4, 6, 8192}, {1, 3, 65536}};
    for (const auto& t : tcs) {
        const int smem = t.stages * t.chunk;
        if (cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) continue;
        const int grid = nsm * t.cps;
        auto big_l = [&](int) {
            TArgs a{buf, big, t.chunk, t.stages, sink};
            tma_read<<<grid, 64, smem>>>(a);
        };
        auto small_l = [&](int r) {
            TArgs a{buf + big + (r % copies) * small, small, t.chunk, t.stages, sink};
            tma_read<<<grid, 64, smem>>>(a);
        };
        const double ub = time_it(big_l, 3), us = time_it(small_l, 12);
        printf("TMA %d CTA/SM x %2d stages x %6d B (%3d KB in flight/SM): 2 GiB %7.1f us = %6.0f GB/s | 135 MB b2b %5.1f us = %6.0f GB/s\n",
               t.cps, t.stages, t.chunk, t.cps * smem / 1024, ub, big / ub / 1e3, us, small / us / 1e3);
        CK(cudaGetLastError());
    }
    // per-SM TMA ceiling: fewer CTAs than SMs (1 CTA/SM placement), same 192 KB ring
    for (int grid : {32, 64, 96, 128, 148}) {
        for (int chunk : {12288, 16384, 49152}) {
            const int stages = (chunk == 12288 ? 16 : 196608 / chunk);
            const int smem = stages * chunk;
            cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            auto big_l = [&](int) {
                TArgs a{buf, big / 4, chunk, stages, sink};
                tma_read<<<grid, 64, smem>>>(a);
            };
            const double ub = time_it(big_l, 3);
            printf("TMA grid %3d x %2d stages x %6d B: 512 MiB %7.1f us = %6.0f GB/s = %5.1f GB/s per CTA\n", grid, stages,
                   chunk, ub, big / 4 / ub / 1e3, big / 4 / ub / 1e3 / grid);
        }
    }
    for (int bps : {2, 4, 8}) {
        const int grid = nsm * bps;
        auto big_l = [&](int) { ldg_read<<<grid, 512>>>(reinterpret_cast<const uint4*>(buf), big / 16, sink); };
        auto small_l = [&](int r) {
            ldg_read<<<grid, 512>>>(reinterpret_cast<const uint4*>(buf + big + (r % copies) * small), small / 16, sink);
        };
        const double ub = time_it(big_l, 3), us = time_it(small_l, 12);
        printf("LDG %d CTA/SM x 512 thr x 8 x 16 B: 2 GiB %7.1f us = %6.0f GB/s | 135 MB b2b %5.1f us = %6.0f GB/s\n", bps,
               ub, big / ub / 1e3, us, small / us / 1e3);
        CK(cudaGetLastError());
    }
    // the decode kernel's access pattern, 8192 x 22016 e3m2 (hi 45 MB, lo 90 MB, 3 rotated copies)
    {
        const int kt = 344, trs = 128;
        const size_t hi_b = (size_t)trs * kt * 1024, lo_b = (size_t)trs * kt * 2048;
        uint8_t* pbuf;
        CK(cudaMalloc(&pbuf, 3 * (hi_b + lo_b)));
        CK(cudaMemset(pbuf, 1, 3 * (hi_b + lo_b)));
        struct PC { int grid, split, ks, stages; };
        for (PC c : {PC{128, 2, 2, 13}, PC{128, 2, 2, 17}, PC{148, 9, 2, 13}, PC{128, 2, 4, 7}, PC{128, 2, 1, 26}, PC{148, 37, 2, 13}}) {
            const int smem = c.stages * 6 * 1024 * c.ks;
            if (cudaFuncSetAttribute(pattern_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) continue;
            auto l = [&](int r) {
                const uint8_t* base = pbuf + (r % 3) * (hi_b + lo_b);
                PArgs a{base, base + hi_b, kt, trs, c.split, c.ks, c.stages, sink};
                pattern_read<<<c.grid, 64, smem>>>(a);
            };
            const double us = time_it(l, 12);
            printf("pattern grid %3d split %2d KS %d stages %2d (%3d KB ring): 135 MB b2b %5.1f us = %6.0f GB/s\n", c.grid,
                   c.split, c.ks, c.stages, smem / 1024, us, (hi_b + lo_b) / us / 1e3);
            CK(cudaGetLastError());
        }
    }
    // launch boundaries: the e3m2 pattern, 6 linears per launch vs 1
    {
        const int kt = 344, trs = 128;
        const size_t hi_b = (size_t)trs * kt * 1024, lo_b = (size_t)trs * kt * 2048;
        uint8_t* pbuf;
        CK(cudaMalloc(&pbuf, 3 * (hi_b + lo_b)));
        CK(cudaMemset(pbuf, 1, 3 * (hi_b + lo_b)));
        for (int grid : {128, 148}) {
            const int split = grid == 128 ? 2 : 37, stages = 13, smem = stages * 6 * 1024 * 2;
            cudaFuncSetAttribute(pattern_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int passes : {1, 6}) {
                auto l = [&](int r) {
                    const uint8_t* base = pbuf + (passes == 1 ? (r % 3) * (hi_b + lo_b) : 0);
                    PArgs a{base, base + hi_b, kt, trs, split, 2, stages, sink};
                    a.passes = passes;
                    a.pass_stride = hi_b + lo_b;
                    pattern_read<<<grid, 64, smem>>>(a);
                };
                const double us = time_it(l, 12) / passes;
                printf("boundary grid %3d split %2d: %d linear(s) per launch: %5.1f us per 135 MB linear = %6.0f GB/s\n",
                       grid, split, passes, us, (hi_b + lo_b) / us / 1e3);
                CK(cudaGetLastError());
            }
        }
        cudaFree(pbuf);
    }
    // the same for e2m2 (4-bit hi 2 KB/tile, 1-bit lo 512 B/tile: 112.7 MB)
    {
        const int kt = 344, trs = 128;
        const size_t hi_b = (size_t)trs * kt * 2048, lo_b = (size_t)trs * kt * 512;
        uint8_t* pbuf;
        CK(cudaMalloc(&pbuf, 3 * (hi_b + lo_b)));
        CK(cudaMemset(pbuf, 1, 3 * (hi_b + lo_b)));
        struct PC { int grid, split, ks, stages; };
        for (PC c : {PC{128, 2, 2, 13}, PC{128, 2, 2, 16}, PC{128, 2, 4, 8}, PC{148, 9, 2, 13}}) {
            const int smem = c.stages * 5 * 1024 * c.ks;
            if (cudaFuncSetAttribute(pattern_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) continue;
            auto l = [&](int r) {
                const uint8_t* base = pbuf + (r % 3) * (hi_b + lo_b);
                PArgs a{base, base + hi_b, kt, trs, c.split, c.ks, c.stages, sink, 2048, 512};
                pattern_read<<<c.grid, 64, smem>>>(a);
            };
            const double us = time_it(l, 12);
            printf("e2m2 pattern grid %3d split %2d KS %d stages %2d (%3d KB ring): %.1f MB b2b %5.1f us = %6.0f GB/s\n", c.grid,
                   c.split, c.ks, c.stages, smem / 1024, (hi_b + lo_b) / 1e6, us, (hi_b + lo_b) / us / 1e3);
            CK(cudaGetLastError());
        }
    }
    printf("done\n");
    return 0;
}
