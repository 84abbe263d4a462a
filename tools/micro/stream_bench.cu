// Micro-benchmark (bring-up only): achievable HBM read bandwidth of
// 1-D TMA bulk copies into an SMEM ring, per stage size / depth / copy size,
// vs a plain vectorised LDG stream.  Each CTA streams a contiguous slice of a
// 3 x 135 MB rotating buffer (L2-cold).
#include <cstdint>
#include <cstdio>

#include "ptx_sm100.cuh"

using namespace fpxk;

__global__ void __launch_bounds__(64, 1) tma_stream(const uint8_t* src, size_t bytes_per_cta, int stage_bytes,
                                                    int stages, int copies, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[32], empty[32];
    const uint32_t warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint8_t* base = src + blockIdx.x * bytes_per_cta;
    const int nst = static_cast<int>(bytes_per_cta / stage_bytes);
    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol = policy_evict_first();
            const int cb = stage_bytes / copies;
            for (int s = 0; s < nst; ++s) {
                const int st = s % stages;
                mbar_wait(&empty[st], ((s / stages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[st], stage_bytes);
                for (int c = 0; c < copies; ++c)
                    bulk_g2s(sm + st * stage_bytes + c * cb, base + (size_t)s * stage_bytes + c * cb, cb, &full[st], pol);
            }
        }
    } else {
        unsigned long long acc = 0;
        if (elect_one()) {
            for (int s = 0; s < nst; ++s) {
                const int st = s % stages;
                mbar_wait(&full[st], (s / stages) & 1);
                acc += sm[st * stage_bytes];
                mbar_arrive(&empty[st]);
            }
        }
        if (acc == 0x1234567) sink[0] = acc;
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

template <int op>
__global__ void sync_cost(unsigned long long* out) {
    __shared__ uint64_t bars[64];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 64; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
        for (int i = 0; i < 64; ++i) mbar_arrive(&bars[i]);  // complete phase 0
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0 = clock64();
        for (int i = 0; i < 4096; ++i) {
            if constexpr (op == 0) mbar_wait(&bars[i & 63], 0);        // completed phase
            if constexpr (op == 1) mbar_wait(&bars[i & 63], 1);        // "previous" phase of a fresh-ish barrier
        }
        out[0] = clock64() - t0;
    }
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
    for (int op = 0; op < 1; ++op) {
        if (op == 0) sync_cost<0><<<1, 32>>>(sink);
        else sync_cost<1><<<1, 32>>>(sink);
        unsigned long long c;
        cudaMemcpy(&c, sink, 8, cudaMemcpyDeviceToHost);
        printf("try_wait %s: %.1f cycles\n", op ? "(prev phase)" : "(completed)", c / 4096.0);
    }
    // LDG reference
    for (int rep = 0; rep < 2; ++rep) {
        float tot = 0;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            ldg_stream<<<148 * 4, 512>>>(reinterpret_cast<const uint4*>(buf + (r % 3) * per), per / 16, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) tot += ms;
        }
        printf("LDG stream: %.1f us  %.0f GB/s\n", tot / 3 * 1e3, per / (tot / 3 * 1e-3) / 1e9);
    }
    const int cfgs[][3] = {{8192, 12, 1}, {8192, 12, 4}, {16384, 12, 1}, {16384, 12, 4}, {16384, 8, 4},
                           {32768, 6, 1}, {32768, 6, 4}, {24576, 8, 4}, {49152, 4, 4}, {4096, 24, 1}, {16384, 12, 8}};
    for (auto& c : cfgs) {
        const int sbytes = c[0], stages = c[1], copies = c[2];
        const size_t per_cta = (per / 148) / sbytes * sbytes;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, sbytes * stages);
        float tot = 0;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            tma_stream<<<148, 64, sbytes * stages>>>(buf + (r % 3) * per, per_cta, sbytes, stages, copies, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) tot += ms;
        }
        const double bytes = (double)per_cta * 148;
        printf("TMA stage %6d B x %2d stages, %d copies/stage: %.1f us  %.0f GB/s\n", sbytes, stages, copies,
               tot / 3 * 1e3, bytes / (tot / 3 * 1e-3) / 1e9);
        fflush(stdout);
    }
    cudaError_t e = cudaGetLastError();
    printf("last error: %s\n", cudaGetErrorString(e));
    return 0;
}
