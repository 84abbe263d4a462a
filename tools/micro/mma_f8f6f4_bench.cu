// Micro-benchmark + probe (bring-up only): tcgen05.mma kind::f8f6f4 with
// A = FP6 e3m2 from TMEM (8-bit containers) and B = FP8 e4m3 from shared
// memory (SW128 K-major), D = fp32 in TMEM.
//   (1) which bits of the 8-bit container hold the e3m2 code (probe: both
//       placements run against a host double-precision product);
//   (2) sustained cycles per MMA (M=128, K=32) for N = 16..128 vs kind::f16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2401_14112_b200/csrc -o mma_f8f6f4_bench mma_f8f6f4_bench.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx_sm100.cuh"

using namespace fpxk;

__host__ __device__ constexpr uint32_t idesc_f8f6f4(uint32_t m, uint32_t n, uint32_t afmt, uint32_t bfmt) {
    return (1u << 4) | (afmt << 7) | (bfmt << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
constexpr uint32_t kE4M3 = 0, kE3M2 = 4, kE2M3 = 3;

FPX_DEV void umma_f8f6f4_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

FPX_DEV void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// ------------------------------------------------------------ probe
// a_codes[128][32] (e3m2 codes), b_codes[N=16][32] (e4m3), shift = bit position of the code in its byte
__global__ void __launch_bounds__(128, 1) probe(const uint8_t* a_codes, const uint8_t* b_codes, int shift,
                                                uint32_t afmt, float* d_out) {
    __shared__ __align__(1024) uint8_t bsm[16 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
    // B: row n = 128 B (K-major), 16-byte chunk c of row n at chunk c ^ (n % 8) (SW128)
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) {
        const int n = i / 128, byte = i % 128, c = byte / 16;
        const int k = byte;  // only k < 32 used by one MMA
        const uint8_t v = k < 32 ? b_codes[n * 32 + k] : 0;
        bsm[n * 128 + ((c ^ (n % 8)) * 16) + byte % 16] = v;
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    // A: lane m = row m, column c holds k = 4c..4c+3 (byte k % 4)
    {
        const uint32_t m = threadIdx.x;
        uint32_t r[8];
        for (int c = 0; c < 8; ++c) {
            uint32_t w = 0;
            for (int j = 0; j < 4; ++j) {
                // shift 9: code in bits 5:0 with junk in bits 7:6
                const uint32_t code = a_codes[m * 32 + 4 * c + j];
                const uint32_t byte = shift == 9 ? (code | (((m * 131 + c * 17 + j * 7) & 3u) << 6)) : ((code << shift) & 0xffu);
                w |= byte << (8 * j);
            }
            r[c] = w;
        }
        tmem_st_32x32b_x8(tmem + ((32 * warp) << 16), r);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        umma_f8f6f4_ts(tmem + 256, tmem, umma_desc_sw128_kmajor(smem_u32(bsm)), idesc_f8f6f4(128, 16, afmt, kE4M3), 0u);
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t v[16];
    tmem_ld_32x32b_x16(tmem + ((32 * warp) << 16) + 256, v);
    tmem_ld_wait();
    for (int n = 0; n < 16; ++n) d_out[threadIdx.x * 16 + n] = __uint_as_float(v[n]);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

double dec_e3m2(int c) {
    const int s = (c >> 5) & 1, e = (c >> 2) & 7, m = c & 3;
    const double v = e == 0 ? std::ldexp(m, -2 - 2) : std::ldexp(4 + m, e - 3 - 2);
    return s ? -v : v;
}
double dec_e2m3(int c) {
    const int s = (c >> 5) & 1, e = (c >> 3) & 3, m = c & 7;
    const double v = e == 0 ? std::ldexp(m, 0 - 3) : std::ldexp(8 + m, e - 1 - 3);
    return s ? -v : v;
}
double dec_e4m3(int c) {
    const int s = (c >> 7) & 1, e = (c >> 3) & 15, m = c & 7;
    const double v = e == 0 ? std::ldexp(m, -6 - 3) : std::ldexp(8 + m, e - 7 - 3);
    return s ? -v : v;
}

// ------------------------------------------------------------ rate
template <int N, bool F8, int R, bool DISTINCT = false>
__global__ void __launch_bounds__(64, 1) rate(unsigned long long* out, int rounds) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* bsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&tslot);
    if (threadIdx.x == 32) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 8 * N * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint64_t bdesc = umma_desc_sw128_kmajor(smem_u32(bsm));
        unsigned long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (r >= 4) mbar_wait(&bar[r % 4], ((r / 4) - 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    // DISTINCT: every MMA of a round reads a different A (TMEM columns
                    // 0..255) and B (a different 1 KB swizzle atom group), like a
                    // streaming kernel; else four A/B addresses are reused
                    const uint32_t ai = DISTINCT ? (k % 32) * 8 : (k & 3) * 8;
                    const uint64_t bi = DISTINCT ? ((k % 8) * (N * 128 / 16) + (k & 3) * 2) : 2 * (k & 3);
                    if constexpr (F8)
                        umma_f8f6f4_ts(tmem + 256, tmem + ai, bdesc + bi, idesc_f8f6f4(128, N, kE3M2, kE4M3), 1u);
                    else
                        umma_f16_ts(tmem + 256, tmem + ai, bdesc + bi, umma_idesc_f16(128, N), 1u);
                }
                umma_commit(&bar[r % 4]);
            }
            __syncwarp();
        }
        for (int r = rounds - 4; r < rounds; ++r) mbar_wait(&bar[r % 4], (r / 4) & 1);
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool F8, int R, bool DISTINCT = false>
void run_rate(unsigned long long* d) {
    unsigned long long h[148];
    const int rounds = 512;
    constexpr int kSmem = 8 * N * 128 + 2048;
    cudaFuncSetAttribute(rate<N, F8, R, DISTINCT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    rate<N, F8, R, DISTINCT><<<148, 64, kSmem>>>(d, rounds);
    if (cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        printf("rate error %s\n", cudaGetErrorString(cudaGetLastError()));
        exit(1);
    }
    double c = 0;
    for (int b = 0; b < 148; ++b) c += h[b];
    c /= 148;
    const double per = c / rounds / R;
    const int K = F8 ? 32 : 16;
    printf("%s M=128 N=%3d K=%d R=%2d %s: %6.1f cycles/MMA -> %5.1f weights/clk/SM\n", F8 ? "f8f6f4 e3m2 x e4m3" : "f16             ",
           N, K, R, DISTINCT ? "distinct A/B" : "reused A/B  ", per, 128.0 * K / per);
}

int main() {
    // ---- probe
    const int M = 128, N = 16, K = 32;
    std::vector<uint8_t> a(M * K), b(N * K);
    srand(7);
    for (auto& x : a) x = rand() % 64;
    for (auto& x : b) {
        int c;
        do c = rand() % 256;
        while ((c & 0x7f) == 0x7f || ((c >> 3) & 15) > 9);  // no NaN, modest range
        x = static_cast<uint8_t>(c);
    }
    uint8_t *da, *db;
    float* dd;
    cudaMalloc(&da, a.size());
    cudaMalloc(&db, b.size());
    cudaMalloc(&dd, M * N * 4);
    cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
    for (uint32_t afmt : {kE3M2, kE2M3}) {
        for (int shift : {0, 2, 9}) {
            probe<<<1, 128>>>(da, db, shift, afmt, dd);
            std::vector<float> d(M * N);
            if (cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
                printf("probe error %s\n", cudaGetErrorString(cudaGetLastError()));
                return 1;
            }
            double maxerr = 0, maxref = 0;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k)
                        ref += (afmt == kE3M2 ? dec_e3m2(a[m * K + k]) : dec_e2m3(a[m * K + k])) * dec_e4m3(b[n * K + k]);
                    maxerr = std::fmax(maxerr, std::fabs(ref - d[m * N + n]));
                    maxref = std::fmax(maxref, std::fabs(ref));
                }
            printf("probe %s code<<%d (9 = junk in bits 7:6): max |D - ref| = %.3g (max |ref| %.3g)%s\n", afmt == kE3M2 ? "e3m2" : "e2m3", shift,
                   maxerr, maxref, maxerr <= 1e-6 * maxref ? "  <== MATCH" : "");
        }
    }
    // ---- rate
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run_rate<16, false, 32>(d);
    run_rate<16, true, 32>(d);
    run_rate<32, true, 32>(d);
    run_rate<48, true, 32>(d);
    run_rate<64, true, 32>(d);
    run_rate<96, true, 32>(d);
    run_rate<128, true, 32>(d);
    run_rate<256, true, 32>(d);
    run_rate<48, true, 8>(d);
    run_rate<16, false, 32, true>(d);
    run_rate<32, false, 32, true>(d);
    run_rate<16, true, 32, true>(d);
    run_rate<32, true, 32, true>(d);
    run_rate<48, true, 32, true>(d);
    run_rate<64, true, 32, true>(d);
    run_rate<96, true, 32, true>(d);
    run_rate<16, false, 12, true>(d);
    run_rate<48, true, 6, true>(d);
    run_rate<96, true, 6, true>(d);
    printf("done\n");
    return 0;
}
