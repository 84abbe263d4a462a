// fpx_kernels.h -- host-side launch entry points of the sm_100a kernels
// (internal to libfpx_b200.so; the public surface is include/fpx_c.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

cudaError_t launch_quantize(const void* w, int w_dtype, uint32_t rows, uint32_t cols, uint32_t rows_p,
                            uint32_t cols_p, int e, int m, double maxrep, uint8_t* codes,
                            uint16_t* scales, unsigned long long* status, cudaStream_t st);
cudaError_t launch_quantize_pack(const void* w, int w_dtype, uint32_t rows, uint32_t cols, uint32_t rows_p,
                                 uint32_t cols_p, int e, int m, double maxrep, uint16_t* scales,
                                 unsigned long long* status, uint8_t* row_skip, int nseg, const int* widths,
                                 uint8_t* const* streams, cudaStream_t st);
cudaError_t launch_prepack(const uint8_t* codes, uint32_t rows_p, uint32_t cols_p, int bits, int nseg,
                           const int* widths, uint8_t* const* streams, cudaStream_t st);
cudaError_t launch_unpack(const uint8_t* const* streams, uint32_t rows_p, uint32_t cols_p, int bits, int nseg,
                          const int* widths, uint8_t* codes, cudaStream_t st);
cudaError_t launch_dequant(const uint8_t* const* streams, int nseg, const int* widths, const uint16_t* scales,
                           uint32_t rows_p, uint32_t cols_p, int e, int m, uint16_t* out, int path,
                           cudaStream_t st);
cudaError_t launch_dequant_codes(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p, int e,
                                 int m, unsigned long long* status, uint16_t* out, cudaStream_t st);
cudaError_t launch_check_scales(const uint16_t* scales, uint32_t n, int rebias, unsigned int* bad,
                                cudaStream_t st);
cudaError_t launch_stage_act(const uint16_t* src, uint32_t k_act, uint32_t n, uint32_t k_pad, uint16_t* dst,
                             cudaStream_t st);
cudaError_t launch_gather_shards(const float* g, uint32_t rows_p, int world, uint32_t m_slot, uint32_t n, float* c,
                                 uint32_t ldc, cudaStream_t st);
cudaError_t launch_gather_permute(const float* g, const uint32_t* row0, const uint32_t* nrows, int world,
                                  uint32_t m_slot, uint32_t n, float* c, uint32_t ldc, cudaStream_t st);

// Fused de-quantise + tcgen05 GEMM (fpx_linear.cu).
struct LinearLaunch {
    int fmt;                   // fpxk::FmtId
    const uint8_t* s_hi;       // stream of the high segment
    const uint8_t* s_lo;       // stream of the low segment
    const uint16_t* scales;    // raw fp16 row scales (rows_p)
    uint32_t rows_p, cols_p;   // padded weight dims (multiples of 64)
    const uint16_t* act;       // col-major activations, row j at act + j*lda, K == cols_p
    uint32_t lda;              // >= cols_p, multiple of 8
    uint32_t n;                // batch (1..256)
    float* c;                  // col-major output, element (m, j) at c[j*ldc + m] (fp16 when out_f16)
    uint32_t ldc;
    int split;                 // K chunks per 128-row tile (>= 1)
    float* ws;                 // split > 1: partial sums
    uint32_t* counters;        // split > 1: per (tile, quarter) arrival counters (zeroed once)
    int grid;                  // persistent CTAs (0 = auto)
    unsigned long long* trace; // debug: per-stage clock64 trace of CTA 0 (7 events x 512 stages), or null
    volatile unsigned long long* prog;  // debug: mapped host progress words (FPX_LINEAR_TRACE=3), or null
    // fused epilogue (fpx_linear_ex): C = act(A.B + bias) + residual, stored fp32 or fp16
    uint32_t out_f16;
    const float* bias;         // rows_p, or null
    uint32_t act_fn;           // 0 none, 1 relu, 2 silu, 3 gelu (tanh)
    const void* resid;         // same dtype / layout / ldc as C, or null
    // Upper bound on the programmatic-dependent-launch mode of this launch
    // (see pdl_mode in fpx_linear.cu): 1 after a library kernel wrote packed
    // weights / scales on the same stream, so nothing is read before
    // griddepcontrol.wait; 2 = no cap.
    uint32_t pdl_cap = 2;
    // N <= 32: workspace for the activations' e4m3 split (kind::f8f6f4 units of
    // the decode kernel): b8 [3 * npad(n)][cols_p] bytes, colf [split][npad(n)]
    // floats; null = kind::f16 only.
    uint8_t* b8 = nullptr;
    float* colf = nullptr;
};

cudaError_t launch_linear(const LinearLaunch& p, cudaStream_t st);
size_t linear_workspace_bytes(uint32_t rows_p, uint32_t n, int split);
size_t linear_split_bytes(uint32_t cols_p, uint32_t n, int split);  // b8 + colf (0 when n > 32)
bool linear_x8_enabled();  // FPX_LINEAR_X8=1: the opt-in kind::f8f6f4 kernel for N <= 32
int linear_default_split(uint32_t rows_p, uint32_t cols_p, uint32_t n, int num_sms);
