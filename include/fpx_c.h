/*
 * fpx_c.h -- C-ABI of libfpx_b200.so, the B200-native (sm_100a) TC-FPx
 * W6A16 linear layer.  Plain pointers and sizes only; no C++ or torch types.
 *
 * This is the drop-in boundary for the reference's C++ API
 * (/root/reference/proj/include/fpx/):
 *   fpx_quantize      <- quantize_matrix        codec.hpp:66   (codec.cpp:105-177)
 *   fpx_prepack       <- pack                   prepack.hpp:84-85 (prepack.cpp:153-209)
 *   fpx_unpack        <- unpack                 prepack.hpp:86  (prepack.cpp:211-260)
 *   fpx_dequantize    <- dequantize_reference(unpack(p))    (codec.cpp:179-193)
 *   fpx_dequantize_codes <- dequantize_reference codec.hpp:72   (codec.cpp:179-193)
 *   fpx_decode_scalar <- decode_scalar          codec.hpp:56   (codec.cpp:49-68)
 *   fpx_encode_scalar <- encode_scalar          codec.hpp:60   (codec.cpp:70-103)
 *   fpx_linear        <- gemm_packed            gemm.hpp:27-28 (gemm.cpp:170-219)
 *   fpx_effective_scale <- effective_scale      codec.hpp:76   (codec.cpp:195-199)
 *   fpx_format_check / fpx_split_for_format / fpx_max_representable
 *                     <- FpxFormat::make / SplitScheme::for_format /
 *                        FpxFormat::max_representable  format.hpp:26-57
 * The C++ value-type wrappers with the reference's exact signatures live in
 * include/fpx_b200.hpp.
 *
 * Conventions
 *   - Status: 0 on success, otherwise 1 + fpx::ErrorCode (error.hpp:10-24),
 *     or FPX_ERR_CUDA / FPX_ERR_DEVICE for runtime failures.  Nothing throws
 *     across this boundary.  fpx_last_error() returns the thread-local
 *     message of the last failure on the calling thread ("error[<code>] ...",
 *     error.cpp:24-35).
 *   - Every device pointer is caller-owned; all work is enqueued on `stream`
 *     (a cudaStream_t; NULL = legacy default stream).  Calls on distinct
 *     streams may run concurrently (reference: pure/reentrant).
 *   - Functions whose reference counterpart throws on data-dependent errors
 *     (NaN row, scale overflow) synchronise `stream` when `status_dev` is
 *     NULL and return the error; pass a device status word to stay async.
 *   - Workspaces (fpx_linear*): one per stream, see fpx_linear below.
 *   - Formats: exp_bits/man_bits as FpxFormat (E 1..5, M 0..6, 3..8 bits).
 *     The fused linear kernel serves e3m2 and e2m3 ([2,4] split) and e2m2
 *     ([4,1] split); pack/unpack/dequantize/quantize serve every format.
 *   - Matrices: weights row-major fp32 or fp16; codes row-major u8 padded to
 *     multiples of 64; scales one fp16 bit pattern per padded row;
 *     activations fp16 col-major K x N (= [N][K] row-major); outputs fp32
 *     col-major (padded rows) x N, leading dimension ldc.
 */
#ifndef FPX_C_H_
#define FPX_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fpx_stream_t; /* == cudaStream_t */

enum fpx_status {
    FPX_OK = 0,
    FPX_ERR_INVALID_FORMAT = 1,
    FPX_ERR_INVALID_CODE = 2,
    FPX_ERR_INVALID_VALUE = 3,
    FPX_ERR_SCALE_OVERFLOW = 4,
    FPX_ERR_SHAPE_MISMATCH = 5,
    FPX_ERR_RAGGED_INPUT = 6,
    FPX_ERR_UNSUPPORTED_SPLIT = 7,
    FPX_ERR_INDEX_OUT_OF_RANGE = 8,
    FPX_ERR_BAD_MAGIC = 9,
    FPX_ERR_BAD_VERSION = 10,
    FPX_ERR_TRUNCATED = 11,
    FPX_ERR_CORRUPT = 12,
    FPX_ERR_IO_FAILURE = 13,
    FPX_ERR_CUDA = 100,   /* CUDA runtime/driver error (message has details) */
    FPX_ERR_DEVICE = 101  /* no sm_100 device / feature unavailable */
};

enum fpx_dtype { FPX_FP32 = 0, FPX_FP16 = 1 }; /* codec.hpp:10 Dtype */

/* ---- library / host-only helpers (no GPU needed) ---------------------- */
const char* fpx_last_error(void);
/* Byte offset carried by the last error on this thread (file errors,
 * error.hpp:35-41 Error::offset), or -1. */
int64_t fpx_last_error_offset(void);
const char* fpx_status_name(int status);   /* error.cpp:5-22 names */
int fpx_version(void);                     /* major*10000 + minor*100 + patch */
int fpx_format_check(int exp_bits, int man_bits);            /* 0 or FPX_ERR_INVALID_FORMAT */
int fpx_split_for_format(int exp_bits, int man_bits, int* widths /* [3] */); /* #segments, 0 = none */
float fpx_max_representable(int exp_bits, int man_bits);
uint16_t fpx_effective_scale(uint16_t row_scale, int exp_bits, int man_bits);
uint32_t fpx_pad64(uint32_t n);
/* Bytes of segment `seg` of a rows_p x cols_p packed matrix (512*w per tile). */
size_t fpx_stream_bytes(uint32_t rows_p, uint32_t cols_p, int width);
/* Scalar codec (host): exact value of a code (FPX_ERR_INVALID_CODE if it has
 * bits above the format's width) / nearest code, ties to even, saturating
 * (FPX_ERR_INVALID_VALUE for NaN). */
int fpx_decode_scalar(uint32_t code, int exp_bits, int man_bits, float* value);
int fpx_encode_scalar(double value, int exp_bits, int man_bits, uint32_t* code);

/* ---- K0: quantize (codec.cpp:105-177) --------------------------------
 * w: rows x cols row-major, dtype FPX_FP32 or FPX_FP16 (device).
 * codes: pad64(rows) x pad64(cols) bytes; scales: pad64(rows) fp16 patterns.
 * Errors (first failing row in row order, like the reference):
 *   FPX_ERR_INVALID_VALUE (NaN in row), FPX_ERR_SCALE_OVERFLOW.
 * status_dev: optional device uint64 receiving (row << 8 | status) of the
 * first failing row, or UINT64_MAX; when NULL the call synchronises. */
int fpx_quantize(const void* w, int dtype, uint32_t rows, uint32_t cols, int exp_bits, int man_bits,
                 uint8_t* codes, uint16_t* scales, uint64_t* status_dev, fpx_stream_t stream);

/* ---- dequantize_reference from the code matrix (codec.cpp:179-193) -----
 * w_f16[r][c] = fp16(decode(codes[r][c])) * scales[r] in fp16 RNE, bit-exact,
 * rows_p x cols_p row-major (codes and w_f16 16-byte aligned).  A code with
 * bits above the format's width is FPX_ERR_INVALID_CODE (first failing row;
 * status_dev as in fpx_quantize, NULL = synchronous). */
int fpx_dequantize_codes(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p, int exp_bits,
                         int man_bits, uint16_t* w_f16, uint64_t* status_dev, fpx_stream_t stream);

/* ---- K0+K1 fused: quantize straight into the packed streams
 * Bit-exact with fpx_quantize followed by fpx_prepack (same scales, same
 * stream bytes, same first-failing-row errors), without the code matrix in
 * HBM: pass 1 computes row scales, pass 2 encodes each 64x64 tile into
 * shared memory and packs it.  streams[i]: fpx_stream_bytes(pad64(rows),
 * pad64(cols), widths[i]); widths/nseg NULL/0 -> the format's preset. */
int fpx_quantize_pack(const void* w, int dtype, uint32_t rows, uint32_t cols, int exp_bits, int man_bits,
                      const int* widths, int nseg, uint8_t* const* streams, uint16_t* scales, uint64_t* status_dev,
                      fpx_stream_t stream);

/* ---- K1: pre-pack (prepack.cpp:153-209) -------------------------------
 * codes: rows_p x cols_p (multiples of 64); widths/nseg: the split (NULL ->
 * the format's preset, format.cpp:59-69); streams[i]: device buffers of
 * fpx_stream_bytes(rows_p, cols_p, widths[i]).  scales (device) are checked
 * for a finite effective scale (prepack.cpp:165-168; synchronises). */
int fpx_prepack(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
                int exp_bits, int man_bits, const int* widths, int nseg, uint8_t* const* streams,
                fpx_stream_t stream);

/* ---- unpack (prepack.cpp:211-260) ------------------------------------- */
int fpx_unpack(const uint8_t* const* streams, uint32_t rows_p, uint32_t cols_p, int exp_bits,
               int man_bits, const int* widths, int nseg, uint8_t* codes, fpx_stream_t stream);

/* ---- K3: de-quantise to fp16 (codec.cpp:179-193, bit-exact) -----------
 * w_f16: rows_p x cols_p row-major fp16 patterns.  e3m2/e2m3 [2,4] and
 * e2m2 [4,1] run the fused kernel's register path; other formats a LUT. */
int fpx_dequantize(const uint8_t* const* streams, int nseg, const int* widths,
                   const uint16_t* scales, uint32_t rows_p, uint32_t cols_p, int exp_bits,
                   int man_bits, uint16_t* w_f16, fpx_stream_t stream);

/* ---- K2: fused FPx linear (gemm.cpp:170-219) ---------------------------
 * C(m, j) = sum_k dequant(W)(m, k) * act(k, j): W packed rows_p x cols_p,
 * act fp16 col-major k_act x n with k_act == cols_p or the original cols
 * (zero-extended, gemm.cpp:15-30), C fp32 col-major, C(m,j) at
 * c[j*ldc + m] for m < rows_p (ldc >= rows_p).
 * split_k: K chunks per 128-row tile; 0 = fpx_linear_default_split().  The
 * result depends only on (W, act, split_k) -- never on scheduling -- so a
 * tile-row shard computed with the full problem's split_k is bit-identical
 * to the same rows of the unsharded result.
 * workspace: device buffer of >= fpx_linear_workspace_size(...) bytes
 * (never NULL: it always holds the 64 KiB split-K arrival-counter table;
 * with FPX_LINEAR_X8=1 it also holds the activations' e4m3 split for the
 * opt-in kind::f8f6f4 kernel at n <= 32, which runs only when the buffer is
 * that large),
 * zero-filled once before first use; the counters self-clean after every
 * launch.  ONE WORKSPACE PER STREAM: two calls that may run concurrently
 * (distinct streams) must not share a workspace.  A call whose launch fails
 * clears the counters itself; fpx_linear_workspace_reset() clears them
 * explicitly (e.g. after a workspace was reused for other data).
 * Launch overlap (n <= 128, the decode kernel): the kernel uses programmatic
 * dependent launch, so it starts while the preceding kernel in the stream
 * drains.  With FPX_LINEAR_PDL unset or 2 it already streams (and
 * de-quantises) the packed weights and row scales then -- they must not be
 * written by a preceding kernel that triggers dependents early
 * (griddepcontrol.launch_dependents); weights are static in inference.  This
 * library's own weight writers (fpx_quantize, fpx_quantize_pack,
 * fpx_prepack) are guarded: the next linear on the same stream defers every
 * read until they completed.  Activations, C and the workspace are only
 * touched after the preceding kernel completed.  FPX_LINEAR_PDL=1 defers
 * every global access until then; 0 disables the overlap. */
int fpx_linear_default_split(uint32_t rows_p, uint32_t cols_p, uint32_t n);
size_t fpx_linear_workspace_size(uint32_t rows_p, uint32_t cols_p, uint32_t k_act, uint32_t n, int split_k);
int fpx_linear_workspace_reset(void* workspace, size_t workspace_bytes, fpx_stream_t stream);
int fpx_linear(const uint8_t* const* streams, int nseg, const uint16_t* scales, uint32_t rows_p,
               uint32_t cols_p, int exp_bits, int man_bits, const uint16_t* act, uint32_t k_act, uint32_t n,
               float* c, uint32_t ldc, int split_k, void* workspace, size_t workspace_bytes,
               fpx_stream_t stream);

/* ---- multi-GPU helpers (tile-row / output-channel sharding) -----------
 * Contiguous tile-row range [*tr0, *tr1) of rank `rank` of `world` for a
 * matrix of rows_p rows (balanced to within one tile-row). */
void fpx_shard_rows(uint32_t rows_p, int rank, int world, uint32_t* tr0, uint32_t* tr1);
/* gathered: [world][n][m_slot] fp32 (device, e.g. from ncclAllGather of each
 * rank's col-major slice padded to m_slot rows); row0/nrows: device arrays
 * of per-rank first row / row count.  Writes col-major c (ldc). */
int fpx_gather_permute(const float* gathered, const uint32_t* row0, const uint32_t* nrows, int world,
                       uint32_t m_slot, uint32_t n, float* c, uint32_t ldc, fpx_stream_t stream);

/* Sharded linear (SURVEY §8b fpx_linear_sharded, §8e): rank `rank` of
 * `world` holds tile-rows fpx_shard_rows(rows_p, rank, world) of the packed
 * weight (shard_streams / shard_scales = that contiguous byte range, zero
 * copy); every rank passes the same activations and receives the FULL
 * col-major C (rows_p x n, ldc).  split_k 0 runs the shard with the full
 * problem's split (fpx_linear_default_split(rows_p, cols_p, n)), so its rows
 * are bit-identical to a 1-GPU call; -1 picks the split that suits the shard
 * (the per-rank default; within the usual tolerance of a 1-GPU call, and
 * what scales: the full problem's split can leave most SMs of a small shard
 * idle); > 0 is used as given.  The slices are all-gathered over NVLink
 * with ncclAllGather on `stream` (nccl_comm: the caller's ncclComm_t) and
 * scattered into C.  NCCL is resolved at run time, no link dependency:
 * FPX_NCCL_LIB if set, else the one libnccl already mapped into the process
 * (e.g. torch's), else libnccl.so.2; two different libnccl files mapped at
 * once is refused (FPX_ERR_DEVICE) rather than guessed.  world == 1 needs
 * no communicator. */
size_t fpx_linear_sharded_workspace_size(uint32_t rows_p, uint32_t cols_p, uint32_t k_act, uint32_t n, int world,
                                         int split_k);
int fpx_linear_sharded(const uint8_t* const* shard_streams, int nseg, const uint16_t* shard_scales, uint32_t rows_p,
                       uint32_t cols_p, int exp_bits, int man_bits, const uint16_t* act, uint32_t k_act, uint32_t n,
                       float* c, uint32_t ldc, int split_k, int rank, int world, void* nccl_comm, void* workspace,
                       size_t workspace_bytes, fpx_stream_t stream);

/* ---- K2 with a fused epilogue ---------------------------
 * The paper positions its kernel as a drop-in linear with fp16 activations
 * in and out.  fpx_linear_ex computes, per output element,
 *   C(m, j) = act( sum_k dequant(W)(m, k) * act(k, j) + bias[m] ) + residual(m, j)
 * in fp32 and stores it as out_dtype (fp16: round-to-nearest-even).  c and
 * residual share the dtype, the col-major layout and ldc.  epi == NULL is
 * fpx_linear.  Activations: SiLU x*sigmoid(x), GELU tanh approximation. */
enum fpx_activation { FPX_ACT_NONE = 0, FPX_ACT_RELU = 1, FPX_ACT_SILU = 2, FPX_ACT_GELU_TANH = 3 };
typedef struct fpx_epilogue {
    int out_dtype;          /* FPX_FP32 or FPX_FP16 */
    const float* bias;      /* rows_p fp32, or NULL */
    int activation;         /* enum fpx_activation */
    const void* residual;   /* same dtype / layout / ldc as c, or NULL */
} fpx_epilogue;
int fpx_linear_ex(const uint8_t* const* streams, int nseg, const uint16_t* scales, uint32_t rows_p,
                  uint32_t cols_p, int exp_bits, int man_bits, const uint16_t* act, uint32_t k_act, uint32_t n,
                  void* c, uint32_t ldc, int split_k, const fpx_epilogue* epi, void* workspace,
                  size_t workspace_bytes, fpx_stream_t stream);

/* ---- PackFile container (io.hpp:13-41, SPEC.md model-io; host only) ----
 * "FPXPACK1" | u16 version=1 | u8 exp_bits | u8 man_bits | u8 nseg |
 * u8 widths[nseg] (high bits first) | u32 orig_rows, orig_cols, padded_rows,
 * padded_cols, tile_m=64, tile_k=64 | u8 scale granularity=0 |
 * u16 scales[padded_rows] | per segment: u64 length + stream bytes.
 * Little-endian throughout.  The reference declares this container
 * (io.hpp:36-37 write_pack_file / read_pack_file) but never implements it.
 * Errors: FPX_ERR_BAD_MAGIC, _BAD_VERSION, _TRUNCATED, _CORRUPT (length /
 * size-law / dimension violations, trailing bytes), _UNSUPPORTED_SPLIT,
 * _INVALID_FORMAT, _IO_FAILURE; fpx_last_error_offset() names the byte. */
typedef struct fpx_pack_header {
    int exp_bits, man_bits, nseg;
    int widths[3];
    uint32_t orig_rows, orig_cols, rows_p, cols_p;
    uint64_t scales_offset;     /* file offset of scales[0] */
    uint64_t stream_offset[3];  /* file offset of each stream's first byte */
    uint64_t stream_bytes[3];
    uint64_t file_bytes;
} fpx_pack_header;
size_t fpx_packfile_bytes(uint32_t rows_p, uint32_t cols_p, const int* widths, int nseg);
/* Serialise host buffers into out[0 .. fpx_packfile_bytes()). */
int fpx_packfile_encode(int exp_bits, int man_bits, const int* widths, int nseg, uint32_t orig_rows,
                        uint32_t orig_cols, uint32_t rows_p, uint32_t cols_p, const uint16_t* scales,
                        const uint8_t* const* streams, uint8_t* out, size_t out_bytes);
/* Validate a complete in-memory file and describe it. */
int fpx_packfile_parse(const uint8_t* bytes, size_t nbytes, fpx_pack_header* hdr);
/* Validate the file at `path` (header, size law, stream lengths, total size)
 * and, unless scales_dev is NULL (header only), copy its scales and streams
 * straight into the caller's device buffers on `stream` through pinned
 * staging (synchronous on return). */
int fpx_packfile_load(const char* path, fpx_pack_header* hdr, uint16_t* scales_dev, uint8_t* const* streams_dev,
                      fpx_stream_t stream);

/* ---- debug ------------------------------------------------------------
 * Only a tracing build records anything (make -C paper_2401_14112_b200 trace
 * -> libfpx_b200_trace.so); the production library compiles the device-side
 * stamps out.  With FPX_LINEAR_TRACE=1 in the environment, every fpx_linear launch records
 * clock64 stamps of CTA 0's pipeline events (7 events x 512 stages, row-major)
 * which this call copies to host (synchronous). */
int fpx_debug_trace(uint64_t* host, size_t words);
/* With FPX_LINEAR_TRACE=3: host pointer (mapped, pinned) to 300 x 32 words,
 * word [cta*32 + warp] = what that warp of the most recent fpx_linear launch
 * is waiting on (bit 63 set, tag<<56 | stage<<32 | smem_addr<<1 | parity), 0 if
 * not waiting; NULL otherwise.  For diagnosing a stuck launch. */
const volatile uint64_t* fpx_debug_progress(void);

#ifdef __cplusplus
}
#endif

#endif /* FPX_C_H_ */
