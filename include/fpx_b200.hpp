// fpx_b200.hpp -- C++ drop-in for the reference library's public API
// (/root/reference/proj/include/fpx/{format,error,codec,prepack,gemm}.hpp),
// served by the sm_100a kernels of libfpx_b200.so through include/fpx_c.h.
//
// Same namespace, type names, member layout, function signatures and error
// behaviour (fpx::Error carrying fpx::ErrorCode) as the reference, so a caller
// of the reference recompiles against this header and links libfpx_b200.so
// instead.  Value types keep their host std::vector payloads; each call
// uploads, runs on the device and downloads.  For repeated use of the same
// weights (inference), DeviceLinear keeps the packed streams resident in HBM.
//
// Reference declarations mirrored here:
//   FpxFormat / SplitScheme          format.hpp:16-59
//   ErrorCode / Error                error.hpp:10-44
//   Dtype / Layout / ScalarMatrix    codec.hpp:10-30
//   half_to_float / float_to_half / half_mul / half_is_finite / half_is_nan
//                                    half.hpp:9-21 (host scalar helpers)
//   QuantizedMatrix                  codec.hpp:37-51
//   decode_scalar / encode_scalar    codec.hpp:56,60 (host scalar codec)
//   quantize_matrix / effective_scale codec.hpp:66,76
//   dequantize_reference             codec.hpp:72 (on the device, bit-exact)
//   PackedWeights / pack / unpack    prepack.hpp:64-86
//   gemm_packed                      gemm.hpp:27-28 (trace pointer: the
//                                    bank-conflict trace is a CPU-simulator
//                                    artefact; a non-null trace is rejected)
//   gemm_reference                   gemm.hpp:32: pack + the same fused
//                                    kernel, so gemm_reference(q, b) ==
//                                    gemm_packed(pack(q), b) bit for bit -- the
//                                    reference's own contract (gemm.hpp:30-31)
//   io.hpp:13-41                     MatrixFile / PackFile containers
// Reference-style includes ("fpx/codec.hpp", "fpx/gemm.hpp", ...) resolve to
// this header through include/fpx/*.hpp.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <filesystem>
#include <vector>

namespace fpx {

// ------------------------------------------------------------------ errors
enum class ErrorCode {
    InvalidFormat,
    InvalidCode,
    InvalidValue,
    ScaleOverflow,
    ShapeMismatch,
    RaggedInput,
    UnsupportedSplit,
    IndexOutOfRange,
    BadMagic,
    BadVersion,
    Truncated,
    Corrupt,
    IoFailure,
};

const char* error_code_name(ErrorCode c);

class Error : public std::runtime_error {
public:
    Error(ErrorCode code, const std::string& message) : std::runtime_error(message), code_(code) {}
    Error(ErrorCode code, const std::string& message, uint64_t offset)
        : std::runtime_error(message), code_(code), offset_(offset) {}
    ErrorCode code() const { return code_; }
    std::optional<uint64_t> offset() const { return offset_; }
    std::string formatted() const;

private:
    ErrorCode code_;
    std::optional<uint64_t> offset_;
};

// Device / runtime failures that have no reference ErrorCode (no sm_100
// GPU, CUDA errors).  Derives from std::runtime_error, not fpx::Error.
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ formats
struct FpxFormat {
    int exp_bits = 3;
    int man_bits = 2;

    int total_bits() const { return 1 + exp_bits + man_bits; }
    int bias() const { return (1 << (exp_bits - 1)) - 1; }
    uint32_t code_count() const { return 1u << total_bits(); }
    uint32_t code_mask() const { return code_count() - 1; }
    uint32_t sign_mask() const { return 1u << (exp_bits + man_bits); }
    float max_representable() const;
    // Code spacing at |x|: 2^(e-M), e = floor(log2|x|) clamped to [1-bias, emax].
    float ulp_at(double magnitude) const;
    std::string name() const;
    bool operator==(const FpxFormat&) const = default;

    static FpxFormat e3m2() { return {3, 2}; }
    static FpxFormat e2m3() { return {2, 3}; }
    static FpxFormat e2m2() { return {2, 2}; }
    static FpxFormat e2m1() { return {2, 1}; }
    static FpxFormat make(int exp_bits, int man_bits);
    static std::optional<FpxFormat> parse(std::string_view name);
};

struct SplitScheme {
    std::vector<int> widths;
    int total() const;
    size_t segment_count() const { return widths.size(); }
    bool operator==(const SplitScheme&) const = default;
    static SplitScheme for_format(const FpxFormat& fmt);
    static SplitScheme make(std::vector<int> widths, const FpxFormat& fmt);
};

// ------------------------------------------------------------------ half.hpp
float half_to_float(uint16_t h);
uint16_t float_to_half(float f);          // RNE, subnormals kept, overflow -> inf
uint16_t half_mul(uint16_t a, uint16_t b);  // fp32 product (exact) rounded RNE to fp16
constexpr bool half_is_finite(uint16_t h) { return (h & 0x7c00u) != 0x7c00u; }
constexpr bool half_is_nan(uint16_t h) { return (h & 0x7c00u) == 0x7c00u && (h & 0x03ffu) != 0; }

// ------------------------------------------------------------------ matrices
enum class Dtype : uint32_t { Fp32 = 0, Fp16 = 1 };
enum class Layout : uint8_t { RowMajor = 0, ColMajor = 1 };

struct ScalarMatrix {
    Dtype dtype = Dtype::Fp32;
    Layout layout = Layout::RowMajor;
    uint32_t rows = 0;
    uint32_t cols = 0;
    std::vector<float> f32;
    std::vector<uint16_t> f16;

    size_t element_count() const { return size_t(rows) * cols; }
    size_t index(uint32_t r, uint32_t c) const {
        return layout == Layout::RowMajor ? size_t(r) * cols + c : size_t(c) * rows + r;
    }
    static ScalarMatrix zeros(Dtype dt, Layout lo, uint32_t rows, uint32_t cols);
};

struct QuantizedMatrix {
    FpxFormat format;
    uint32_t rows = 0;  // padded to 64
    uint32_t cols = 0;  // padded to 64
    uint32_t orig_rows = 0;
    uint32_t orig_cols = 0;
    std::vector<uint8_t> codes;    // row-major, one code per byte
    std::vector<uint16_t> scales;  // fp16 bits per padded row
    uint8_t code_at(uint32_t r, uint32_t c) const { return codes[size_t(r) * cols + c]; }
    bool operator==(const QuantizedMatrix&) const = default;
};

// prepack.hpp:15-21 tiling constants
inline constexpr uint32_t kTileDim = 64;
inline constexpr uint32_t kSlicesPerTile = 4;
inline constexpr uint32_t kChunksPerSlice = 4;
inline constexpr uint32_t kPairsPerChunk = 4;
inline constexpr uint32_t kWarpSize = 32;
inline constexpr uint32_t kCodesPerThread = 128;
inline constexpr uint32_t kCodesPerThreadSlice = 32;

struct PackedWeights {
    FpxFormat format;
    SplitScheme split;
    uint32_t rows = 0;
    uint32_t cols = 0;
    uint32_t orig_rows = 0;
    uint32_t orig_cols = 0;
    std::vector<std::vector<uint8_t>> streams;  // one per segment, 512*w bytes per tile
    std::vector<uint16_t> scales;
    uint32_t tile_rows() const { return rows / 64; }
    uint32_t tile_cols() const { return cols / 64; }
    static size_t tile_stream_bytes(int w) { return size_t(512) * w; }
    bool operator==(const PackedWeights&) const = default;
};

struct BankAccessTrace;  // reference simulator type; not supported on the GPU path

// ------------------------------------------------------------------ API
ScalarMatrix to_fp32(const ScalarMatrix& m);
ScalarMatrix to_fp16(const ScalarMatrix& m);
// Exact value of a code (InvalidCode if it has bits above the format's width).
float decode_scalar(uint32_t code, const FpxFormat& fmt);
// Nearest code, ties to even, saturating; InvalidValue on NaN.
uint32_t encode_scalar(double value, const FpxFormat& fmt);
QuantizedMatrix quantize_matrix(const ScalarMatrix& m, const FpxFormat& fmt);
// fp16 row-major padded W = fp16(decode(code)) x scale, fp16 RNE (K3 on the device).
ScalarMatrix dequantize_reference(const QuantizedMatrix& q);
uint16_t effective_scale(uint16_t row_scale, const FpxFormat& fmt);
PackedWeights pack(const QuantizedMatrix& q);
PackedWeights pack(const QuantizedMatrix& q, const SplitScheme& split);
QuantizedMatrix unpack(const PackedWeights& p);
// fp16 row-major (padded) W, bit-exact with the reference's
// dequantize_reference(unpack(p)).
ScalarMatrix dequantize(const PackedWeights& p);
// C fp32 col-major (padded rows x n) = dequant(A) x B, B fp16 col-major.
ScalarMatrix gemm_packed(const PackedWeights& a, const ScalarMatrix& b, BankAccessTrace* trace = nullptr);
// Same C as gemm_packed(pack(q), b), bit for bit (gemm.hpp:30-32).
ScalarMatrix gemm_reference(const QuantizedMatrix& q, const ScalarMatrix& b);

inline constexpr char kMatrixMagic[8] = {'F', 'P', 'X', 'M', 'A', 'T', '1', 0};
inline constexpr char kPackMagic[8] = {'F', 'P', 'X', 'P', 'A', 'C', 'K', '1'};
inline constexpr uint16_t kPackVersion = 1;
// io.hpp:27-41 -- MatrixFile ("FPXMAT1\0") and PackFile ("FPXPACK1")
// containers, little-endian, strict validation (Truncated / BadMagic /
// BadVersion / Corrupt errors carry the byte offset).
std::vector<uint8_t> serialize_matrix(const ScalarMatrix& m);
ScalarMatrix deserialize_matrix(const std::vector<uint8_t>& bytes);
std::vector<uint8_t> serialize_packed(const PackedWeights& p);
PackedWeights deserialize_packed(const std::vector<uint8_t>& bytes);
void write_matrix_file(const std::filesystem::path& path, const ScalarMatrix& m);
ScalarMatrix read_matrix_file(const std::filesystem::path& path);
void write_pack_file(const std::filesystem::path& path, const PackedWeights& p);
PackedWeights read_pack_file(const std::filesystem::path& path);
ScalarMatrix read_raw_blob(const std::filesystem::path& path, Dtype dtype, uint32_t rows, uint32_t cols);

// Weights resident in HBM for repeated linears (the inference use).
class DeviceLinear {
public:
    explicit DeviceLinear(const PackedWeights& p, int split_k = 0);
    ~DeviceLinear();
    DeviceLinear(const DeviceLinear&) = delete;
    DeviceLinear& operator=(const DeviceLinear&) = delete;
    ScalarMatrix forward(const ScalarMatrix& b);
    uint32_t rows() const { return rows_; }
    uint32_t cols() const { return cols_; }

private:
    FpxFormat format_;
    uint32_t rows_ = 0, cols_ = 0, orig_cols_ = 0;
    int split_k_ = 0;
    std::vector<void*> d_streams_;
    void* d_scales_ = nullptr;
    void* d_ws_ = nullptr;
    size_t ws_bytes_ = 0;
};

}  // namespace fpx
