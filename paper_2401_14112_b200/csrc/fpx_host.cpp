// fpx_host.cpp -- the C++ drop-in API of include/fpx_b200.hpp, implemented
// over the C-ABI (include/fpx_c.h).  Host value types in, host value types
// out; every computation runs in the sm_100a kernels.  Argument checks and
// messages follow the reference (codec.cpp:105-110, prepack.cpp:157-168,
// gemm.cpp:20-30) so callers see the same fpx::Error codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>

#include "fpx_b200.hpp"
#include "fpx_c.h"

namespace fpx {

namespace {

[[noreturn]] void throw_status(int st) {
    std::string msg = fpx_last_error();
    // the C-ABI message is "error[<name>] text"; fpx::Error keeps the text
    if (msg.rfind("error[", 0) == 0) {
        const size_t close = msg.find("] ");
        if (close != std::string::npos) msg = msg.substr(close + 2);
    }
    const int64_t off = fpx_last_error_offset();
    if (off >= 0) {
        const std::string suffix = " (at byte " + std::to_string(off) + ")";
        if (msg.size() >= suffix.size() && msg.compare(msg.size() - suffix.size(), suffix.size(), suffix) == 0)
            msg.resize(msg.size() - suffix.size());
        if (st >= 1 && st <= 13) throw Error(static_cast<ErrorCode>(st - 1), msg, static_cast<uint64_t>(off));
    }
    if (st >= 1 && st <= 13) throw Error(static_cast<ErrorCode>(st - 1), msg);
    throw DeviceError(std::string("error[") + fpx_status_name(st) + "] " + msg);
}

void check(int st) {
    if (st != 0) throw_status(st);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(std::string("error[cuda] ") + what + ": " + cudaGetErrorString(e));
}

// RAII device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t bytes) : n(bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void upload(const void* src, size_t bytes) {
        if (bytes) cuda_check(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    void download(void* dst, size_t bytes) const {
        if (bytes) cuda_check(cudaMemcpy(dst, p, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }
};

}  // namespace

// ------------------------------------------------------------------ half.hpp
// half.cpp:7-70 semantics: exact widening, RNE narrowing with subnormals,
// multiply = exact fp32 product narrowed once.
uint16_t float_to_half(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint16_t s = static_cast<uint16_t>((x >> 16) & 0x8000u);
    const uint32_t a = x & 0x7fffffffu;
    if (a >= 0x7f800000u) return a > 0x7f800000u ? uint16_t(s | 0x7e00u | ((a & 0x7fffffu) >> 13)) : uint16_t(s | 0x7c00u);
    const int e16 = int(a >> 23) - 112;
    if (e16 >= 31) return s | 0x7c00u;
    const uint32_t sig = (a & 0x7fffffu) | 0x800000u;
    int drop;
    uint32_t base;
    if (e16 >= 1) {
        drop = 13;
        base = (uint32_t(e16) << 10) | ((sig >> 13) & 0x3ffu);
    } else {
        if (e16 < -10) return s;
        drop = 14 - e16;
        base = sig >> drop;
    }
    const uint32_t rem = sig & ((1u << drop) - 1u), half = 1u << (drop - 1);
    if (rem > half || (rem == half && (base & 1u))) ++base;
    return static_cast<uint16_t>(s | base);
}

float half_to_float(uint16_t h) {
    const uint32_t s = uint32_t(h & 0x8000u) << 16, e = (h >> 10) & 31u, m = h & 1023u;
    float v;
    if (e == 0) v = std::ldexp(float(m), -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = std::ldexp(float(1024 + m), int(e) - 25);
    uint32_t bits;
    std::memcpy(&bits, &v, 4);
    bits |= s;
    std::memcpy(&v, &bits, 4);
    return v;
}

uint16_t half_mul(uint16_t a, uint16_t b) { return float_to_half(half_to_float(a) * half_to_float(b)); }

// ------------------------------------------------------------------ errors
const char* error_code_name(ErrorCode c) { return fpx_status_name(static_cast<int>(c) + 1); }

std::string Error::formatted() const {
    std::string s = std::string("error[") + error_code_name(code_) + "] " + what();
    if (offset_) s += " (at byte " + std::to_string(*offset_) + ")";
    return s;
}

// ------------------------------------------------------------------ formats
float FpxFormat::max_representable() const { return fpx_max_representable(exp_bits, man_bits); }

float FpxFormat::ulp_at(double magnitude) const {
    magnitude = std::fabs(magnitude);
    const int e_min = 1 - bias(), e_max = (1 << exp_bits) - 1 - bias();
    int e = e_min;
    if (magnitude >= std::ldexp(1.0, e_min)) e = std::min(static_cast<int>(std::floor(std::log2(magnitude))), e_max);
    return static_cast<float>(std::ldexp(1.0, e - man_bits));
}

std::string FpxFormat::name() const { return "e" + std::to_string(exp_bits) + "m" + std::to_string(man_bits); }

FpxFormat FpxFormat::make(int e, int m) {
    check(fpx_format_check(e, m));
    return {e, m};
}

std::optional<FpxFormat> FpxFormat::parse(std::string_view name) {
    if (name.size() != 4 || name[0] != 'e' || name[2] != 'm' || name[1] < '0' || name[1] > '9' || name[3] < '0' ||
        name[3] > '9')
        return std::nullopt;
    const int e = name[1] - '0', m = name[3] - '0';
    if (fpx_format_check(e, m) != 0) return std::nullopt;
    return FpxFormat{e, m};
}

int SplitScheme::total() const {
    int t = 0;
    for (int w : widths) t += w;
    return t;
}

SplitScheme SplitScheme::for_format(const FpxFormat& fmt) {
    int w[3];
    const int n = fpx_split_for_format(fmt.exp_bits, fmt.man_bits, w);
    if (n == 0) throw Error(ErrorCode::InvalidFormat, "no split for " + fmt.name());
    return SplitScheme{std::vector<int>(w, w + n)};
}

SplitScheme SplitScheme::make(std::vector<int> widths, const FpxFormat& fmt) {
    SplitScheme s{std::move(widths)};
    for (int w : s.widths)
        if (w != 1 && w != 2 && w != 4) throw Error(ErrorCode::UnsupportedSplit, "segment widths must be 1, 2 or 4");
    if (s.total() != fmt.total_bits())
        throw Error(ErrorCode::UnsupportedSplit,
                    "segment widths must sum to " + std::to_string(fmt.total_bits()) + " for " + fmt.name());
    return s;
}

// ------------------------------------------------------------------ matrices
ScalarMatrix ScalarMatrix::zeros(Dtype dt, Layout lo, uint32_t rows, uint32_t cols) {
    ScalarMatrix m;
    m.dtype = dt;
    m.layout = lo;
    m.rows = rows;
    m.cols = cols;
    if (dt == Dtype::Fp32) m.f32.assign(size_t(rows) * cols, 0.0f);
    else m.f16.assign(size_t(rows) * cols, 0);
    return m;
}

ScalarMatrix to_fp32(const ScalarMatrix& m) {
    if (m.dtype == Dtype::Fp32) return m;
    ScalarMatrix out = ScalarMatrix::zeros(Dtype::Fp32, m.layout, m.rows, m.cols);
    for (size_t i = 0; i < m.f16.size(); ++i) out.f32[i] = half_to_float(m.f16[i]);
    return out;
}

ScalarMatrix to_fp16(const ScalarMatrix& m) {
    if (m.dtype == Dtype::Fp16) return m;
    ScalarMatrix out = ScalarMatrix::zeros(Dtype::Fp16, m.layout, m.rows, m.cols);
    for (size_t i = 0; i < m.f32.size(); ++i) out.f16[i] = float_to_half(m.f32[i]);
    return out;
}

float decode_scalar(uint32_t code, const FpxFormat& fmt) {
    float v = 0.0f;
    check(fpx_decode_scalar(code, fmt.exp_bits, fmt.man_bits, &v));
    return v;
}

uint32_t encode_scalar(double value, const FpxFormat& fmt) {
    uint32_t code = 0;
    check(fpx_encode_scalar(value, fmt.exp_bits, fmt.man_bits, &code));
    return code;
}

uint16_t effective_scale(uint16_t row_scale, const FpxFormat& fmt) {
    return fpx_effective_scale(row_scale, fmt.exp_bits, fmt.man_bits);
}

// ------------------------------------------------------------------ K0
QuantizedMatrix quantize_matrix(const ScalarMatrix& m, const FpxFormat& fmt) {
    if (m.dtype != Dtype::Fp32 || m.layout != Layout::RowMajor)
        throw Error(ErrorCode::InvalidValue, "quantize expects a row-major fp32 matrix");
    if (m.rows == 0 || m.cols == 0) throw Error(ErrorCode::ShapeMismatch, "empty matrix");
    QuantizedMatrix q;
    q.format = fmt;
    q.orig_rows = m.rows;
    q.orig_cols = m.cols;
    q.rows = fpx_pad64(m.rows);
    q.cols = fpx_pad64(m.cols);
    DevBuf w(m.element_count() * 4), codes(size_t(q.rows) * q.cols), scales(size_t(q.rows) * 2);
    w.upload(m.f32.data(), m.element_count() * 4);
    check(fpx_quantize(w.p, FPX_FP32, m.rows, m.cols, fmt.exp_bits, fmt.man_bits, codes.as<uint8_t>(),
                       scales.as<uint16_t>(), nullptr, nullptr));
    q.codes.resize(size_t(q.rows) * q.cols);
    q.scales.resize(q.rows);
    codes.download(q.codes.data(), q.codes.size());
    scales.download(q.scales.data(), q.scales.size() * 2);
    return q;
}

// ------------------------------------------------------------------ K1
PackedWeights pack(const QuantizedMatrix& q) { return pack(q, SplitScheme::for_format(q.format)); }

PackedWeights pack(const QuantizedMatrix& q, const SplitScheme& split) {
    if (q.rows == 0 || q.cols == 0 || q.rows % 64 || q.cols % 64)
        throw Error(ErrorCode::ShapeMismatch,
                    "matrix dims must be padded to multiples of 64 at quantize time before packing");
    if (split.total() != q.format.total_bits())
        throw Error(ErrorCode::UnsupportedSplit, "split widths do not cover " + q.format.name());
    PackedWeights p;
    p.format = q.format;
    p.split = split;
    p.rows = q.rows;
    p.cols = q.cols;
    p.orig_rows = q.orig_rows ? q.orig_rows : q.rows;
    p.orig_cols = q.orig_cols ? q.orig_cols : q.cols;
    p.scales = q.scales;
    DevBuf codes(q.codes.size()), scales(q.scales.size() * 2);
    codes.upload(q.codes.data(), q.codes.size());
    scales.upload(q.scales.data(), q.scales.size() * 2);
    std::vector<DevBuf*> outs;
    std::vector<uint8_t*> ptrs;
    for (int w : split.widths) {
        outs.push_back(new DevBuf(fpx_stream_bytes(q.rows, q.cols, w)));
        ptrs.push_back(outs.back()->as<uint8_t>());
    }
    const int st = fpx_prepack(codes.as<uint8_t>(), scales.as<uint16_t>(), q.rows, q.cols, q.format.exp_bits,
                               q.format.man_bits, split.widths.data(), int(split.widths.size()), ptrs.data(), nullptr);
    if (st == 0) {
        for (DevBuf* b : outs) {
            p.streams.emplace_back(b->n);
            b->download(p.streams.back().data(), b->n);
        }
    }
    for (DevBuf* b : outs) delete b;
    check(st);
    return p;
}

QuantizedMatrix unpack(const PackedWeights& p) {
    QuantizedMatrix q;
    q.format = p.format;
    q.rows = p.rows;
    q.cols = p.cols;
    q.orig_rows = p.orig_rows;
    q.orig_cols = p.orig_cols;
    q.scales = p.scales;
    std::vector<DevBuf*> ins;
    std::vector<const uint8_t*> ptrs;
    for (const auto& s : p.streams) {
        ins.push_back(new DevBuf(s.size()));
        ins.back()->upload(s.data(), s.size());
        ptrs.push_back(ins.back()->as<uint8_t>());
    }
    DevBuf codes(size_t(p.rows) * p.cols);
    const int st = fpx_unpack(ptrs.data(), p.rows, p.cols, p.format.exp_bits, p.format.man_bits,
                              p.split.widths.data(), int(p.split.widths.size()), codes.as<uint8_t>(), nullptr);
    for (DevBuf* b : ins) delete b;
    check(st);
    q.codes.resize(codes.n);
    codes.download(q.codes.data(), codes.n);
    return q;
}

// ------------------------------------------------------------------ K3
ScalarMatrix dequantize(const PackedWeights& p) {
    std::vector<DevBuf*> ins;
    std::vector<const uint8_t*> ptrs;
    for (const auto& s : p.streams) {
        ins.push_back(new DevBuf(s.size()));
        ins.back()->upload(s.data(), s.size());
        ptrs.push_back(ins.back()->as<uint8_t>());
    }
    DevBuf scales(p.scales.size() * 2), out(size_t(p.rows) * p.cols * 2);
    scales.upload(p.scales.data(), p.scales.size() * 2);
    const int st = fpx_dequantize(ptrs.data(), int(ptrs.size()), p.split.widths.data(), scales.as<uint16_t>(), p.rows,
                                  p.cols, p.format.exp_bits, p.format.man_bits, out.as<uint16_t>(), nullptr);
    for (DevBuf* b : ins) delete b;
    check(st);
    ScalarMatrix w = ScalarMatrix::zeros(Dtype::Fp16, Layout::RowMajor, p.rows, p.cols);
    out.download(w.f16.data(), w.f16.size() * 2);
    return w;
}

ScalarMatrix dequantize_reference(const QuantizedMatrix& q) {
    if (q.rows == 0 || q.cols == 0 || q.rows % 64 || q.cols % 64 || q.codes.size() != size_t(q.rows) * q.cols ||
        q.scales.size() != q.rows)
        throw Error(ErrorCode::ShapeMismatch, "quantized matrix must be padded to multiples of 64 with one scale per row");
    DevBuf codes(q.codes.size()), scales(q.scales.size() * 2), out(q.codes.size() * 2);
    codes.upload(q.codes.data(), q.codes.size());
    scales.upload(q.scales.data(), q.scales.size() * 2);
    check(fpx_dequantize_codes(codes.as<uint8_t>(), scales.as<uint16_t>(), q.rows, q.cols, q.format.exp_bits,
                               q.format.man_bits, out.as<uint16_t>(), nullptr, nullptr));
    ScalarMatrix w = ScalarMatrix::zeros(Dtype::Fp16, Layout::RowMajor, q.rows, q.cols);
    out.download(w.f16.data(), w.f16.size() * 2);
    return w;
}

// ------------------------------------------------------------------ K2
static void check_problem(uint32_t a_cols, uint32_t a_orig_cols, const ScalarMatrix& b) {
    if (b.dtype != Dtype::Fp16 || b.layout != Layout::ColMajor)
        throw Error(ErrorCode::ShapeMismatch, "activations must be fp16 col-major");
    if (b.rows != a_cols && b.rows != a_orig_cols)
        throw Error(ErrorCode::ShapeMismatch, "weight cols " + std::to_string(a_cols) + " (orig " +
                                                  std::to_string(a_orig_cols) + ") do not match activation rows " +
                                                  std::to_string(b.rows));
}

DeviceLinear::DeviceLinear(const PackedWeights& p, int split_k)
    : format_(p.format), rows_(p.rows), cols_(p.cols), orig_cols_(p.orig_cols), split_k_(split_k) {
    for (const auto& s : p.streams) {
        void* d = nullptr;
        cuda_check(cudaMalloc(&d, s.size()), "cudaMalloc");
        cuda_check(cudaMemcpy(d, s.data(), s.size(), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
        d_streams_.push_back(d);
    }
    cuda_check(cudaMalloc(&d_scales_, p.scales.size() * 2), "cudaMalloc");
    cuda_check(cudaMemcpy(d_scales_, p.scales.data(), p.scales.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
}

DeviceLinear::~DeviceLinear() {
    for (void* d : d_streams_) cudaFree(d);
    if (d_scales_) cudaFree(d_scales_);
    if (d_ws_) cudaFree(d_ws_);
}

ScalarMatrix DeviceLinear::forward(const ScalarMatrix& b) {
    check_problem(cols_, orig_cols_, b);
    const uint32_t n = b.cols;
    ScalarMatrix c = ScalarMatrix::zeros(Dtype::Fp32, Layout::ColMajor, rows_, n);
    if (n == 0) return c;
    const size_t need = fpx_linear_workspace_size(rows_, cols_, b.rows, n, split_k_) + 256;
    if (need > ws_bytes_) {
        if (d_ws_) cudaFree(d_ws_);
        cuda_check(cudaMalloc(&d_ws_, need), "cudaMalloc");
        cuda_check(cudaMemset(d_ws_, 0, need), "cudaMemset");  // counter table starts zeroed
        ws_bytes_ = need;
    }
    DevBuf act(b.f16.size() * 2), out(c.f32.size() * 4);
    act.upload(b.f16.data(), b.f16.size() * 2);
    std::vector<const uint8_t*> ptrs;
    for (void* d : d_streams_) ptrs.push_back(static_cast<const uint8_t*>(d));
    check(fpx_linear(ptrs.data(), int(ptrs.size()), static_cast<const uint16_t*>(d_scales_), rows_, cols_,
                     format_.exp_bits, format_.man_bits, act.as<uint16_t>(), b.rows, n, out.as<float>(), rows_,
                     split_k_, d_ws_, ws_bytes_, nullptr));
    out.download(c.f32.data(), c.f32.size() * 4);
    return c;
}

ScalarMatrix gemm_packed(const PackedWeights& a, const ScalarMatrix& b, BankAccessTrace* trace) {
    if (trace != nullptr)
        throw Error(ErrorCode::InvalidValue, "bank-access tracing is a CPU-simulator feature; pass nullptr");
    check_problem(a.cols, a.orig_cols, b);
    DeviceLinear lin(a);
    return lin.forward(b);
}

ScalarMatrix gemm_reference(const QuantizedMatrix& q, const ScalarMatrix& b) {
    check_problem(q.cols, q.orig_cols ? q.orig_cols : q.cols, b);
    return gemm_packed(pack(q), b);
}

// ------------------------------------------------------------------ io.hpp
// PackFile over the C-ABI container code (fpx_io.cpp); MatrixFile here.
// Both little-endian with strict validation (SPEC.md model-io).
namespace {
constexpr const char* kMatMagic = kMatrixMagic;

template <typename T>
void put(std::vector<uint8_t>& o, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) o.push_back(static_cast<uint8_t>(static_cast<uint64_t>(v) >> (8 * i)));
}
template <typename T>
T get(const std::vector<uint8_t>& b, size_t& off, const char* what) {
    if (b.size() < off || b.size() - off < sizeof(T))
        throw Error(ErrorCode::Truncated, std::string("matrix file ends inside ") + what, off);
    uint64_t x = 0;
    for (size_t i = 0; i < sizeof(T); ++i) x |= static_cast<uint64_t>(b[off + i]) << (8 * i);
    off += sizeof(T);
    return static_cast<T>(x);
}
std::vector<uint8_t> read_all(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw Error(ErrorCode::IoFailure, "cannot open " + path.string());
    return std::vector<uint8_t>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}
void write_all(const std::filesystem::path& path, const std::vector<uint8_t>& b) {
    std::ofstream f(path, std::ios::binary);
    if (!f || !f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size())))
        throw Error(ErrorCode::IoFailure, "cannot write " + path.string());
}
}  // namespace

std::vector<uint8_t> serialize_matrix(const ScalarMatrix& m) {
    std::vector<uint8_t> o(kMatMagic, kMatMagic + 8);
    put<uint32_t>(o, static_cast<uint32_t>(m.dtype));
    put<uint32_t>(o, m.rows);
    put<uint32_t>(o, m.cols);
    put<uint8_t>(o, static_cast<uint8_t>(m.layout));
    for (int i = 0; i < 3; ++i) put<uint8_t>(o, 0);
    if (m.dtype == Dtype::Fp32)
        for (float v : m.f32) {
            uint32_t u;
            std::memcpy(&u, &v, 4);
            put<uint32_t>(o, u);
        }
    else
        for (uint16_t v : m.f16) put<uint16_t>(o, v);
    return o;
}

ScalarMatrix deserialize_matrix(const std::vector<uint8_t>& b) {
    if (b.size() < 8) throw Error(ErrorCode::Truncated, "matrix file ends inside the magic", 0);
    if (std::memcmp(b.data(), kMatMagic, 8) != 0) throw Error(ErrorCode::BadMagic, "not an FPXMAT1 file", 0);
    size_t off = 8;
    const uint32_t dt = get<uint32_t>(b, off, "the dtype");
    if (dt > 1) throw Error(ErrorCode::Corrupt, "dtype " + std::to_string(dt), 8);
    const uint32_t rows = get<uint32_t>(b, off, "the dimensions"), cols = get<uint32_t>(b, off, "the dimensions");
    const uint8_t lo = get<uint8_t>(b, off, "the layout");
    if (lo > 1) throw Error(ErrorCode::Corrupt, "layout " + std::to_string(lo), off - 1);
    off += 3;
    const size_t es = dt == 0 ? 4 : 2, n = size_t(rows) * cols;
    if (b.size() < off || b.size() - off < n * es)
        throw Error(ErrorCode::Truncated, "matrix file ends inside the payload", b.size());
    if (b.size() - off != n * es) throw Error(ErrorCode::Corrupt, "trailing bytes after the payload", off + n * es);
    ScalarMatrix m = ScalarMatrix::zeros(static_cast<Dtype>(dt), static_cast<Layout>(lo), rows, cols);
    if (dt == 0)
        std::memcpy(m.f32.data(), b.data() + off, n * 4);  // little-endian host (x86-64 / aarch64)
    else
        std::memcpy(m.f16.data(), b.data() + off, n * 2);
    return m;
}

std::vector<uint8_t> serialize_packed(const PackedWeights& p) {
    const int nseg = static_cast<int>(p.split.widths.size());
    std::vector<const uint8_t*> sp;
    for (const auto& s : p.streams) sp.push_back(s.data());
    std::vector<uint8_t> out(fpx_packfile_bytes(p.rows, p.cols, p.split.widths.data(), nseg));
    for (int i = 0; i < nseg; ++i)
        if (i >= static_cast<int>(p.streams.size()) ||
            p.streams[i].size() != fpx_stream_bytes(p.rows, p.cols, p.split.widths[i]))
            throw Error(ErrorCode::ShapeMismatch, "stream " + std::to_string(i) + " does not match the size law");
    if (p.scales.size() != p.rows) throw Error(ErrorCode::ShapeMismatch, "one scale per padded row");
    check(fpx_packfile_encode(p.format.exp_bits, p.format.man_bits, p.split.widths.data(), nseg, p.orig_rows,
                              p.orig_cols, p.rows, p.cols, p.scales.data(), sp.data(), out.data(), out.size()));
    return out;
}

PackedWeights deserialize_packed(const std::vector<uint8_t>& b) {
    fpx_pack_header h;
    check(fpx_packfile_parse(b.data(), b.size(), &h));
    PackedWeights p;
    p.format = FpxFormat::make(h.exp_bits, h.man_bits);
    p.split = SplitScheme::make(std::vector<int>(h.widths, h.widths + h.nseg), p.format);
    p.rows = h.rows_p;
    p.cols = h.cols_p;
    p.orig_rows = h.orig_rows;
    p.orig_cols = h.orig_cols;
    p.scales.resize(h.rows_p);
    std::memcpy(p.scales.data(), b.data() + h.scales_offset, size_t(h.rows_p) * 2);
    for (int i = 0; i < h.nseg; ++i)
        p.streams.emplace_back(b.begin() + static_cast<std::ptrdiff_t>(h.stream_offset[i]),
                               b.begin() + static_cast<std::ptrdiff_t>(h.stream_offset[i] + h.stream_bytes[i]));
    return p;
}

void write_matrix_file(const std::filesystem::path& path, const ScalarMatrix& m) { write_all(path, serialize_matrix(m)); }
ScalarMatrix read_matrix_file(const std::filesystem::path& path) { return deserialize_matrix(read_all(path)); }
void write_pack_file(const std::filesystem::path& path, const PackedWeights& p) { write_all(path, serialize_packed(p)); }
PackedWeights read_pack_file(const std::filesystem::path& path) { return deserialize_packed(read_all(path)); }

ScalarMatrix read_raw_blob(const std::filesystem::path& path, Dtype dtype, uint32_t rows, uint32_t cols) {
    const std::vector<uint8_t> b = read_all(path);
    const size_t es = dtype == Dtype::Fp32 ? 4 : 2, n = size_t(rows) * cols;
    if (b.size() != n * es)
        throw Error(b.size() < n * es ? ErrorCode::Truncated : ErrorCode::Corrupt,
                    "raw blob holds " + std::to_string(b.size()) + " bytes, expected " + std::to_string(n * es),
                    std::min(b.size(), n * es));
    ScalarMatrix m = ScalarMatrix::zeros(dtype, Layout::RowMajor, rows, cols);
    if (dtype == Dtype::Fp32) std::memcpy(m.f32.data(), b.data(), n * 4);
    else std::memcpy(m.f16.data(), b.data(), n * 2);
    return m;
}

}  // namespace fpx
