// fpx_capi.cu -- implementation of the C-ABI in include/fpx_c.h: argument
// validation with the reference's error codes/messages, tensor-map encoding,
// workspace carving, and dispatch to the sm_100a kernels.  No exception and
// no host compute fallback: if the device or a kernel is unavailable the
// call fails with FPX_ERR_DEVICE / FPX_ERR_CUDA.
#include <dlfcn.h>
#include <link.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fpx_c.h"
#include "fpx_internal.h"
#include "fpx_kernels.h"

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_last_offset = -1;

const char* kNames[] = {"ok",            "invalid-format", "invalid-code",       "invalid-value",
                        "scale-overflow", "shape-mismatch", "ragged-input",       "unsupported-split",
                        "index-out-of-range", "bad-magic",   "bad-version",        "truncated",
                        "corrupt",       "io-failure"};

int fail(int status, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = std::string("error[") + fpx_status_name(status) + "] " + buf;
    g_last_offset = -1;
    return status;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(FPX_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define FPX_CUDA(call)                                       \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
    } while (0)

int bias_of(int e) { return (1 << (e - 1)) - 1; }

// Device gate: the kernels are sm_100a-only (tcgen05/TMEM/TMA).
int check_device(bool need_sm100) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(FPX_ERR_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
    if (!need_sm100) return FPX_OK;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(FPX_ERR_DEVICE, "device %d is sm_%d%d; libfpx_b200 kernels are built for sm_100a", dev,
                    major, minor);
    return FPX_OK;
}

// Per-call status words and skip flags come from a stream-ordered pool the
// library owns, one per device, that keeps its memory between calls (release
// threshold = max).  The default pool returns everything at each
// synchronisation, which made every cudaMallocAsync of a few bytes remap
// memory: ~0.4 ms per quantize / prepack call on B200.
static cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if (cudaError_t e = cudaMemPoolCreate(&pools[dev], &props)) return e;
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(ptr, bytes, pool, s);
}

int resolve_split(int e, int m, const int* widths, int nseg, int* w_out) {
    if (widths == nullptr || nseg == 0) {
        nseg = fpx_split_for_format(e, m, w_out);
        return nseg;
    }
    if (nseg < 1 || nseg > 3) return -1;
    int tot = 0;
    for (int i = 0; i < nseg; ++i) {
        if (widths[i] != 1 && widths[i] != 2 && widths[i] != 4) return -1;
        w_out[i] = widths[i];
        tot += widths[i];
    }
    return tot == 1 + e + m ? nseg : -1;
}

int num_sms() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

uint32_t npad_of(uint32_t n) {
    uint32_t p = 16;
    while (p < n) p *= 2;
    return p;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

constexpr size_t kLinearCounterBytes = 64 * 1024;  // split-K arrival counters (4 per 128-row tile)

// Debug-only pipeline trace: device buffer of kTraceWords clock64 /
// globaltimer stamps written by fpx_linear (CTA 0 per-stage events + a
// per-CTA timeline).  FPX_LINEAR_TRACE=1: one buffer, cleared per call.
// FPX_LINEAR_TRACE=2: calls alternate between two buffers that are cleared
// only on allocation, so two consecutive launches can be compared.
constexpr size_t kTraceWords = 32 * 512;
unsigned long long* g_trace = nullptr;
unsigned long long* debug_trace_buffer() {
    static int mode = [] {
        const char* e = std::getenv("FPX_LINEAR_TRACE");
        return e ? std::atoi(e) : 0;
    }();
    static unsigned calls = 0;
    if (mode <= 0 || mode == 3) return nullptr;
    if (!g_trace) {
        if (cudaMalloc(&g_trace, 2 * kTraceWords * sizeof(unsigned long long)) != cudaSuccess) return g_trace = nullptr;
        cudaMemset(g_trace, 0, 2 * kTraceWords * sizeof(unsigned long long));
    }
    if (mode == 1) {
        cudaMemset(g_trace, 0, kTraceWords * sizeof(unsigned long long));
        return g_trace;
    }
    return g_trace + (calls++ & 1u) * kTraceWords;
}

// FPX_LINEAR_TRACE=3: per (CTA, warp) "currently waiting on" words in mapped
// host memory (readable by the host while a launch is stuck).
constexpr size_t kProgWords = 300 * 32;
unsigned long long* g_prog_host = nullptr;
volatile unsigned long long* debug_progress_buffer() {
    static const bool on = [] {
        const char* e = std::getenv("FPX_LINEAR_TRACE");
        return e && std::atoi(e) == 3;
    }();
    if (!on) return nullptr;
    if (!g_prog_host) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&g_prog_host), kProgWords * 8, cudaHostAllocMapped) != cudaSuccess)
            return nullptr;
        std::memset(g_prog_host, 0, kProgWords * 8);
    }
    void* dev = nullptr;
    if (cudaHostGetDevicePointer(&dev, g_prog_host, 0) != cudaSuccess) return nullptr;
    return static_cast<volatile unsigned long long*>(dev);
}

// PDL guard.  The fused linear's default launch mode streams packed weights
// and row scales before griddepcontrol.wait (pdl_mode 2, fpx_linear.cu).
// When one of this library's own kernels has just written packed weights or
// scales on a stream (quantize, quantize_pack, prepack), the next linear on
// that stream is capped at mode 1 -- every global read after the wait, i.e.
// after the writer completed and its stores are visible -- and the mark is
// cleared.  Writers on other streams reach the linear only through an event
// wait, which is never a programmatic edge.
std::mutex g_dirty_mu;
std::vector<cudaStream_t> g_dirty;

void mark_weights_written(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_dirty_mu);
    for (cudaStream_t d : g_dirty)
        if (d == s) return;
    g_dirty.push_back(s);
}

bool take_weights_written(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_dirty_mu);
    for (size_t i = 0; i < g_dirty.size(); ++i)
        if (g_dirty[i] == s) {
            g_dirty[i] = g_dirty.back();
            g_dirty.pop_back();
            return true;
        }
    return false;
}

}  // namespace

extern "C" {

const char* fpx_last_error(void) { return g_last_error.c_str(); }
int64_t fpx_last_error_offset(void) { return g_last_offset; }

const char* fpx_status_name(int s) {
    if (s >= 0 && s <= 13) return kNames[s];
    if (s == FPX_ERR_CUDA) return "cuda";
    if (s == FPX_ERR_DEVICE) return "device";
    return "unknown";
}

int fpx_version(void) { return 100; }

int fpx_format_check(int e, int m) {
    const int t = 1 + e + m;
    if (e < 1 || e > 5 || m < 0 || m > 6 || t < 3 || t > 8)
        return fail(FPX_ERR_INVALID_FORMAT, "unsupported minifloat format e%dm%d", e, m);
    return FPX_OK;
}

int fpx_split_for_format(int e, int m, int* widths) {
    static const int kW[9][3] = {{0}, {0}, {0}, {2, 1}, {4}, {4, 1}, {2, 4}, {4, 2, 1}, {4, 4}};
    static const int kN[9] = {0, 0, 0, 2, 1, 2, 2, 3, 2};
    const int t = 1 + e + m;
    if (t < 3 || t > 8) return 0;
    for (int i = 0; i < kN[t]; ++i) widths[i] = kW[t][i];
    return kN[t];
}

float fpx_max_representable(int e, int m) {
    const double frac = 2.0 - std::ldexp(1.0, -m);
    return static_cast<float>(std::ldexp(frac, ((1 << e) - 1) - bias_of(e)));
}

uint16_t fpx_effective_scale(uint16_t s, int e, int m) {
    (void)m;
    // fp16 -> fp32 exact, * 2^(15-bias) exact, fp32 -> fp16 RNE
    uint32_t sign = (s >> 15) & 1u, ex = (s >> 10) & 31u, man = s & 1023u;
    float v = ex == 0 ? std::ldexp(float(man), -24) : (ex == 31 ? INFINITY : std::ldexp(float(1024 + man), int(ex) - 25));
    if (ex == 31 && man) v = NAN;
    if (sign) v = -v;
    const float r = v * std::ldexp(1.0f, 15 - bias_of(e));
    // float -> half RNE via the hardware-independent path
    uint32_t x;
    std::memcpy(&x, &r, 4);
    const uint16_t hs = static_cast<uint16_t>((x >> 16) & 0x8000u);
    const uint32_t a = x & 0x7fffffffu;
    if (a >= 0x7f800000u) return a > 0x7f800000u ? uint16_t(hs | 0x7e00u | ((a & 0x7fffffu) >> 13)) : uint16_t(hs | 0x7c00u);
    const int e16 = int(a >> 23) - 112;
    if (e16 >= 31) return hs | 0x7c00u;
    const uint32_t sig = (a & 0x7fffffu) | 0x800000u;
    int drop;
    uint32_t base;
    if (e16 >= 1) {
        drop = 13;
        base = (uint32_t(e16) << 10) | ((sig >> 13) & 0x3ffu);
    } else {
        if (e16 < -10) return hs;
        drop = 14 - e16;
        base = sig >> drop;
    }
    const uint32_t rem = sig & ((1u << drop) - 1u), halfway = 1u << (drop - 1);
    if (rem > halfway || (rem == halfway && (base & 1u))) ++base;
    return static_cast<uint16_t>(hs | base);
}

uint32_t fpx_pad64(uint32_t n) { return (n + 63u) / 64u * 64u; }

// codec.cpp:49-68: exact value of a code, (-1)^S 1.M 2^(E-bias) or
// 0.M 2^(1-bias), computed in double and narrowed to float (exact for every
// format of at most 8 bits).
int fpx_decode_scalar(uint32_t code, int e, int m, float* out) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (code >= (1u << (1 + e + m)))
        return fail(FPX_ERR_INVALID_CODE, "code %u out of range for e%dm%d", code, e, m);
    const uint32_t sign = code >> (e + m), ef = (code >> m) & ((1u << e) - 1u), mf = code & ((1u << m) - 1u);
    const double v = ef == 0 ? std::ldexp(double(mf), 1 - bias_of(e) - m)
                             : std::ldexp(double((1u << m) + mf), int(ef) - bias_of(e) - m);
    const float f = static_cast<float>(v);
    if (out) *out = sign ? -f : f;
    return FPX_OK;
}

// codec.cpp:70-103: nearest code, ties to even, saturating beyond
// max_representable; NaN is InvalidValue.  The same arithmetic as the
// quantize kernel's encode (fpx_codec.cu encode_dev).
int fpx_encode_scalar(double v, int e, int m, uint32_t* out) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (std::isnan(v)) return fail(FPX_ERR_INVALID_VALUE, "cannot encode NaN");
    const uint32_t smask = 1u << (e + m);
    const uint32_t sign = std::signbit(v) ? smask : 0u;
    const double a = std::fabs(v);
    uint32_t code;
    if (a > static_cast<double>(fpx_max_representable(e, m))) {
        code = sign | (smask - 1u);
    } else {
        const int emin = 1 - bias_of(e);
        int ex = a >= std::ldexp(1.0, emin) ? std::ilogb(a) : emin;
        uint32_t k = static_cast<uint32_t>(std::nearbyint(std::ldexp(a, m - ex)));
        const uint32_t unit = 1u << m;
        if (k == 2u * unit) k = unit, ++ex;
        code = k < unit ? (sign | k) : (sign | (static_cast<uint32_t>(ex + bias_of(e)) << m) | (k - unit));
    }
    if (out) *out = code;
    return FPX_OK;
}

size_t fpx_stream_bytes(uint32_t rows_p, uint32_t cols_p, int width) {
    return static_cast<size_t>(rows_p / 64u) * (cols_p / 64u) * 512u * static_cast<size_t>(width);
}

// ---------------------------------------------------------------- K0
int fpx_quantize(const void* w, int dtype, uint32_t rows, uint32_t cols, int e, int m, uint8_t* codes,
                 uint16_t* scales, uint64_t* status_dev, fpx_stream_t stream) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (dtype != FPX_FP32 && dtype != FPX_FP16)
        return fail(FPX_ERR_INVALID_VALUE, "quantize expects a row-major fp32 matrix");
    if (rows == 0 || cols == 0) return fail(FPX_ERR_SHAPE_MISMATCH, "empty matrix");
    if (!w || !codes || !scales) return fail(FPX_ERR_INVALID_VALUE, "null buffer");
    if (int st = check_device(false)) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(status_dev);
    bool own = false;
    if (!status) {
        FPX_CUDA(scratch_alloc(reinterpret_cast<void**>(&status), sizeof(unsigned long long), s));
        own = true;
    }
    FPX_CUDA(cudaMemsetAsync(status, 0xff, sizeof(unsigned long long), s));
    const double maxrep = static_cast<double>(fpx_max_representable(e, m));
    FPX_CUDA(launch_quantize(w, dtype, rows, cols, fpx_pad64(rows), fpx_pad64(cols), e, m, maxrep, codes, scales,
                             status, s));
    mark_weights_written(s);
    if (!own) return FPX_OK;
    unsigned long long host = 0;
    FPX_CUDA(cudaMemcpyAsync(&host, status, sizeof host, cudaMemcpyDeviceToHost, s));
    FPX_CUDA(cudaFreeAsync(status, s));
    FPX_CUDA(cudaStreamSynchronize(s));
    if (host == ~0ull) return FPX_OK;
    const unsigned long long row = host >> 8;
    const int code = static_cast<int>(host & 0xffu);
    if (code == FPX_ERR_INVALID_VALUE) return fail(code, "row %llu contains NaN", row);
    return fail(code, "row %llu scale does not fit in fp16 (or its 2^%d-folded effective scale overflows)", row,
                15 - bias_of(e));
}

// ---------------------------------------------------------------- codes -> W
int fpx_dequantize_codes(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p, int e, int m,
                         uint16_t* w_f16, uint64_t* status_dev, fpx_stream_t stream) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (rows_p == 0 || cols_p == 0 || rows_p % 64 || cols_p % 64)
        return fail(FPX_ERR_SHAPE_MISMATCH, "quantized dims must be multiples of 64");
    if (!codes || !scales || !w_f16) return fail(FPX_ERR_INVALID_VALUE, "null buffer");
    if ((reinterpret_cast<uintptr_t>(codes) | reinterpret_cast<uintptr_t>(w_f16)) % 16u)
        return fail(FPX_ERR_INVALID_VALUE, "codes and w_f16 must be 16-byte aligned");
    if (int st = check_device(false)) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(status_dev);
    const bool own = status == nullptr;
    if (own) FPX_CUDA(scratch_alloc(reinterpret_cast<void**>(&status), sizeof(unsigned long long), s));
    FPX_CUDA(cudaMemsetAsync(status, 0xff, sizeof(unsigned long long), s));
    FPX_CUDA(launch_dequant_codes(codes, scales, rows_p, cols_p, e, m, status, w_f16, s));
    if (!own) return FPX_OK;
    unsigned long long host = 0;
    FPX_CUDA(cudaMemcpyAsync(&host, status, sizeof host, cudaMemcpyDeviceToHost, s));
    FPX_CUDA(cudaFreeAsync(status, s));
    FPX_CUDA(cudaStreamSynchronize(s));
    if (host == ~0ull) return FPX_OK;
    return fail(FPX_ERR_INVALID_CODE, "row %llu holds a code out of range for e%dm%d", host >> 8, e, m);
}

// ---------------------------------------------------------------- K0+K1 fused
int fpx_quantize_pack(const void* w, int dtype, uint32_t rows, uint32_t cols, int e, int m, const int* widths,
                      int nseg, uint8_t* const* streams, uint16_t* scales, uint64_t* status_dev,
                      fpx_stream_t stream) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (dtype != FPX_FP32 && dtype != FPX_FP16)
        return fail(FPX_ERR_INVALID_VALUE, "quantize expects a row-major fp32 matrix");
    if (rows == 0 || cols == 0) return fail(FPX_ERR_SHAPE_MISMATCH, "empty matrix");
    int wv[3];
    const int ns = resolve_split(e, m, widths, nseg, wv);
    if (ns <= 0) return fail(FPX_ERR_UNSUPPORTED_SPLIT, "segment widths must be 1, 2 or 4 and sum to %d", 1 + e + m);
    if (!w || !scales || !streams) return fail(FPX_ERR_INVALID_VALUE, "null buffer");
    for (int i = 0; i < ns; ++i)
        if (!streams[i]) return fail(FPX_ERR_INVALID_VALUE, "null stream buffer");
    if (int st = check_device(false)) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const uint32_t rows_p = fpx_pad64(rows), cols_p = fpx_pad64(cols);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(status_dev);
    uint8_t* scratch = nullptr;  // [status (own) | row skip flags]
    const size_t skip_off = 16;
    FPX_CUDA(scratch_alloc(reinterpret_cast<void**>(&scratch), skip_off + rows_p, s));
    const bool own = status == nullptr;
    if (own) status = reinterpret_cast<unsigned long long*>(scratch);
    FPX_CUDA(cudaMemsetAsync(status, 0xff, sizeof(unsigned long long), s));
    const double maxrep = static_cast<double>(fpx_max_representable(e, m));
    uint8_t* sp[3] = {streams[0], ns > 1 ? streams[1] : nullptr, ns > 2 ? streams[2] : nullptr};
    FPX_CUDA(launch_quantize_pack(w, dtype, rows, cols, rows_p, cols_p, e, m, maxrep, scales, status,
                                  scratch + skip_off, ns, wv, sp, s));
    mark_weights_written(s);
    if (!own) {
        FPX_CUDA(cudaFreeAsync(scratch, s));
        return FPX_OK;
    }
    unsigned long long host = 0;
    FPX_CUDA(cudaMemcpyAsync(&host, status, sizeof host, cudaMemcpyDeviceToHost, s));
    FPX_CUDA(cudaFreeAsync(scratch, s));
    FPX_CUDA(cudaStreamSynchronize(s));
    if (host == ~0ull) return FPX_OK;
    const unsigned long long row = host >> 8;
    const int code = static_cast<int>(host & 0xffu);
    if (code == FPX_ERR_INVALID_VALUE) return fail(code, "row %llu contains NaN", row);
    return fail(code, "row %llu scale does not fit in fp16 (or its 2^%d-folded effective scale overflows)", row,
                15 - bias_of(e));
}

// ---------------------------------------------------------------- K1
int fpx_prepack(const uint8_t* codes, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p, int e, int m,
                const int* widths, int nseg, uint8_t* const* streams, fpx_stream_t stream) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (rows_p == 0 || cols_p == 0 || rows_p % 64 || cols_p % 64)
        return fail(FPX_ERR_SHAPE_MISMATCH,
                    "matrix dims must be padded to multiples of 64 at quantize time before packing");
    int w[3];
    const int ns = resolve_split(e, m, widths, nseg, w);
    if (ns <= 0) return fail(FPX_ERR_UNSUPPORTED_SPLIT, "split widths do not cover e%dm%d", e, m);
    if (int st = check_device(false)) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (scales) {
        unsigned int* bad = nullptr;
        FPX_CUDA(scratch_alloc(reinterpret_cast<void**>(&bad), sizeof(unsigned int), s));
        FPX_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned int), s));
        FPX_CUDA(launch_check_scales(scales, rows_p, 15 - bias_of(e), bad, s));
        unsigned int hb = 0;
        FPX_CUDA(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, s));
        FPX_CUDA(cudaFreeAsync(bad, s));
        FPX_CUDA(cudaStreamSynchronize(s));
        if (hb) return fail(FPX_ERR_SCALE_OVERFLOW, "effective scale overflows fp16");
    }
    FPX_CUDA(launch_prepack(codes, rows_p, cols_p, 1 + e + m, ns, w, streams, s));
    mark_weights_written(s);
    return FPX_OK;
}

int fpx_unpack(const uint8_t* const* streams, uint32_t rows_p, uint32_t cols_p, int e, int m, const int* widths,
               int nseg, uint8_t* codes, fpx_stream_t stream) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (rows_p == 0 || cols_p == 0 || rows_p % 64 || cols_p % 64)
        return fail(FPX_ERR_SHAPE_MISMATCH, "packed dims must be multiples of 64");
    int w[3];
    const int ns = resolve_split(e, m, widths, nseg, w);
    if (ns <= 0) return fail(FPX_ERR_UNSUPPORTED_SPLIT, "split widths do not cover e%dm%d", e, m);
    if (int st = check_device(false)) return st;
    FPX_CUDA(launch_unpack(streams, rows_p, cols_p, 1 + e + m, ns, w, codes, reinterpret_cast<cudaStream_t>(stream)));
    return FPX_OK;
}

// ---------------------------------------------------------------- K3
int fpx_dequantize(const uint8_t* const* streams, int nseg, const int* widths, const uint16_t* scales,
                   uint32_t rows_p, uint32_t cols_p, int e, int m, uint16_t* w_f16, fpx_stream_t stream) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (rows_p == 0 || cols_p == 0 || rows_p % 64 || cols_p % 64)
        return fail(FPX_ERR_SHAPE_MISMATCH, "packed dims must be multiples of 64");
    int w[3];
    const int ns = resolve_split(e, m, widths, nseg, w);
    if (ns <= 0) return fail(FPX_ERR_UNSUPPORTED_SPLIT, "split widths do not cover e%dm%d", e, m);
    if (int st = check_device(false)) return st;
    // FPX_DEQUANT_PATH = cvt (default, the fused kernel's path) | swar | lut
    const char* pe = std::getenv("FPX_DEQUANT_PATH");
    const int path = !pe ? 0 : (pe[0] == 's' ? 1 : (pe[0] == 'l' ? 2 : 0));
    FPX_CUDA(launch_dequant(streams, ns, w, scales, rows_p, cols_p, e, m, w_f16, path,
                            reinterpret_cast<cudaStream_t>(stream)));
    return FPX_OK;
}

// ---------------------------------------------------------------- K2
int fpx_linear_default_split(uint32_t rows_p, uint32_t cols_p, uint32_t n) {
    return linear_default_split(rows_p, cols_p, n < 256 ? n : 256, num_sms());
}

// The kernel reads activations through a 3-D tensor map {64, n, K/64} whose
// k-tile stride is 64 elements, so it needs rows of exactly cols_p (padded K)
// elements, 16-byte aligned.  Anything else (K_act < cols_p, i.e. the
// reference's zero-extension of b beyond b.rows, gemm.cpp:15-18, or an
// unaligned pointer) is first staged into a zero-padded [n][cols_p] buffer.
static bool act_needs_stage(const uint16_t* act, uint32_t k_act, uint32_t cols_p) {
    return k_act != cols_p || (reinterpret_cast<uintptr_t>(act) % 16u) != 0;
}

// Workspace layout: [split-K arrival counters, kLinearCounterBytes, always at
// offset 0 so they stay valid (self-cleaning) across calls of any shape]
// [fp32 split-K partials][staged activations][N <= 32: the activations'
// e4m3 split for the kind::f8f6f4 units (B8, then per-chunk column scales)].
struct WsLayout {
    size_t part_off, stage_off, split_off, split_bytes, total, total_x8;
};

static WsLayout ws_layout(uint32_t rows_p, uint32_t cols_p, uint32_t n, int split_k, bool stage) {
    const uint32_t nb = n < 256 ? n : 256;
    WsLayout l;
    l.part_off = kLinearCounterBytes;
    l.stage_off = l.part_off + align256(linear_workspace_bytes(rows_p, nb, split_k));
    l.split_off = l.stage_off + (stage ? align256(static_cast<size_t>(cols_p) * n * sizeof(uint16_t)) : 0);
    l.split_bytes = linear_x8_enabled() ? linear_split_bytes(cols_p, nb, split_k) : 0;
    l.total = l.split_off;  // required; the split area is optional (without it N <= 32 runs kind::f16 only)
    l.total_x8 = l.split_off + l.split_bytes;
    return l;
}

size_t fpx_linear_workspace_size(uint32_t rows_p, uint32_t cols_p, uint32_t k_act, uint32_t n, int split_k) {
    if (split_k <= 0) split_k = fpx_linear_default_split(rows_p, cols_p, n);
    // A 16-byte-misaligned activation pointer also needs the staging area;
    // callers passing such pointers should size with k_act != cols_p.
    return ws_layout(rows_p, cols_p, n, split_k, k_act != cols_p).total_x8;
}

static int linear_impl(const uint8_t* const* streams, int nseg, const uint16_t* scales, uint32_t rows_p,
                       uint32_t cols_p, int e, int m, const uint16_t* act, uint32_t k_act, uint32_t n, void* c,
                       uint32_t ldc, int split_k, void* workspace, size_t workspace_bytes, fpx_stream_t stream,
                       const fpx_epilogue* epi) {
    if (fpx_format_check(e, m)) return FPX_ERR_INVALID_FORMAT;
    if (epi != nullptr) {
        if (epi->out_dtype != FPX_FP32 && epi->out_dtype != FPX_FP16)
            return fail(FPX_ERR_INVALID_VALUE, "epilogue out_dtype must be FPX_FP32 or FPX_FP16");
        if (epi->activation < FPX_ACT_NONE || epi->activation > FPX_ACT_GELU_TANH)
            return fail(FPX_ERR_INVALID_VALUE, "unknown epilogue activation %d", epi->activation);
    }
    const bool out16 = epi != nullptr && epi->out_dtype == FPX_FP16;
    const size_t esz = out16 ? 2 : 4;
    int fmt = -1;
    int w[3];
    const int ns = resolve_split(e, m, nullptr, 0, w);
    if (e == 3 && m == 2) fmt = 0;
    else if (e == 2 && m == 3) fmt = 1;
    else if (e == 2 && m == 2) fmt = 2;
    if (fmt < 0 || nseg != ns)
        return fail(FPX_ERR_UNSUPPORTED_SPLIT, "fused linear serves e3m2/e2m3 ([2,4]) and e2m2 ([4,1]); got e%dm%d", e,
                    m);
    if (rows_p == 0 || cols_p == 0 || rows_p % 64 || cols_p % 64)
        return fail(FPX_ERR_SHAPE_MISMATCH, "packed dims must be multiples of 64");
    if (k_act == 0 || k_act > cols_p)
        return fail(FPX_ERR_SHAPE_MISMATCH, "weight cols %u do not match activation rows %u", cols_p, k_act);
    if (ldc < rows_p) return fail(FPX_ERR_SHAPE_MISMATCH, "ldc %u < rows %u", ldc, rows_p);
    if (n == 0) return FPX_OK;
    if (int st = check_device(true)) return st;
    const int kt = static_cast<int>(cols_p / 64);
    if (split_k <= 0) split_k = fpx_linear_default_split(rows_p, cols_p, n);
    if (split_k > kt) split_k = kt;
    if (split_k > 1 && (rows_p + 127) / 128 * 4 * sizeof(uint32_t) > kLinearCounterBytes)
        return fail(FPX_ERR_SHAPE_MISMATCH, "rows %u exceed the split-K counter table", rows_p);
    const bool stage = act_needs_stage(act, k_act, cols_p);
    const WsLayout lay = ws_layout(rows_p, cols_p, n, split_k, stage);
    if (workspace == nullptr || workspace_bytes < lay.total)
        return fail(FPX_ERR_INVALID_VALUE, "workspace of %zu bytes required (got %zu)", lay.total, workspace_bytes);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const uint16_t* a = act;
    if (stage) {
        uint16_t* staged = reinterpret_cast<uint16_t*>(ws + lay.stage_off);
        FPX_CUDA(launch_stage_act(act, k_act, n, cols_p, staged, s));
        a = staged;
    }
    uint32_t* counters = reinterpret_cast<uint32_t*>(ws);
    float* part = reinterpret_cast<float*>(ws + lay.part_off);
    const char* g = std::getenv("FPX_LINEAR_GRID");
    const int grid = g ? std::atoi(g) : num_sms();
    const uint32_t pdl_cap = take_weights_written(s) ? 1u : 2u;
    const uint32_t chunk = 256u;  // widest accumulator of the fused kernels
    for (uint32_t n0 = 0; n0 < n; n0 += chunk) {
        LinearLaunch L{};
        L.fmt = fmt;
        L.s_hi = streams[0];
        L.s_lo = streams[1];
        L.scales = scales;
        L.rows_p = rows_p;
        L.cols_p = cols_p;
        L.act = a + static_cast<size_t>(n0) * cols_p;
        L.lda = cols_p;
        L.n = (n - n0) < chunk ? (n - n0) : chunk;
        L.c = reinterpret_cast<float*>(static_cast<uint8_t*>(c) + static_cast<size_t>(n0) * ldc * esz);
        L.ldc = ldc;
        if (epi != nullptr) {
            L.out_f16 = out16 ? 1u : 0u;
            L.bias = epi->bias;
            L.act_fn = static_cast<uint32_t>(epi->activation);
            L.resid = epi->residual == nullptr
                          ? nullptr
                          : static_cast<const uint8_t*>(epi->residual) + static_cast<size_t>(n0) * ldc * esz;
        }
        L.split = split_k;
        L.ws = part;
        L.counters = counters;
        L.grid = grid;
        L.trace = debug_trace_buffer();
        L.prog = debug_progress_buffer();
        L.pdl_cap = pdl_cap;
        if (lay.split_bytes != 0 && L.n <= 32 && workspace_bytes >= lay.total_x8) {
            const uint32_t npad = L.n <= 16 ? 16u : 32u;
            L.b8 = ws + lay.split_off;
            L.colf = reinterpret_cast<float*>(ws + lay.split_off + align256(static_cast<size_t>(3) * npad * cols_p));
        }
        const cudaError_t err = launch_linear(L, s);
        if (err != cudaSuccess) {
            // A launch that did not run to completion may leave split-K
            // arrival counters behind; clear them so the workspace stays
            // valid for the next call (a sticky device fault makes every
            // later call fail anyway).
            (void)cudaGetLastError();
            if (split_k > 1) (void)cudaMemsetAsync(counters, 0, kLinearCounterBytes, s);
            if (err == cudaErrorNotSupported) return fail(FPX_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
            return cuda_fail(err, "fpx_linear_kernel launch");
        }
    }
    return FPX_OK;
}

int fpx_linear_workspace_reset(void* workspace, size_t workspace_bytes, fpx_stream_t stream) {
    if (workspace == nullptr || workspace_bytes < kLinearCounterBytes)
        return fail(FPX_ERR_INVALID_VALUE, "workspace of at least %zu bytes required", kLinearCounterBytes);
    FPX_CUDA(cudaMemsetAsync(workspace, 0, kLinearCounterBytes, reinterpret_cast<cudaStream_t>(stream)));
    return FPX_OK;
}

int fpx_linear(const uint8_t* const* streams, int nseg, const uint16_t* scales, uint32_t rows_p, uint32_t cols_p,
               int e, int m, const uint16_t* act, uint32_t k_act, uint32_t n, float* c, uint32_t ldc, int split_k,
               void* workspace, size_t workspace_bytes, fpx_stream_t stream) {
    return linear_impl(streams, nseg, scales, rows_p, cols_p, e, m, act, k_act, n, c, ldc, split_k, workspace,
                       workspace_bytes, stream, nullptr);
}

int fpx_linear_ex(const uint8_t* const* streams, int nseg, const uint16_t* scales, uint32_t rows_p,
                  uint32_t cols_p, int e, int m, const uint16_t* act, uint32_t k_act, uint32_t n, void* c,
                  uint32_t ldc, int split_k, const fpx_epilogue* epi, void* workspace, size_t workspace_bytes,
                  fpx_stream_t stream) {
    return linear_impl(streams, nseg, scales, rows_p, cols_p, e, m, act, k_act, n, c, ldc, split_k, workspace,
                       workspace_bytes, stream, epi);
}

// ---------------------------------------------------------------- multi-GPU
const volatile uint64_t* fpx_debug_progress(void) { return reinterpret_cast<const volatile uint64_t*>(g_prog_host); }

int fpx_debug_trace(uint64_t* host, size_t words) {
    if (!g_trace) return fail(FPX_ERR_INVALID_VALUE, "no trace recorded (set FPX_LINEAR_TRACE=1)");
    if (words > 2 * kTraceWords) words = 2 * kTraceWords;
    FPX_CUDA(cudaMemcpy(host, g_trace, words * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return FPX_OK;
}

void fpx_shard_rows(uint32_t rows_p, int rank, int world, uint32_t* tr0, uint32_t* tr1) {
    const uint64_t trs = rows_p / 64u;
    if (world <= 0) world = 1;
    *tr0 = static_cast<uint32_t>(trs * rank / world);
    *tr1 = static_cast<uint32_t>(trs * (rank + 1) / world);
}

int fpx_gather_permute(const float* gathered, const uint32_t* row0, const uint32_t* nrows, int world, uint32_t m_slot,
                       uint32_t n, float* c, uint32_t ldc, fpx_stream_t stream) {
    if (world <= 0) return fail(FPX_ERR_INVALID_VALUE, "world must be positive");
    if (int st = check_device(false)) return st;
    FPX_CUDA(launch_gather_permute(gathered, row0, nrows, world, m_slot, n, c, ldc,
                                   reinterpret_cast<cudaStream_t>(stream)));
    return FPX_OK;
}

// ---------------------------------------------------------------- sharded linear
// NCCL is resolved at call time, never linked: the ncclComm_t the caller
// passes must come from the very library whose ncclAllGather runs.  The
// library is (1) FPX_NCCL_LIB when set, else (2) the one libnccl already
// mapped into the process (e.g. torch's), else (3) libnccl.so.2 from the
// loader path.  Two different libnccl files mapped at once is ambiguous --
// a communicator from one is garbage to the other -- and fails loudly.
struct NcclScan {
    std::string paths[4];
    int n = 0;
};

static int nccl_scan_cb(struct dl_phdr_info* info, size_t, void* data) {
    auto* sc = static_cast<NcclScan*>(data);
    const char* name = info->dlpi_name;
    if (name == nullptr || std::strstr(name, "libnccl") == nullptr) return 0;
    for (int i = 0; i < sc->n; ++i)
        if (sc->paths[i] == name) return 0;
    if (sc->n < 4) sc->paths[sc->n++] = name;
    return 0;
}

typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
static nccl_allgather_fn nccl_allgather(std::string* why) {
    static std::mutex mu;
    static nccl_allgather_fn fn = nullptr;
    static std::string err;
    std::lock_guard<std::mutex> lk(mu);
    if (fn != nullptr) return fn;
    void* h = nullptr;
    if (const char* env = std::getenv("FPX_NCCL_LIB")) {
        h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) err = std::string("FPX_NCCL_LIB ") + env + ": " + dlerror();
    } else {
        NcclScan sc;
        dl_iterate_phdr(nccl_scan_cb, &sc);
        if (sc.n > 1) {
            err = "two NCCL libraries are loaded (" + sc.paths[0] + ", " + sc.paths[1] +
                  "); set FPX_NCCL_LIB to the one that created the communicator";
        } else if (sc.n == 1) {
            h = dlopen(sc.paths[0].c_str(), RTLD_NOW | RTLD_NOLOAD);
            if (h == nullptr) err = "cannot re-open " + sc.paths[0];
        } else {
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (h == nullptr) err = "libnccl.so.2 not found (load NCCL first)";
        }
    }
    if (h != nullptr) {
        fn = reinterpret_cast<nccl_allgather_fn>(dlsym(h, "ncclAllGather"));
        if (fn == nullptr) err = "ncclAllGather not exported by the NCCL library";
    }
    if (why) *why = err;
    return fn;
}

static uint32_t shard_slot_rows(uint32_t rows_p, int world) {
    const uint32_t trs = rows_p / 64u;
    return (trs + static_cast<uint32_t>(world) - 1u) / static_cast<uint32_t>(world) * 64u;
}

size_t fpx_linear_sharded_workspace_size(uint32_t rows_p, uint32_t cols_p, uint32_t k_act, uint32_t n, int world,
                                         int split_k) {
    if (world <= 0) world = 1;
    const uint32_t slot = shard_slot_rows(rows_p, world);
    if (split_k == -1) split_k = fpx_linear_default_split(slot, cols_p, n);
    if (split_k <= 0) split_k = fpx_linear_default_split(rows_p, cols_p, n);
    const size_t lin = align256(ws_layout(slot, cols_p, n, split_k, k_act != cols_p).total_x8);
    return lin + align256(size_t(slot) * n * 4) + align256(size_t(world) * slot * n * 4);
}

int fpx_linear_sharded(const uint8_t* const* shard_streams, int nseg, const uint16_t* shard_scales, uint32_t rows_p,
                       uint32_t cols_p, int e, int m, const uint16_t* act, uint32_t k_act, uint32_t n, float* c,
                       uint32_t ldc, int split_k, int rank, int world, void* nccl_comm, void* workspace,
                       size_t workspace_bytes, fpx_stream_t stream) {
    if (world <= 0 || rank < 0 || rank >= world) return fail(FPX_ERR_INVALID_VALUE, "rank %d of world %d", rank, world);
    if (rows_p == 0 || rows_p % 64) return fail(FPX_ERR_SHAPE_MISMATCH, "packed rows must be a multiple of 64");
    if (ldc < rows_p) return fail(FPX_ERR_SHAPE_MISMATCH, "ldc %u < rows %u", ldc, rows_p);
    if (n == 0) return FPX_OK;
    if (world > 1 && nccl_comm == nullptr) return fail(FPX_ERR_INVALID_VALUE, "world > 1 needs an NCCL communicator");
    std::string why;
    nccl_allgather_fn ag = world > 1 ? nccl_allgather(&why) : nullptr;
    if (world > 1 && ag == nullptr) return fail(FPX_ERR_DEVICE, "%s", why.c_str());
    uint32_t tr0 = 0, tr1 = 0;
    fpx_shard_rows(rows_p, rank, world, &tr0, &tr1);
    const uint32_t slot = shard_slot_rows(rows_p, world), m_local = (tr1 - tr0) * 64u;
    // 0: the FULL problem's split -- shard rows bit-identical to a 1-GPU run;
    // -1: the split that suits this shard (every rank's rows are computed
    // identically for a given world size, within the tolerance of a 1-GPU run).
    if (split_k == -1) split_k = fpx_linear_default_split(slot, cols_p, n);
    if (split_k <= 0) split_k = fpx_linear_default_split(rows_p, cols_p, n);
    const size_t need = fpx_linear_sharded_workspace_size(rows_p, cols_p, k_act, n, world, split_k);
    if (workspace == nullptr || workspace_bytes < need)
        return fail(FPX_ERR_INVALID_VALUE, "workspace of %zu bytes required (got %zu)", need, workspace_bytes);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const size_t lin = align256(ws_layout(slot, cols_p, n, split_k, k_act != cols_p).total_x8);
    float* local = reinterpret_cast<float*>(ws + lin);
    float* gathered = reinterpret_cast<float*>(ws + lin + align256(size_t(slot) * n * 4));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (m_local > 0) {
        const int st = fpx_linear(shard_streams, nseg, shard_scales, m_local, cols_p, e, m, act, k_act, n, local, slot,
                                  split_k, ws, lin, stream);
        if (st != FPX_OK) return st;
    }
    if (nccl_comm == nullptr) {  // world == 1 without a communicator: the slice is all of C
        FPX_CUDA(launch_gather_shards(local, rows_p, 1, slot, n, c, ldc, s));
        return FPX_OK;
    }
    if (ag == nullptr && (ag = nccl_allgather(&why)) == nullptr) return fail(FPX_ERR_DEVICE, "%s", why.c_str());
    const int nst = ag(local, gathered, size_t(slot) * n, /*ncclFloat32*/ 7, nccl_comm, s);
    if (nst != 0) return fail(FPX_ERR_CUDA, "ncclAllGather failed (ncclResult %d)", nst);
    FPX_CUDA(launch_gather_shards(gathered, rows_p, world, slot, n, c, ldc, s));
    return FPX_OK;
}

}  // extern "C"

namespace fpxi {
int set_error(int status, const std::string& msg, int64_t offset) {
    g_last_error = std::string("error[") + fpx_status_name(status) + "] " + msg;
    if (offset >= 0) g_last_error += " (at byte " + std::to_string(offset) + ")";
    g_last_offset = offset;
    return status;
}
}  // namespace fpxi
