// fpx_io.cpp -- PackFile container I/O of the C-ABI (host only).
//
// Format (declared by the reference, io.hpp:13-22 and SPEC.md model-io
// "PackFile", never implemented there), all fields little-endian:
//   magic "FPXPACK1" | u16 version=1 | u8 exp_bits | u8 man_bits |
//   u8 segment count | u8 widths[count] (high bits first) | u32 orig_rows |
//   u32 orig_cols | u32 padded_rows | u32 padded_cols | u32 tile_m=64 |
//   u32 tile_k=64 | u8 scale granularity (0 = row) |
//   scales: padded_rows x u16 (fp16 bits) |
//   per segment: u64 byte length, then the stream bytes (prepack layout).
// Validation is strict (SPEC: "strict validation, bit-exact round trip"):
// every violation names its ErrorCode and the byte offset it was found at.
// fpx_packfile_load streams the payload from disk straight into caller-owned
// device buffers through two pinned staging buffers, so a pre-packed weight
// never exists as a pageable host copy.
#include <cuda_runtime_api.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fpx_c.h"
#include "fpx_internal.h"

namespace {

constexpr char kMagic[8] = {'F', 'P', 'X', 'P', 'A', 'C', 'K', '1'};
constexpr uint16_t kVersion = 1;

size_t header_bytes(int nseg) { return 8 + 2 + 1 + 1 + 1 + static_cast<size_t>(nseg) + 6 * 4 + 1; }

template <typename T>
void put_le(uint8_t*& p, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) *p++ = static_cast<uint8_t>(static_cast<uint64_t>(v) >> (8 * i));
}

// Byte source of a pack file: an in-memory buffer or a FILE*.  The parser
// reads only the header, the scales window bounds and the stream lengths, so
// a multi-GB file is validated without reading its payload.
struct Source {
    const uint8_t* mem = nullptr;
    FILE* f = nullptr;
    size_t size = 0;
    bool read(size_t off, size_t n, void* dst) const {
        if (off > size || size - off < n) return false;
        if (mem) {
            std::memcpy(dst, mem + off, n);
            return true;
        }
        return std::fseek(f, static_cast<long>(off), SEEK_SET) == 0 && std::fread(dst, 1, n, f) == n;
    }
};

// Bounds-checked little-endian field reader: a short read is Truncated at
// the offset where the field starts.
struct Reader {
    const Source& src;
    size_t off = 0;
    int status = FPX_OK;
    template <typename T>
    bool get(T& v, const char* what) {
        if (status != FPX_OK) return false;
        uint8_t b[sizeof(T)];
        if (!src.read(off, sizeof(T), b)) {
            status = fpxi::set_error(FPX_ERR_TRUNCATED, std::string("pack file ends inside ") + what,
                                     static_cast<int64_t>(off));
            return false;
        }
        uint64_t x = 0;
        for (size_t i = 0; i < sizeof(T); ++i) x |= static_cast<uint64_t>(b[i]) << (8 * i);
        v = static_cast<T>(x);
        off += sizeof(T);
        return true;
    }
};

int split_ok(int e, int m, const int* w, int nseg) {
    if (fpx_format_check(e, m) != FPX_OK) return FPX_ERR_INVALID_FORMAT;
    if (nseg < 1 || nseg > 3) return FPX_ERR_UNSUPPORTED_SPLIT;
    int tot = 0;
    for (int i = 0; i < nseg; ++i) {
        if (w[i] != 1 && w[i] != 2 && w[i] != 4) return FPX_ERR_UNSUPPORTED_SPLIT;
        tot += w[i];
    }
    return tot == 1 + e + m ? FPX_OK : FPX_ERR_UNSUPPORTED_SPLIT;
}

}  // namespace

extern "C" {

size_t fpx_packfile_bytes(uint32_t rows_p, uint32_t cols_p, const int* widths, int nseg) {
    size_t t = header_bytes(nseg) + static_cast<size_t>(rows_p) * 2;
    for (int i = 0; i < nseg; ++i) t += 8 + fpx_stream_bytes(rows_p, cols_p, widths[i]);
    return t;
}

int fpx_packfile_encode(int exp_bits, int man_bits, const int* widths, int nseg, uint32_t orig_rows,
                        uint32_t orig_cols, uint32_t rows_p, uint32_t cols_p, const uint16_t* scales,
                        const uint8_t* const* streams, uint8_t* out, size_t out_bytes) {
    if (const int st = split_ok(exp_bits, man_bits, widths, nseg))
        return fpxi::set_error(st, "format / split not packable");
    if (rows_p % 64 || cols_p % 64 || rows_p == 0 || cols_p == 0 || orig_rows > rows_p || orig_cols > cols_p ||
        fpx_pad64(orig_rows) != rows_p || fpx_pad64(orig_cols) != cols_p)
        return fpxi::set_error(FPX_ERR_SHAPE_MISMATCH, "padded dims must be pad64 of the original dims");
    const size_t need = fpx_packfile_bytes(rows_p, cols_p, widths, nseg);
    if (out == nullptr || out_bytes < need)
        return fpxi::set_error(FPX_ERR_INVALID_VALUE, "output buffer smaller than fpx_packfile_bytes()");
    if (scales == nullptr || streams == nullptr) return fpxi::set_error(FPX_ERR_INVALID_VALUE, "null buffer");
    uint8_t* p = out;
    std::memcpy(p, kMagic, 8);
    p += 8;
    put_le<uint16_t>(p, kVersion);
    put_le<uint8_t>(p, static_cast<uint8_t>(exp_bits));
    put_le<uint8_t>(p, static_cast<uint8_t>(man_bits));
    put_le<uint8_t>(p, static_cast<uint8_t>(nseg));
    for (int i = 0; i < nseg; ++i) put_le<uint8_t>(p, static_cast<uint8_t>(widths[i]));
    put_le<uint32_t>(p, orig_rows);
    put_le<uint32_t>(p, orig_cols);
    put_le<uint32_t>(p, rows_p);
    put_le<uint32_t>(p, cols_p);
    put_le<uint32_t>(p, 64);
    put_le<uint32_t>(p, 64);
    put_le<uint8_t>(p, 0);
    for (uint32_t r = 0; r < rows_p; ++r) put_le<uint16_t>(p, scales[r]);
    for (int i = 0; i < nseg; ++i) {
        const size_t len = fpx_stream_bytes(rows_p, cols_p, widths[i]);
        put_le<uint64_t>(p, len);
        std::memcpy(p, streams[i], len);
        p += len;
    }
    return FPX_OK;
}

static int parse_source(const Source& src, fpx_pack_header* h) {
    std::memset(h, 0, sizeof *h);
    const size_t nbytes = src.size;
    Reader r{src};
    char magic[8];
    if (!src.read(0, 8, magic)) return fpxi::set_error(FPX_ERR_TRUNCATED, "pack file ends inside the magic", 0);
    if (std::memcmp(magic, kMagic, 8) != 0) return fpxi::set_error(FPX_ERR_BAD_MAGIC, "not an FPXPACK1 file", 0);
    r.off = 8;
    uint16_t ver = 0;
    uint8_t e = 0, m = 0, ns = 0;
    if (!r.get(ver, "the version")) return r.status;
    if (ver != kVersion)
        return fpxi::set_error(FPX_ERR_BAD_VERSION, "pack file version " + std::to_string(ver) + ", expected 1", 8);
    if (!r.get(e, "exp_bits") || !r.get(m, "man_bits")) return r.status;
    if (fpx_format_check(e, m) != FPX_OK)
        return fpxi::set_error(FPX_ERR_INVALID_FORMAT, "format e" + std::to_string(e) + "m" + std::to_string(m), 10);
    const size_t ns_off = r.off;
    if (!r.get(ns, "the segment count")) return r.status;
    if (ns < 1 || ns > 3)
        return fpxi::set_error(FPX_ERR_UNSUPPORTED_SPLIT, std::to_string(ns) + " segments", static_cast<int64_t>(ns_off));
    for (int i = 0; i < ns; ++i) {
        uint8_t w = 0;
        if (!r.get(w, "the segment widths")) return r.status;
        h->widths[i] = w;
    }
    if (split_ok(e, m, h->widths, ns) != FPX_OK)
        return fpxi::set_error(FPX_ERR_UNSUPPORTED_SPLIT, "segment widths do not split the format",
                               static_cast<int64_t>(ns_off + 1));
    const size_t dim_off = r.off;
    uint32_t dims[6];
    for (int i = 0; i < 6; ++i)
        if (!r.get(dims[i], "the dimensions")) return r.status;
    uint8_t gran = 0;
    if (!r.get(gran, "the scale granularity")) return r.status;
    if (dims[4] != 64 || dims[5] != 64)
        return fpxi::set_error(FPX_ERR_CORRUPT, "tile shape must be 64x64", static_cast<int64_t>(dim_off + 16));
    if (gran != 0)
        return fpxi::set_error(FPX_ERR_CORRUPT, "only row-wise scales (granularity 0)", static_cast<int64_t>(r.off - 1));
    if (dims[2] == 0 || dims[3] == 0 || dims[2] % 64 || dims[3] % 64 || fpx_pad64(dims[0]) != dims[2] ||
        fpx_pad64(dims[1]) != dims[3])
        return fpxi::set_error(FPX_ERR_CORRUPT, "inconsistent dimensions", static_cast<int64_t>(dim_off));
    h->exp_bits = e;
    h->man_bits = m;
    h->nseg = ns;
    h->orig_rows = dims[0];
    h->orig_cols = dims[1];
    h->rows_p = dims[2];
    h->cols_p = dims[3];
    h->scales_offset = r.off;
    const size_t scale_bytes = static_cast<size_t>(h->rows_p) * 2;
    if (nbytes - r.off < scale_bytes)
        return fpxi::set_error(FPX_ERR_TRUNCATED, "pack file ends inside the scales", static_cast<int64_t>(nbytes));
    r.off += scale_bytes;
    for (int i = 0; i < ns; ++i) {
        const size_t len_off = r.off;
        uint64_t len = 0;
        if (!r.get(len, "a stream length")) return r.status;
        const size_t want = fpx_stream_bytes(h->rows_p, h->cols_p, h->widths[i]);
        if (len != want)
            return fpxi::set_error(FPX_ERR_CORRUPT,
                                   "stream " + std::to_string(i) + " length " + std::to_string(len) + ", size law " +
                                       std::to_string(want),
                                   static_cast<int64_t>(len_off));
        if (nbytes - r.off < len)
            return fpxi::set_error(FPX_ERR_TRUNCATED, "pack file ends inside stream " + std::to_string(i),
                                   static_cast<int64_t>(nbytes));
        h->stream_offset[i] = r.off;
        h->stream_bytes[i] = len;
        r.off += len;
    }
    if (r.off != nbytes)
        return fpxi::set_error(FPX_ERR_CORRUPT, "trailing bytes after the last stream", static_cast<int64_t>(r.off));
    h->file_bytes = nbytes;
    return FPX_OK;
}

int fpx_packfile_parse(const uint8_t* bytes, size_t nbytes, fpx_pack_header* h) {
    if (h == nullptr) return fpxi::set_error(FPX_ERR_INVALID_VALUE, "null header");
    if (bytes == nullptr && nbytes) return fpxi::set_error(FPX_ERR_INVALID_VALUE, "null buffer");
    Source src;
    src.mem = bytes;
    src.size = nbytes;
    return parse_source(src, h);
}

int fpx_packfile_load(const char* path, fpx_pack_header* hdr, uint16_t* scales_dev, uint8_t* const* streams_dev,
                      fpx_stream_t stream) {
    if (path == nullptr || hdr == nullptr) return fpxi::set_error(FPX_ERR_INVALID_VALUE, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (f == nullptr) return fpxi::set_error(FPX_ERR_IO_FAILURE, std::string("cannot open ") + path);
    std::fseek(f, 0, SEEK_END);
    const long fsize = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    Source src;
    src.f = f;
    src.size = static_cast<size_t>(fsize < 0 ? 0 : fsize);
    int st = parse_source(src, hdr);
    if (st != FPX_OK || scales_dev == nullptr) {
        std::fclose(f);
        return st;
    }
    if (streams_dev == nullptr) {
        std::fclose(f);
        return fpxi::set_error(FPX_ERR_INVALID_VALUE, "null stream buffers");
    }
    // payload -> device through two pinned staging buffers
    constexpr size_t kChunk = size_t(16) << 20;
    void* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cleanup = [&](int status) {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
            if (pin[i]) cudaFreeHost(pin[i]);
        }
        std::fclose(f);
        return status;
    };
    for (int i = 0; i < 2; ++i) {
        if (cudaHostAlloc(&pin[i], kChunk, cudaHostAllocDefault) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
            return cleanup(fpxi::set_error(FPX_ERR_CUDA, "pinned staging buffer"));
    }
    int slot = 0;
    auto copy_range = [&](uint64_t off, uint64_t len, uint8_t* dst) -> int {
        std::fseek(f, static_cast<long>(off), SEEK_SET);
        while (len) {
            const size_t n = len < kChunk ? static_cast<size_t>(len) : kChunk;
            if (cudaEventSynchronize(ev[slot]) != cudaSuccess) return fpxi::set_error(FPX_ERR_CUDA, "staging sync");
            if (std::fread(pin[slot], 1, n, f) != n)
                return fpxi::set_error(FPX_ERR_IO_FAILURE, "short read", static_cast<int64_t>(off));
            if (cudaMemcpyAsync(dst, pin[slot], n, cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream)) !=
                    cudaSuccess ||
                cudaEventRecord(ev[slot], reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess)
                return fpxi::set_error(FPX_ERR_CUDA, "host-to-device copy");
            dst += n;
            off += n;
            len -= n;
            slot ^= 1;
        }
        return FPX_OK;
    };
    if ((st = copy_range(hdr->scales_offset, static_cast<uint64_t>(hdr->rows_p) * 2,
                         reinterpret_cast<uint8_t*>(scales_dev))) != FPX_OK)
        return cleanup(st);
    for (int i = 0; i < hdr->nseg; ++i)
        if ((st = copy_range(hdr->stream_offset[i], hdr->stream_bytes[i], streams_dev[i])) != FPX_OK)
            return cleanup(st);
    return cleanup(FPX_OK);
}

}  // extern "C"
