// Native CTC1 / CTA1 ingest into a device store (tm_store_load_ctc1/cta1).
//
// Byte layout of the reference containers (src/io.cpp:121-194,198-279):
// little-endian header {magic[4], version u32 = 1, q u32, m u32, n1 n2 n3 u32,
// k0 f64, eps f64, kernel id u8} = 45 bytes, then per tensor {r1 r2 r3 u32,
// core f1-fastest, U1 U2 U3 column-major, complex f64 pairs}; CTA1 appends V
// (m2 x r_c, column-major) and m2 is recovered from the remaining length.
// Errors carry the byte offset where parsing stopped, as tuckmat::ParseError
// does (include/tuckmat/errors.hpp:39-45).  The 12-byte rank triplets leave
// payloads unaligned, so records are copied, not cast.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tuckmat_b200.h"
#include "tm_io_internal.hpp"

extern "C" void tmb_set_last_error(const char* msg);  // tm_capi.cu

namespace tmb_io {
namespace {

struct Reader {
    std::string path;
    std::vector<char> buf;
    uint64_t pos = 0;

    Reader() = default;
    explicit Reader(const std::string& p) : path(p) {
        std::ifstream in(p, std::ios::binary | std::ios::ate);
        if (!in) fail_at("cannot open '" + p + "'", 0);
        const std::streamsize size = in.tellg();
        in.seekg(0);
        buf.resize(static_cast<size_t>(size));
        in.read(buf.data(), size);
        if (!in) fail_at("short read from '" + p + "'", 0);
    }
    [[noreturn]] static void fail_at(const std::string& m, uint64_t off) {
        throw ParseFail(m + " (byte offset " + std::to_string(off) + ")", off);
    }
    [[noreturn]] void fail(const std::string& m) const { fail_at("'" + path + "': " + m, pos); }
    void need(size_t n, const char* what) const {
        if (buf.size() - pos < n) fail(std::string("truncated while reading ") + what);
    }
    uint64_t remaining() const { return buf.size() - pos; }
    void magic(const char* tag) {
        need(4, "magic");
        if (std::memcmp(buf.data() + pos, tag, 4) != 0) fail(std::string("bad magic, expected ") + std::string(tag, 4));
        pos += 4;
    }
    uint32_t u32() {
        need(4, "u32");
        uint32_t v = 0;
        for (int s = 0; s < 4; ++s) v |= uint32_t(static_cast<unsigned char>(buf[pos++])) << (8 * s);
        return v;
    }
    double f64() {
        need(8, "f64");
        uint64_t b = 0;
        for (int s = 0; s < 8; ++s) b |= uint64_t(static_cast<unsigned char>(buf[pos++])) << (8 * s);
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    }
    uint8_t u8() {
        need(1, "u8");
        return static_cast<uint8_t>(buf[pos++]);
    }
    // n complex128 scalars appended to out (little-endian host assumed: x86-64).
    void c128s(uint64_t n, std::vector<double>& out) {
        need(size_t(16 * n), "f64");
        const size_t o = out.size();
        out.resize(o + 2 * n);
        std::memcpy(out.data() + o, buf.data() + pos, size_t(16 * n));
        pos += 16 * n;
    }
};

struct Header {
    uint32_t q, m, dims[3];
    double k0, eps;
    uint8_t op;
};

Header read_header(Reader& r, const char* tag) {
    r.magic(tag);
    const uint32_t version = r.u32();
    if (version != 1) r.fail("unsupported version " + std::to_string(version));
    Header h{};
    h.q = r.u32();
    h.m = r.u32();
    for (int g = 0; g < 3; ++g) h.dims[g] = r.u32();
    h.k0 = r.f64();
    h.eps = r.f64();
    h.op = r.u8();
    if (h.q < 1 || h.m < 1 || h.dims[0] < 1 || h.dims[1] < 1 || h.dims[2] < 1) r.fail("non-positive header dimensions");
    if (h.op > 1) r.fail("unknown kernel id " + std::to_string(h.op));
    return h;
}

void read_tensors(Reader& r, const Header& h, uint64_t count, std::vector<int32_t>& ranks, std::vector<double>& pay) {
    ranks.reserve(size_t(3 * count));
    for (uint64_t i = 0; i < count; ++i) {
        uint32_t rk[3];
        for (int g = 0; g < 3; ++g) {
            rk[g] = r.u32();
            if (rk[g] == 0 || rk[g] > h.dims[g])
                r.fail("tucker rank " + std::to_string(rk[g]) + " out of range for mode " + std::to_string(g + 1));
            ranks.push_back(int32_t(rk[g]));
        }
        const uint64_t n = uint64_t(rk[0]) * rk[1] * rk[2] + uint64_t(h.dims[0]) * rk[0] + uint64_t(h.dims[1]) * rk[1] +
                           uint64_t(h.dims[2]) * rk[2];
        r.c128s(n, pay);
    }
}

}  // namespace

Parsed parse(const std::string& path, bool aca) {
    Reader r(path);
    const Header h = read_header(r, aca ? "CTA1" : "CTC1");
    Parsed out;
    out.q = h.q;
    out.m = h.m;
    for (int g = 0; g < 3; ++g) out.dims[g] = h.dims[g];
    out.k0 = h.k0;
    out.eps = h.eps;
    out.op = h.op;
    read_tensors(r, h, uint64_t(h.m) * h.q, out.ranks, out.payload);
    if (!aca) {
        if (r.pos != r.buf.size()) r.fail(std::to_string(r.buf.size() - r.pos) + " trailing bytes");
        return out;
    }
    const uint64_t rest = r.remaining();
    const uint64_t col_bytes = 16ull * h.m;
    if (col_bytes == 0 || rest % col_bytes != 0 || rest / col_bytes == 0)
        r.fail("V block of " + std::to_string(rest) + " bytes is not a positive multiple of 16*r_c");
    out.m2 = rest / col_bytes;
    r.c128s(out.m2 * h.m, out.v);
    return out;
}

namespace {

// Streaming reader: the header and the 12-byte rank triplet of every record
// are read up front (seeking over the payloads), the payloads later on
// demand, straight into the builder's pinned staging buffers.
struct StreamScan {
    std::string path;
    std::ifstream in;
    uint64_t size = 0;
    Header h{};
    std::vector<int32_t> ranks;
    std::vector<uint64_t> pay_off;   // file offset of each record's payload
    std::vector<uint64_t> pay_len;   // complex elements
    std::vector<double> v;
    uint64_t m2 = 0;

    [[noreturn]] void fail(const std::string& m, uint64_t off) const {
        throw ParseFail("'" + path + "': " + m + " (byte offset " + std::to_string(off) + ")", off);
    }
    void read_at(uint64_t off, void* dst, uint64_t n, const char* what) {
        if (off + n > size) fail(std::string("truncated while reading ") + what, off > size ? size : off);
        in.seekg(std::streamoff(off));
        in.read(static_cast<char*>(dst), std::streamsize(n));
        if (!in) fail(std::string("read error in ") + what, off);
    }

    StreamScan(const std::string& p, bool aca) : path(p) {
        in.open(p, std::ios::binary | std::ios::ate);
        if (!in) throw ParseFail("cannot open '" + p + "' (byte offset 0)", 0);
        size = uint64_t(in.tellg());
        // the header through the common Reader logic (45 bytes)
        unsigned char hb[45];
        read_at(0, hb, std::min<uint64_t>(45, size), "header");
        Reader r;
        r.path = p;
        r.buf.assign(reinterpret_cast<char*>(hb), reinterpret_cast<char*>(hb) + std::min<uint64_t>(45, size));
        h = read_header(r, aca ? "CTA1" : "CTC1");
        const uint64_t count = uint64_t(h.m) * h.q;
        ranks.reserve(size_t(3 * count));
        pay_off.reserve(size_t(count));
        pay_len.reserve(size_t(count));
        uint64_t pos = 45;
        for (uint64_t i = 0; i < count; ++i) {
            unsigned char rb[12];
            if (pos + 12 > size) fail("truncated while reading u32", pos + 4 * ((size - pos) / 4));
            read_at(pos, rb, 12, "u32");
            uint32_t rk[3];
            for (int g = 0; g < 3; ++g) {
                rk[g] = uint32_t(rb[4 * g]) | uint32_t(rb[4 * g + 1]) << 8 | uint32_t(rb[4 * g + 2]) << 16 |
                        uint32_t(rb[4 * g + 3]) << 24;
                if (rk[g] == 0 || rk[g] > h.dims[g])
                    fail("tucker rank " + std::to_string(rk[g]) + " out of range for mode " + std::to_string(g + 1),
                         pos + 4 * uint64_t(g) + 4);
                ranks.push_back(int32_t(rk[g]));
            }
            pos += 12;
            const uint64_t n = uint64_t(rk[0]) * rk[1] * rk[2] + uint64_t(h.dims[0]) * rk[0] +
                               uint64_t(h.dims[1]) * rk[1] + uint64_t(h.dims[2]) * rk[2];
            if (pos + 16 * n > size) fail("truncated while reading f64", pos);
            pay_off.push_back(pos);
            pay_len.push_back(n);
            pos += 16 * n;
        }
        if (!aca) {
            if (pos != size) fail(std::to_string(size - pos) + " trailing bytes", pos);
            return;
        }
        const uint64_t rest = size - pos;
        const uint64_t col_bytes = 16ull * h.m;
        if (col_bytes == 0 || rest % col_bytes != 0 || rest / col_bytes == 0)
            fail("V block of " + std::to_string(rest) + " bytes is not a positive multiple of 16*r_c", pos);
        m2 = rest / col_bytes;
        v.resize(size_t(2 * m2 * h.m));
        read_at(pos, v.data(), rest, "f64");
    }

    // payloads of records [t0, t1), contiguous, into dst
    void fill(int64_t t0, int64_t t1, double* dst) {
        for (int64_t i = t0; i < t1; ++i) {
            read_at(pay_off[size_t(i)], dst, 16 * pay_len[size_t(i)], "f64");
            dst += 2 * pay_len[size_t(i)];
        }
    }
};

}  // namespace

}  // namespace tmb_io

namespace {

template <typename F>
int guarded_io(F&& f) {
    try {
        return f();
    } catch (const tmb_io::ParseFail& e) {
        tmb_set_last_error(e.what());
        return TM_PARSE_ERROR;
    } catch (const std::bad_alloc&) {
        tmb_set_last_error("host allocation failed");
        return TM_CAPACITY_ERROR;
    }
}

int create_from(const tmb_io::Parsed& p, int device, int dtype, tm_store** out) {
    tm_store_desc d{};
    d.q = int32_t(p.q);
    d.ncols = p.m;
    for (int g = 0; g < 3; ++g) d.dims[g] = p.dims[g];
    d.ranks = p.ranks.data();
    d.payload = p.payload.data();
    if (!p.v.empty()) {
        d.v = p.v.data();
        d.m2 = int64_t(p.m2);
    }
    return tm_store_create(&d, device, dtype, out);
}

int create_streamed(const std::string& path, bool aca, int device, int dtype, tm_store** out) {
    tmb_io::StreamScan sc(path, aca);
    tm_store_desc d{};
    d.q = int32_t(sc.h.q);
    d.ncols = sc.h.m;
    for (int g = 0; g < 3; ++g) d.dims[g] = sc.h.dims[g];
    d.ranks = sc.ranks.data();
    d.payload = nullptr;
    if (aca) {
        d.v = sc.v.data();
        d.m2 = int64_t(sc.m2);
    }
    return tmb_io::create_store_streaming(
        &d, [&](std::int64_t t0, std::int64_t t1, double* dst) { sc.fill(t0, t1, dst); }, device, dtype, out);
}

}  // namespace

extern "C" {

// load_ctc1 (src/io.cpp:212-230) into a device store, streamed (SURVEY
// §8f-3): only the rank triplets are read up front; payloads go from the file
// through two pinned 256 MiB staging buffers to the device in bounded chunks
// (read of chunk c overlapping the copy + pack of chunk c - 1), converted to
// the store's precision on the device — no whole-file host buffer.
TM_API int tm_store_load_ctc1(const char* path, int device, int dtype, tm_store** out) {
    return guarded_io([&]() -> int { return create_streamed(path ? path : "", false, device, dtype, out); });
}

// load_cta1 (src/io.cpp:249-279) into a device store carrying V, streamed.
TM_API int tm_store_load_cta1(const char* path, int device, int dtype, tm_store** out) {
    return guarded_io([&]() -> int { return create_streamed(path ? path : "", true, device, dtype, out); });
}

}  // extern "C"
