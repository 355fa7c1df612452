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

}  // namespace

extern "C" {

// load_ctc1 (src/io.cpp:212-230) into a device store.
TM_API int tm_store_load_ctc1(const char* path, int device, int dtype, tm_store** out) {
    return guarded_io([&]() -> int { return create_from(tmb_io::parse(path ? path : "", false), device, dtype, out); });
}

// load_cta1 (src/io.cpp:249-279) into a device store carrying V.
TM_API int tm_store_load_cta1(const char* path, int device, int dtype, tm_store** out) {
    return guarded_io([&]() -> int { return create_from(tmb_io::parse(path ? path : "", true), device, dtype, out); });
}

}  // extern "C"
