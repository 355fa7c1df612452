// Host-side CTC1 / CTA1 parser shared by the C ABI loaders and the C++
// drop-in (reference byte layout: src/io.cpp:121-194, 198-279).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tuckmat_b200.h"

namespace tmb_io {

struct ParseFail : std::runtime_error {
    std::uint64_t offset;
    ParseFail(const std::string& m, std::uint64_t off) : std::runtime_error(m), offset(off) {}
};

struct Parsed {
    std::uint32_t q = 0, m = 0, dims[3] = {0, 0, 0};
    double k0 = 0, eps = 0;
    std::uint8_t op = 0;
    std::vector<std::int32_t> ranks;  // [col][comp][mode]
    std::vector<double> payload;      // CTC1 tensor payloads, complex128 pairs
    std::vector<double> v;            // CTA1 only: V, m2 x r_c column-major
    std::uint64_t m2 = 0;
};

// aca = false: "CTC1"; aca = true: "CTA1".  Throws ParseFail.
Parsed parse(const std::string& path, bool aca);

// Streaming ingest: the store builder asks for the payloads
// of tensors [t0, t1) ([col][comp] order, complex128 pairs, contiguous) in
// bounded chunks; `dst` is pinned host memory.  Throws ParseFail.
using PayloadFill = std::function<void(std::int64_t t0, std::int64_t t1, double* dst)>;

// Build a device store from `d` (ranks, optional V; payload unused) with the
// payload streamed through `fill` (tm_capi.cu).  Returns a TM_* status.
int create_store_streaming(const tm_store_desc* d, const PayloadFill& fill, int device, int dtype, tm_store** out);

}  // namespace tmb_io
