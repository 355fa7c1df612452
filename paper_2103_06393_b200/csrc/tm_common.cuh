// Shared device-side types of the B200 Tucker-matvec library.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tmb {

// Complex scalar per precision: interleaved (re, im), 8 or 16 bytes.
template <typename R>
struct Cx;
template <>
struct Cx<float> {
    using T = float2;
};
template <>
struct Cx<double> {
    using T = double2;
};

template <typename C>
__device__ __forceinline__ C cmake(decltype(C{}.x) re, decltype(C{}.x) im) {
    C c;
    c.x = re;
    c.y = im;
    return c;
}

// acc += a * b
template <typename C>
__device__ __forceinline__ void cfma(C& acc, const C& a, const C& b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

// acc += conj(a) * b
template <typename C>
__device__ __forceinline__ void cfma_conj(C& acc, const C& a, const C& b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

template <typename C>
__device__ __forceinline__ C cmul(const C& a, const C& b) {
    C r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}

// Per-tensor descriptor of the device store.  Tensors are indexed
// component-major, t = k * ncols + j, so a CTA that owns component k walks
// the columns of its component through consecutive descriptors.  Offsets
// are element offsets into the store arena.  Layout of one tensor in the
// arena (all 16-byte aligned segments):
//   core  r1*r2*r3, f1-fastest (as the reference, include/tuckmat/tensor.hpp:53-55)
//   U1t   n1 x r1 row-major (rank-fastest: one grid row = r1 contiguous scalars)
//   U2t   n2 x r2 row-major
//   U3t   n3 x r3 row-major
// Row-major factors make the rows of one output tile a single contiguous
// span, so each CTA's factor loads are fully coalesced.
struct TDesc {
    int64_t off_core;
    int64_t off_u1;
    int64_t off_u2;
    int64_t off_u3;
    int32_t r1, r2, r3, pad;
};

}  // namespace tmb
