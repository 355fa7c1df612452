// Auxiliary kernels: store packing (K6) and the ACA V products (K5).
#pragma once

#include "tm_common.cuh"

namespace tmb {

// One CTA per tensor.  Source: CTC1 payload order (core f1-fastest, then
// U1, U2, U3 column-major; complex128), tensors in [col][comp] order.
// Destination: arena segments of TDesc (component-major tensor index),
// factors transposed to row-major, scalars rounded to C's precision.
struct PackJob {
    int64_t src_off;   // element offset of the tensor in the staged payload
    int64_t dst_tensor;  // component-major tensor index k*ncols + j
};

template <typename C>
__global__ void pack_kernel(const double2* __restrict__ src, const PackJob* __restrict__ jobs,
                            const TDesc* __restrict__ td, int n1, int n2, int n3, C* __restrict__ arena) {
    using R = decltype(C{}.x);
    const PackJob job = jobs[blockIdx.x];
    const TDesc d = td[job.dst_tensor];
    const double2* s = src + job.src_off;
    const int ncore = d.r1 * d.r2 * d.r3;
    for (int e = threadIdx.x; e < ncore; e += blockDim.x) {
        const double2 v = s[e];
        arena[d.off_core + e] = cmake<C>(R(v.x), R(v.y));
    }
    s += ncore;
    const int ns[3] = {n1, n2, n3};
    const int rs[3] = {d.r1, d.r2, d.r3};
    const int64_t offs[3] = {d.off_u1, d.off_u2, d.off_u3};
    for (int g = 0; g < 3; ++g) {
        const int n = ns[g], r = rs[g];
        // dst[i*r + a] = src[i + n*a]
        for (int e = threadIdx.x; e < n * r; e += blockDim.x) {
            const int i = e / r, a = e - i * r;
            const double2 v = s[i + int64_t(n) * a];
            arena[offs[g] + e] = cmake<C>(R(v.x), R(v.y));
        }
        s += int64_t(n) * r;
    }
}

template <typename C>
__global__ void convert_kernel(const double2* __restrict__ src, int64_t n, C* __restrict__ dst) {
    using R = decltype(C{}.x);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = cmake<C>(R(src[i].x), R(src[i].y));
}

// w[l + rc c] = sum_i conj(V[i + m2 l]) x[i + ldx c]   (aca_forward's V^H x,
// src/matvec.cpp:157).  One warp per (l, c); f64 accumulation.
template <typename C>
__global__ void aca_vhx_kernel(const C* __restrict__ v, int64_t m2, int64_t rc, const C* __restrict__ x, int64_t ldx,
                               int64_t p, C* __restrict__ w) {
    using R = decltype(C{}.x);
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= rc * p) return;
    const int64_t l = wid % rc, c = wid / rc;
    const C* vl = v + m2 * l;
    const C* xc = x + ldx * c;
    double sx = 0, sy = 0;
    for (int64_t i = lane; i < m2; i += 32) {
        const C a = vl[i], b = xc[i];
        sx += double(a.x) * double(b.x) + double(a.y) * double(b.y);
        sy += double(a.x) * double(b.y) - double(a.y) * double(b.x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    if (lane == 0) w[l + rc * c] = cmake<C>(R(sx), R(sy));
}

// z[i + ldz c] = sum_l V[i + m2 l] t[l + rc c]   (aca_adjoint's V t,
// src/matvec.cpp:174).  One thread per (i, c); f64 accumulation.
template <typename C>
__global__ void aca_vt_kernel(const C* __restrict__ v, int64_t m2, int64_t rc, const C* __restrict__ t, int64_t p,
                              C* __restrict__ z, int64_t ldz) {
    using R = decltype(C{}.x);
    const int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= m2 * p) return;
    const int64_t i = id % m2, c = id / m2;
    double sx = 0, sy = 0;
    for (int64_t l = 0; l < rc; ++l) {
        const C a = v[i + m2 * l], b = t[l + rc * c];
        sx += double(a.x) * double(b.x) - double(a.y) * double(b.y);
        sy += double(a.x) * double(b.y) + double(a.y) * double(b.x);
    }
    z[i + ldz * c] = cmake<C>(R(sx), R(sy));
}

// y(:, c) = 0 for a (rows x p) block with leading dimension ldy.
template <typename C>
__global__ void zero_kernel(C* __restrict__ y, int64_t rows, int64_t p, int64_t ldy) {
    using R = decltype(C{}.x);
    const int64_t n = rows * p;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        y[(i % rows) + ldy * (i / rows)] = cmake<C>(R(0), R(0));
}

// Batched element extraction: out[r + ldout j] = T_jk[v] for
// the requested global rows rows[r] = k n_v + v, v = i1 + n1 (i2 + n2 i3) —
// the reference's element() (src/tensor.cpp:183-196) for every column j, i.e.
// row_of_compressed_u (src/aca.cpp:234-244) on ACA stores.  One thread per
// (row, column): the three factor rows contracted into the core, O(r1 r2 r3).
// Accumulation in double for the c128 store, float for c64 (as the products).
template <typename C>
__global__ void rows_kernel(const TDesc* __restrict__ td, const C* __restrict__ arena, int64_t ncols, int64_t n1,
                            int64_t n2, int64_t nv, const int64_t* __restrict__ rows, C* __restrict__ out,
                            int64_t ldout) {
    using R = decltype(C{}.x);
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (j >= ncols) return;
    const int64_t row = rows[r];
    const int64_t k = row / nv, v = row - k * nv;
    const int64_t i1 = v % n1, i2 = (v / n1) % n2, i3 = v / (n1 * n2);
    const TDesc d = td[k * ncols + j];
    const C* G = arena + d.off_core;
    const C* u1 = arena + d.off_u1 + i1 * d.r1;
    const C* u2 = arena + d.off_u2 + i2 * d.r2;
    const C* u3 = arena + d.off_u3 + i3 * d.r3;
    C e = cmake<C>(R(0), R(0));
    for (int c = 0; c < d.r3; ++c) {
        C sc = cmake<C>(R(0), R(0));
        for (int b = 0; b < d.r2; ++b) {
            C sb = cmake<C>(R(0), R(0));
            const C* g = G + int64_t(d.r1) * (b + int64_t(d.r2) * c);
            for (int a = 0; a < d.r1; ++a) cfma(sb, u1[a], g[a]);
            cfma(sc, u2[b], sb);
        }
        cfma(e, u3[c], sc);
    }
    out[r + ldout * j] = e;
}

}  // namespace tmb
