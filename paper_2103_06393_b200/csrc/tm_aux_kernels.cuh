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

// y[i] += x[i] (the emulated communicator's reduce, tm_shard.cuh)
template <typename C>
__global__ void add_kernel(C* __restrict__ y, const C* __restrict__ x, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        C a = y[i];
        const C b = x[i];
        a.x += b.x;
        a.y += b.y;
        y[i] = a;
    }
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

// ------------------------------------------------ column assembly (§8f-1)
// assemble_column (src/scene.cpp:127-150) on the device, complex128: for
// each requested source column and every voxel, the E-field (op 0,
// src/scene.cpp:84-103) or H-field (op 1, :105-118) kernel of the RWG-like
// edge source {midpoint, unit direction, weight} at the voxel centre (q = 3)
// or the PWL stand-in's 2 x 2 x 2 Gauss moments against {1, x~, y~, z~}
// (q = 12; points at +-h / (2 sqrt 3), weights 1/8) — the definitions of
// the oracle's voxel_field and compress.assemble_columns.  Output
// out[(b * q + comp) * nv + v], v = i1 + n1 (i2 + n2 i3) (component-major
// rows, voxel f1-fastest: src/compress.cpp:52-65).  One thread per (voxel,
// column).  Returns nonzero in *bad when an observation point coincides
// with a source (the reference's SingularityError, R < 1e-12).
struct AsmScene {
    double ox, oy, oz, h, k0;
    int n1, n2, n3, q, op;
};

__device__ __forceinline__ void asm_field(const AsmScene& sc, const double* __restrict__ s, double px, double py,
                                          double pz, double2 (&f)[3], int* __restrict__ bad) {
    const double rx = px - s[0], ry = py - s[1], rz = pz - s[2];
    const double R = sqrt(rx * rx + ry * ry + rz * rz);
    if (R < 1e-12) {
        atomicExch(bad, 1);
        f[0] = f[1] = f[2] = make_double2(0.0, 0.0);
        return;
    }
    const double iR = 1.0 / R;
    const double hx = rx * iR, hy = ry * iR, hz = rz * iR;
    double sn, cs;
    sincos(sc.k0 * R, &sn, &cs);
    const double m = 1.0 / (4.0 * 3.14159265358979323846 * R);
    const double gr = m * cs, gi = -m * sn;  // g = exp(-i k0 R) / (4 pi R)
    const double w = s[6], dx = s[3], dy = s[4], dz = s[5];
    if (sc.op == 0) {
        const double ar0 = sc.k0 * sc.k0 - iR * iR, ai0 = -sc.k0 * iR;          // a = g (k0^2 - 1/R^2 - i k0/R)
        const double br0 = -sc.k0 * sc.k0 + 3.0 * iR * iR, bi0 = 3.0 * sc.k0 * iR;  // b = g (-k0^2 + 3/R^2 + 3 i k0/R)
        const double ar = gr * ar0 - gi * ai0, ai = gr * ai0 + gi * ar0;
        const double br = gr * br0 - gi * bi0, bi = gr * bi0 + gi * br0;
        const double pr = hx * dx + hy * dy + hz * dz;
        const double d[3] = {dx, dy, dz}, hh[3] = {hx, hy, hz};
#pragma unroll
        for (int c = 0; c < 3; ++c)
            f[c] = make_double2(w * (ar * d[c] + br * pr * hh[c]), w * (ai * d[c] + bi * pr * hh[c]));
    } else {
        const double cr = -(gr * iR - gi * sc.k0), ci = -(gr * sc.k0 + gi * iR);  // gc = -g (1/R + i k0)
        const double x0 = hy * dz - hz * dy, x1 = hz * dx - hx * dz, x2 = hx * dy - hy * dx;  // rh x d
        f[0] = make_double2(w * cr * x0, w * ci * x0);
        f[1] = make_double2(w * cr * x1, w * ci * x1);
        f[2] = make_double2(w * cr * x2, w * ci * x2);
    }
}

__global__ void assemble_kernel(AsmScene sc, const double* __restrict__ src, const int64_t* __restrict__ cols,
                                int64_t nb, double2* __restrict__ out, int* __restrict__ bad) {
    const int64_t nv = int64_t(sc.n1) * sc.n2 * sc.n3;
    const int64_t b = blockIdx.y;
    const double* s = src + 7 * cols[b];
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv; v += int64_t(gridDim.x) * blockDim.x) {
        const int i1 = int(v % sc.n1);
        const int64_t rest = v / sc.n1;
        const int i2 = int(rest % sc.n2), i3 = int(rest / sc.n2);
        const double cx = sc.ox + sc.h * (i1 + 0.5), cy = sc.oy + sc.h * (i2 + 0.5), cz = sc.oz + sc.h * (i3 + 0.5);
        double2* o = out + (b * sc.q) * nv + v;
        if (sc.q == 3) {
            double2 f[3];
            asm_field(sc, s, cx, cy, cz, f, bad);
#pragma unroll
            for (int c = 0; c < 3; ++c) o[c * nv] = f[c];
        } else {
            double2 acc[12];
#pragma unroll
            for (int e = 0; e < 12; ++e) acc[e] = make_double2(0.0, 0.0);
            const double off = 0.5 / sqrt(3.0);
#pragma unroll
            for (int gz = 0; gz < 2; ++gz)
#pragma unroll
                for (int gy = 0; gy < 2; ++gy)
#pragma unroll
                    for (int gx = 0; gx < 2; ++gx) {
                        const double lx = gx ? off : -off, ly = gy ? off : -off, lz = gz ? off : -off;
                        double2 f[3];
                        asm_field(sc, s, cx + sc.h * lx, cy + sc.h * ly, cz + sc.h * lz, f, bad);
                        const double phi[4] = {1.0, lx, ly, lz};
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int mu = 0; mu < 4; ++mu) {
                                const double wq = 0.125 * phi[mu];
                                acc[4 * c + mu].x += wq * f[c].x;
                                acc[4 * c + mu].y += wq * f[c].y;
                            }
                    }
#pragma unroll
            for (int e = 0; e < 12; ++e) o[e * nv] = acc[e];
        }
    }
}
