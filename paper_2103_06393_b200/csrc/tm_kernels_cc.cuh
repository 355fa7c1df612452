// CUDA-core (FFMA / DFMA) forward and adjoint kernels on the device store.
//
// Both kernels tile the output grid of one component k into CTA tiles of
// ROWS = TI1 x TI2 voxel rows (i1 fastest) times TI3 = 32*CN voxels along
// mode 3, and walk every column j of the store for that tile.  Per column
// the CTA decompresses only its tile, in three stages (the reference's
// reconstruct -> mode_product x3, src/tensor.cpp:89-120,176-181, but
// restricted to the tile and never materialising the n^3 tensor):
//   V[i1, r2, r3] = sum_r1 U1[i1, r1] G[r1, r2, r3]          (mode 1, tile rows)
//   W[row, r3]    = s_j * sum_r2 V[i1, r2, r3] U2[i2, r2]    (mode 2)
//   T[row, i3]    = sum_r3 W[row, r3] U3[i3, r3]             (mode 3, registers)
// The forward (Algorithm 1, src/matvec.cpp:17-65) folds s_j = x_j into W and
// accumulates T into per-thread registers over all j — the tile of y is
// written exactly once.  The adjoint (Algorithm 2, src/matvec.cpp:67-102)
// keeps the tile of Phi in registers and forms
//   z_j = sum_{row,i3} conj(T[row,i3]) Phi[row,i3]
//       = sum_{r3,row} conj(W[row,r3]) sum_i3 conj(U3[i3,r3]) Phi[row,i3]
// so it never forms T either; per-tile partial z_j are reduced across the
// CTA with warp shuffles and written to a partials buffer that a second
// kernel sums over tiles and components in a fixed order (deterministic).
//
// Thread mapping: warp w owns RM consecutive tile rows, lane l owns CN
// consecutive i3.  In the mode-3 loop the W values are warp-uniform
// (shared-memory broadcast) and the U3 values are lane-contiguous, so each
// r3 step costs RM+CN complex smem loads for RM*CN complex FMAs.
#pragma once

#include "tm_common.cuh"

namespace tmb {

struct CcGeom {
    int64_t ncols;    // columns j of the store
    int n1, n2, n3;
    int q;
    int nt1, nt2;     // tile counts along modes 1 and 2
    int rmax1, rmax2, rmax3;
    int jb;           // columns staged per shared-memory round
    int ntiles;       // nt1 * nt2 * nt3: blockIdx.x = tile + ntiles * part
    int nsplit;       // column ranges per tile (> 1 when tiles x q x p < the SMs)
    int64_t part_stride;  // forward with nsplit > 1: elements between the parts' partial y blocks
    int k0;               // forward: first component (blockIdx.y = k - k0; tm_forward_components)
};

// Column range [ja, jz) of split part `part` (contiguous, balanced by count).
__device__ __forceinline__ void cc_columns(const CcGeom& g, int part, int64_t& ja, int64_t& jz) {
    ja = g.ncols * part / g.nsplit;
    jz = g.ncols * (part + 1) / g.nsplit;
}

// Shared-memory plan (elements of C) for one staged column.
template <int TI1, int TI2, int TI3>
__host__ __device__ inline int64_t cc_slot_elems(int rmax1, int rmax2, int rmax3) {
    auto a2 = [](int64_t v) { return (v + 1) & ~int64_t(1); };  // keep 16-byte alignment for float2
    return a2(int64_t(TI1) * rmax1) + a2(int64_t(TI2) * rmax2) + a2(int64_t(rmax3) * TI3) +
           a2(int64_t(TI1) * rmax2 * rmax3) + a2(int64_t(rmax3) * TI1 * TI2);
}

template <typename C, int TI1, int TI2, int TI3>
struct CcSlot {
    C* u1;  // [TI1][r1]
    C* u2;  // [TI2][r2]
    C* u3;  // [r3][TI3]   (transposed: lane-contiguous along i3)
    C* v;   // [TI1][r2*r3]
    C* w;   // [r3][ROWS]
    __device__ CcSlot(C* base, const CcGeom& g) {
        auto a2 = [](int64_t v) { return (v + 1) & ~int64_t(1); };
        u1 = base;
        u2 = u1 + a2(int64_t(TI1) * g.rmax1);
        u3 = u2 + a2(int64_t(TI2) * g.rmax2);
        v = u3 + a2(int64_t(g.rmax3) * TI3);
        w = v + a2(int64_t(TI1) * g.rmax2 * g.rmax3);
    }
};

// Stage a chunk of up to jb columns into shared memory and decompress the
// tile's W for each (stages mode 1 and mode 2).  `scale` supplies s_j.
template <typename C, int TI1, int TI2, int TI3, int NT, typename ScaleFn>
__device__ __forceinline__ void cc_stage_chunk(const TDesc* __restrict__ td, const C* __restrict__ arena,
                                               const CcGeom& g, int k, int64_t j0, int nj, int i1_0, int i2_0,
                                               int i3_0, C* smem, int64_t slot, ScaleFn scale) {
    constexpr int ROWS = TI1 * TI2;
    const int tid = threadIdx.x;
    using R = decltype(C{}.x);
    const C zero = cmake<C>(R(0), R(0));
    // --- loads: factor rows of the tile --------------------------------------
    for (int jj = 0; jj < nj; ++jj) {
        const TDesc d = td[int64_t(k) * g.ncols + j0 + jj];
        CcSlot<C, TI1, TI2, TI3> s(smem + jj * slot, g);
        const C* u1 = arena + d.off_u1 + int64_t(i1_0) * d.r1;
        const int n1v = min(TI1, g.n1 - i1_0);
        for (int e = tid; e < TI1 * d.r1; e += NT) s.u1[e] = (e < n1v * d.r1) ? u1[e] : zero;
        const C* u2 = arena + d.off_u2 + int64_t(i2_0) * d.r2;
        const int n2v = min(TI2, g.n2 - i2_0);
        for (int e = tid; e < TI2 * d.r2; e += NT) s.u2[e] = (e < n2v * d.r2) ? u2[e] : zero;
        const C* u3 = arena + d.off_u3 + int64_t(i3_0) * d.r3;
        const int n3v = min(TI3, g.n3 - i3_0);
        for (int e = tid; e < TI3 * d.r3; e += NT) {
            const int i = e / d.r3, r = e - i * d.r3;
            s.u3[r * TI3 + i] = (i < n3v) ? u3[e] : zero;
        }
    }
    __syncthreads();
    // --- mode 1: V[i1l][b + r2*c] = sum_a U1[i1l][a] G[a + r1*(b + r2*c)] ------
    for (int jj = 0; jj < nj; ++jj) {
        const TDesc d = td[int64_t(k) * g.ncols + j0 + jj];
        CcSlot<C, TI1, TI2, TI3> s(smem + jj * slot, g);
        const C* G = arena + d.off_core;
        const int r23 = d.r2 * d.r3;
        for (int e = tid; e < TI1 * r23; e += NT) {
            const int i1l = e / r23, bc = e - i1l * r23;
            C acc = zero;
            const C* gp = G + int64_t(bc) * d.r1;
            const C* up = s.u1 + i1l * d.r1;
            // independent core loads in flight (L2 latency, not FMA, bounds this loop)
#pragma unroll 4
            for (int a = 0; a < d.r1; ++a) cfma(acc, up[a], __ldg(reinterpret_cast<const C*>(gp + a)));
            s.v[e] = acc;
        }
    }
    __syncthreads();
    // --- mode 2: W[c][row] = s_j * sum_b V[i1l][b + r2*c] U2[i2l][b] ----------
    for (int jj = 0; jj < nj; ++jj) {
        const TDesc d = td[int64_t(k) * g.ncols + j0 + jj];
        CcSlot<C, TI1, TI2, TI3> s(smem + jj * slot, g);
        const C sj = scale(j0 + jj);
        const int r23 = d.r2 * d.r3;
        for (int e = tid; e < ROWS * d.r3; e += NT) {
            const int c = e / ROWS, row = e - c * ROWS;
            const int i1l = row % TI1, i2l = row / TI1;
            C acc = zero;
            const C* vp = s.v + i1l * r23 + d.r2 * c;
            const C* up = s.u2 + i2l * d.r2;
#pragma unroll 4
            for (int b = 0; b < d.r2; ++b) cfma(acc, vp[b], up[b]);
            s.w[e] = cmul(acc, sj);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------- forward --
template <typename C, int RM, int CN, int NW, int TI1>
__global__ void __launch_bounds__(NW * 32)
    fwd_cc_kernel(const TDesc* __restrict__ td, const C* __restrict__ arena, CcGeom g, const C* __restrict__ x,
                  int64_t ldx, C* __restrict__ y, int64_t ldy) {
    constexpr int NT = NW * 32;
    constexpr int ROWS = RM * NW;
    constexpr int TI2 = ROWS / TI1;
    constexpr int TI3 = 32 * CN;
    static_assert(ROWS % TI1 == 0, "tile rows must be a multiple of TI1");
    using R = decltype(C{}.x);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* smem = reinterpret_cast<C*>(smem_raw);

    const int tile = int(blockIdx.x % unsigned(g.ntiles)), part = int(blockIdx.x / unsigned(g.ntiles));
    const int t1 = tile % g.nt1;
    const int t2 = (tile / g.nt1) % g.nt2;
    const int t3 = tile / (g.nt1 * g.nt2);
    const int k = g.k0 + int(blockIdx.y);
    const int c = blockIdx.z;
    const int i1_0 = t1 * TI1, i2_0 = t2 * TI2, i3_0 = t3 * TI3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = cc_slot_elems<TI1, TI2, TI3>(g.rmax1, g.rmax2, g.rmax3);
    const C* xc = x + ldx * c;
    int64_t ja, jz;
    cc_columns(g, part, ja, jz);

    C acc[RM][CN];
#pragma unroll
    for (int a = 0; a < RM; ++a)
#pragma unroll
        for (int b = 0; b < CN; ++b) acc[a][b] = cmake<C>(R(0), R(0));

    for (int64_t j0 = ja; j0 < jz; j0 += g.jb) {
        const int nj = int(jz - j0 < int64_t(g.jb) ? jz - j0 : int64_t(g.jb));
        cc_stage_chunk<C, TI1, TI2, TI3, NT>(td, arena, g, k, j0, nj, i1_0, i2_0, i3_0, smem, slot,
                                             [&](int64_t j) { return xc[j]; });
        for (int jj = 0; jj < nj; ++jj) {
            const int r3 = td[int64_t(k) * g.ncols + j0 + jj].r3;
            CcSlot<C, TI1, TI2, TI3> s(smem + jj * slot, g);
            const C* wp = s.w + warp * RM;
            const C* up = s.u3 + lane * CN;
#pragma unroll 2
            for (int r = 0; r < r3; ++r) {
                C wv[RM], uv[CN];
#pragma unroll
                for (int a = 0; a < RM; ++a) wv[a] = wp[r * ROWS + a];
#pragma unroll
                for (int b = 0; b < CN; ++b) uv[b] = up[r * TI3 + b];
#pragma unroll
                for (int a = 0; a < RM; ++a)
#pragma unroll
                    for (int b = 0; b < CN; ++b) cfma(acc[a][b], wv[a], uv[b]);
            }
        }
        __syncthreads();  // smem is restaged by the next chunk
    }

    // --- epilogue: y[k n_v + i1 + n1 (i2 + n2 i3), c] (a split part: its
    // partial block, summed in part order by cc_split_reduce_kernel) ------------
    const int64_t nv = int64_t(g.n1) * g.n2 * g.n3;
    C* yc = y + g.part_stride * part + ldy * c + int64_t(k) * nv;
#pragma unroll
    for (int a = 0; a < RM; ++a) {
        const int row = warp * RM + a;
        const int i1 = i1_0 + row % TI1, i2 = i2_0 + row / TI1;
        if (i1 >= g.n1 || i2 >= g.n2) continue;
#pragma unroll
        for (int b = 0; b < CN; ++b) {
            const int i3 = i3_0 + lane * CN + b;
            if (i3 < g.n3) yc[i1 + int64_t(g.n1) * (i2 + int64_t(g.n2) * i3)] = acc[a][b];
        }
    }
}

// ---------------------------------------------------------------- adjoint --
// part layout: part[((c * ncols + j) * q + k) * ntiles + tile]
template <typename C, int RM, int CN, int NW, int TI1>
__global__ void __launch_bounds__(NW * 32)
    adj_cc_kernel(const TDesc* __restrict__ td, const C* __restrict__ arena, CcGeom g, const C* __restrict__ phi,
                  int64_t ldphi, C* __restrict__ part) {
    constexpr int NT = NW * 32;
    constexpr int ROWS = RM * NW;
    constexpr int TI2 = ROWS / TI1;
    constexpr int TI3 = 32 * CN;
    constexpr int JBMAX = 8;
    using R = decltype(C{}.x);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* smem = reinterpret_cast<C*>(smem_raw);

    const int ntiles = g.ntiles;
    const int tile = int(blockIdx.x % unsigned(ntiles)), part_id = int(blockIdx.x / unsigned(ntiles));
    const int t1 = tile % g.nt1;
    const int t2 = (tile / g.nt1) % g.nt2;
    const int t3 = tile / (g.nt1 * g.nt2);
    const int k = blockIdx.y;
    const int c = blockIdx.z;
    const int i1_0 = t1 * TI1, i2_0 = t2 * TI2, i3_0 = t3 * TI3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = cc_slot_elems<TI1, TI2, TI3>(g.rmax1, g.rmax2, g.rmax3);
    C* red = smem + slot * g.jb;  // [JBMAX][NW]

    // Tile of Phi in registers (zero outside the grid).
    const int64_t nv = int64_t(g.n1) * g.n2 * g.n3;
    const C* pc = phi + ldphi * c + int64_t(k) * nv;
    C ph[RM][CN];
#pragma unroll
    for (int a = 0; a < RM; ++a) {
        const int row = warp * RM + a;
        const int i1 = i1_0 + row % TI1, i2 = i2_0 + row / TI1;
#pragma unroll
        for (int b = 0; b < CN; ++b) {
            const int i3 = i3_0 + lane * CN + b;
            ph[a][b] = (i1 < g.n1 && i2 < g.n2 && i3 < g.n3)
                           ? pc[i1 + int64_t(g.n1) * (i2 + int64_t(g.n2) * i3)]
                           : cmake<C>(R(0), R(0));
        }
    }
    const C one = cmake<C>(R(1), R(0));
    int64_t ja, jz;  // this part's columns (each column's partials come from exactly one part)
    cc_columns(g, part_id, ja, jz);

    for (int64_t j0 = ja; j0 < jz; j0 += g.jb) {
        const int nj = int(jz - j0 < int64_t(g.jb) ? jz - j0 : int64_t(g.jb));
        cc_stage_chunk<C, TI1, TI2, TI3, NT>(td, arena, g, k, j0, nj, i1_0, i2_0, i3_0, smem, slot,
                                             [&](int64_t) { return one; });
        for (int jj = 0; jj < nj; ++jj) {
            const int r3 = td[int64_t(k) * g.ncols + j0 + jj].r3;
            CcSlot<C, TI1, TI2, TI3> s(smem + jj * slot, g);
            const C* wp = s.w + warp * RM;
            const C* up = s.u3 + lane * CN;
            C accj = cmake<C>(R(0), R(0));
#pragma unroll 2
            for (int r = 0; r < r3; ++r) {
                C uv[CN];
#pragma unroll
                for (int b = 0; b < CN; ++b) uv[b] = up[r * TI3 + b];
#pragma unroll
                for (int a = 0; a < RM; ++a) {
                    C qv = cmake<C>(R(0), R(0));
#pragma unroll
                    for (int b = 0; b < CN; ++b) cfma_conj(qv, uv[b], ph[a][b]);
                    cfma_conj(accj, wp[r * ROWS + a], qv);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                accj.x += __shfl_xor_sync(0xffffffffu, accj.x, o);
                accj.y += __shfl_xor_sync(0xffffffffu, accj.y, o);
            }
            if (lane == 0) red[jj * NW + warp] = accj;
        }
        __syncthreads();
        if (threadIdx.x < nj) {
            const int jj = threadIdx.x;
            C sum = cmake<C>(R(0), R(0));
            for (int w = 0; w < NW; ++w) {
                sum.x += red[jj * NW + w].x;
                sum.y += red[jj * NW + w].y;
            }
            part[((int64_t(c) * g.ncols + j0 + jj) * g.q + k) * ntiles + tile] = sum;
        }
        // the next chunk's first __syncthreads (after its loads) orders these
        // reads of `red` before it is rewritten
        static_assert(JBMAX >= 1, "");
    }
}

// Forward with split columns: y[row + ldy c] = sum_s yp[s stride + rows c + row],
// in part order (deterministic).
template <typename C>
__global__ void cc_split_reduce_kernel(const C* __restrict__ yp, int nsplit, int64_t stride, int64_t rows, int64_t p,
                                       C* __restrict__ y, int64_t ldy, int64_t r0 = 0, int64_t nr = -1) {
    // rows [r0, r0 + nr) of each column (all rows when nr < 0)
    if (nr < 0) nr = rows;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nr * p;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = e / nr, r = r0 + (e - c * nr);
        const int64_t ei = r + rows * c;
        C acc = yp[ei];
        for (int sp = 1; sp < nsplit; ++sp) {
            const C v = yp[sp * stride + ei];
            acc.x += v.x;
            acc.y += v.y;
        }
        y[r + ldy * c] = acc;
    }
}

// z[j + ldz c] = sum_{k, tile} part[...] in a fixed order, accumulated in f64.
template <typename C>
__global__ void adj_reduce_kernel(const C* __restrict__ part, int64_t ncols, int64_t p, int64_t nred, C* __restrict__ z,
                                  int64_t ldz) {
    using R = decltype(C{}.x);
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= ncols * p) return;
    const int64_t j = wid % ncols, c = wid / ncols;
    const C* src = part + wid * nred;
    double sx = 0.0, sy = 0.0;
    for (int64_t i = lane; i < nred; i += 32) {
        sx += double(src[i].x);
        sy += double(src[i].y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    if (lane == 0) z[j + ldz * c] = cmake<C>(R(sx), R(sy));
}

}  // namespace tmb
