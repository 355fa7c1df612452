// Batched multi-RHS forward on the tensor cores (K3 fwd_mrhs), complex64.
//
// Y[v, c] = sum_j T_j[v] X[j, c] for up to MR_P = 32 right-hand sides per
// launch — the reference's stacked_forward with p > 1 (src/matvec.cpp:17-65,
// per column a rank-1 update y_k += vec(T_jk) x(j,:)).  The decompressed
// column T_j is formed once per voxel tile (not once per right-hand side)
// and the accumulation is a dense GEMM on tcgen05:
//
//   M = voxels of the tile, N = right-hand sides, K = columns j.
//
// Tile: 1 i1 x 16 i2 x 32 i3 = 512 voxels = 4 MMA M-tiles of 128 voxels
// (lane = i2 + 16 (i3 % 8), M-tile = i3 / 8).  Per column the 8 producer
// warps form W[i2, c] = sum_b V[i1, b, c] U2[i2, b] (FFMA2; V = U1 x_1 G from
// the store's V arena), then T[i2, i3] = sum_c W[i2, c] U3[i3, c] and its
// 3xTF32 split into the A planes of the 4 M-tiles (one K slot per column).
// X arrives by TMA as 6 planes [-Xi][Xr][Xi] x {hi, lo} (built per call by
// mrhs_split_x_kernel), and one thread issues, per 8-column stage and
// M-tile, the complex-as-real product [Yr | Yi] += Tr.[Xr | Xi] +
// Ti.[-Xi | Xr] as 6 MMAs M=128 N=2*32 K=8.  The accumulators use the
// forward's chained accumulation (tm_kernels_tc.cuh): chains of `chain`
// stages in TMEM columns [0, 256), folded by 4 fold warps into a running
// sum at [256, 512), the last chain written to y.
//
// Warp roles (448 threads, 1 CTA / SM, persistent over tiles): warp 0 TMA
// (X planes), warp 1 MMA, warp 2 factor loader, warp 3 TMEM allocator,
// warps 4-11 producers, warps 12-15 fold + epilogue.
#pragma once

#include "tm_common.cuh"
#include "tm_kernels_tc.cuh"
#include "tm_sm100.cuh"

namespace tmb {

constexpr int MR_P = 32;          // right-hand sides per launch
constexpr int MR_TI2 = 16, MR_TI3 = 32;
constexpr int MR_NMT = 4;         // M-tiles per tile (8 i3 each)
constexpr int MR_NST = 2;         // stages (8 columns each)
constexpr int MR_JR = 3;          // factor-ring slots
constexpr int MR_NPW = 8;         // producer warps
constexpr int MR_PW0 = 4, MR_FW0 = MR_PW0 + MR_NPW;
constexpr int MR_THREADS = (MR_FW0 + 4) * 32;
constexpr int MR_A_PLANE = 128 * 32;                        // 4 KB
constexpr int MR_A_MT = 4 * MR_A_PLANE;                     // 16 KB per M-tile
constexpr int MR_A_STAGE = MR_NMT * MR_A_MT;                // 64 KB
constexpr int MR_B_PLANE = MR_P * 32;                       // 1 KB
constexpr int MR_B_STAGE = TC_BPLANES * MR_B_PLANE;         // 6 KB
constexpr int MR_WLD = 17;                                  // W row stride (float4)

struct MrGeom {
    int64_t ncols;
    int n1, n2, n3, q;
    int nt2, nt3;
    int64_t ntiles;   // q * n1 * nt2 * nt3
    int nks;          // stages per tile (ceil(ncols / 8))
    int chain;
    int slot_bytes, v_off, u2_off, u3_off;  // slot layout (bytes)
    int64_t t_begin, t_end;  // tile range of this launch
};

struct MrTile {
    int k, i1, i2_0, i3_0;
};

// i3 block fastest, then i2 block, then i1 (V rows of one i1 group stay hot).
__device__ __forceinline__ MrTile mr_tile(const MrGeom& g, int64_t t) {
    MrTile r;
    const int64_t per_k = int64_t(g.n1) * g.nt2 * g.nt3;
    r.k = int(t / per_k);
    int64_t rem = t - int64_t(r.k) * per_k;
    r.i1 = int(rem / (int64_t(g.nt2) * g.nt3));
    rem -= int64_t(r.i1) * g.nt2 * g.nt3;
    const int t2 = int(rem / g.nt3), t3 = int(rem - int64_t(t2) * g.nt3);
    r.i2_0 = t2 * MR_TI2;
    r.i3_0 = t3 * MR_TI3;
    return r;
}

__global__ void __launch_bounds__(MR_THREADS, 1)
    fwd_mrhs_kernel(const __grid_constant__ CUtensorMap xmap, const TcDesc* __restrict__ tcd,
                    const float2* __restrict__ varena, const float2* __restrict__ u2arena,
                    const float2* __restrict__ arena, MrGeom g, float2* __restrict__ y, int64_t ldy, int p) {
    using namespace sm100;
    extern __shared__ __align__(1024) unsigned char mr_smem_raw[];
    unsigned char* sm = mr_smem_raw + ((1024u - (smem_u32(mr_smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = sm;
    unsigned char* sB = sA + MR_NST * MR_A_STAGE;
    unsigned char* sSlot = sB + MR_NST * MR_B_STAGE;
    float4* sW = reinterpret_cast<float4*>(sSlot + MR_JR * g.slot_bytes);  // [2][16][MR_WLD]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sW + 2 * MR_TI2 * MR_WLD);
    uint64_t* full = bars;               // [NST]
    uint64_t* empty = full + MR_NST;     // [NST]
    uint64_t* ffull = empty + MR_NST;    // [JR]
    uint64_t* fempty = ffull + MR_JR;    // [JR]
    uint64_t* cfull = fempty + MR_JR;
    uint64_t* cfree = cfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfree + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < MR_NST; ++s) {
            mbar_init(&full[s], 1 + MR_NPW);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < MR_JR; ++s) {
            mbar_init(&ffull[s], 1);
            mbar_init(&fempty[s], MR_NPW);
        }
        mbar_init(cfull, 1);
        mbar_init(cfree, 4);
        fence_mbar_init();
    }
    if (warp == 3) tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) tma_prefetch_desc(&xmap);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ X-plane TMA producer
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = g.t_begin + blockIdx.x; t < g.t_end; t += gridDim.x) {
                for (int kk = 0; kk < g.nks; ++kk) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], uint32_t(MR_B_STAGE));
                    unsigned char* dst = sB + s * MR_B_STAGE;
#pragma unroll
                    for (int pl = 0; pl < TC_BPLANES; ++pl)
                        tma_load_3d(dst + pl * MR_B_PLANE, &xmap, &full[s], kk * 8, 0, pl);
                    if (++s == MR_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t idesc = umma_idesc_tf32(128, 2 * MR_P, false, false);
            uint32_t s = 0, ph = 0, gch = 0;
            for (int64_t t = g.t_begin + blockIdx.x; t < g.t_end; t += gridDim.x) {
                int cpos = 0;
                for (int kk = 0; kk < g.nks; ++kk) {
                    if (cpos == 0) {
                        mbar_wait(cfree, (gch & 1) ^ 1);
                        tc_fence_after();
                    }
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t b0 = smem_u32(sB + s * MR_B_STAGE);
                    const uint64_t B1h = umma_smem_desc(b0 + 1 * MR_B_PLANE, 256, 6);
                    const uint64_t B2h = umma_smem_desc(b0 + 0 * MR_B_PLANE, 256, 6);
                    const uint64_t B1l = umma_smem_desc(b0 + 4 * MR_B_PLANE, 256, 6);
                    const uint64_t B2l = umma_smem_desc(b0 + 3 * MR_B_PLANE, 256, 6);
                    const uint32_t acc = cpos > 0 ? 1u : 0u;
#pragma unroll
                    for (int mt = 0; mt < MR_NMT; ++mt) {
                        const uint32_t a0 = smem_u32(sA + s * MR_A_STAGE + mt * MR_A_MT);
                        uint64_t A[4];
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) A[pl] = umma_smem_desc(a0 + pl * MR_A_PLANE, 256, 6);
                        const uint32_t yd = tmem + uint32_t(mt * 2 * MR_P);
                        mma_tf32(yd, A[0], B1h, idesc, acc);
                        mma_tf32(yd, A[0], B1l, idesc, 1);
                        mma_tf32(yd, A[1], B1h, idesc, 1);
                        mma_tf32(yd, A[2], B2h, idesc, 1);
                        mma_tf32(yd, A[2], B2l, idesc, 1);
                        mma_tf32(yd, A[3], B2h, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (++s == MR_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                    if (++cpos == g.chain || kk == g.nks - 1) {
                        mma_commit(cfull);
                        cpos = 0;
                        ++gch;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---------------------------------------------------- factor loader
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = g.t_begin + blockIdx.x; t < g.t_end; t += gridDim.x) {
                const MrTile tl = mr_tile(g, t);
                const TcDesc* tdk = tcd + int64_t(tl.k) * g.ncols;
                for (int64_t j = 0; j < g.ncols; ++j) {
                    mbar_wait(&fempty[s], ph ^ 1);
                    const TcDesc d = tdk[j];
                    unsigned char* slot = sSlot + s * g.slot_bytes;
                    const uint32_t r23 = uint32_t(d.r2 * d.r3);
                    const uint32_t ld2 = uint32_t(d.r2 | 1);
                    const uint32_t bv = round16(uint32_t(TC_TI1) * r23 * 8u);  // the 4-row V group of i1
                    const uint32_t b2 = uint32_t(MR_TI2) * ld2 * 8u;
                    const uint32_t b3 = round16(uint32_t(MR_TI3 * d.r3) * 8u);
                    mbar_arrive_expect_tx(&ffull[s], uint32_t(sizeof(TcDesc)) + bv + b2 + b3);
                    bulk_g2s(slot, tdk + j, uint32_t(sizeof(TcDesc)), &ffull[s]);
                    bulk_g2s(slot + g.v_off, varena + d.off_v + int64_t(tl.i1 & ~3) * r23, bv, &ffull[s]);
                    bulk_g2s(slot + g.u2_off, u2arena + d.off_u2 + int64_t(tl.i2_0) * ld2, b2, &ffull[s]);
                    bulk_g2s(slot + g.u3_off, arena + d.off_u3 + int64_t(tl.i3_0) * d.r3, b3, &ffull[s]);
                    if (++s == MR_JR) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp >= MR_PW0 && warp < MR_FW0) {
        // -------------------------------------------------------- producers
        const int pt = threadIdx.x - MR_PW0 * 32;  // 0..255
        // phase A thread: W[i2a, ca] (ca = pt / 16, up to 16 c values)
        const int i2a = pt & 15, ca = pt >> 4;
        // phase B thread: voxels (i2b, i3 = 2 ib) and (i2b, 2 ib + 1)
        const int i2b = pt & 15, ib = pt >> 4;  // ib 0..15
        uint32_t fs = 0, fph = 0, s = 0, ph = 0, kpos = 0;
        int wb = 0;
        // A-plane byte offset of each of my two voxels (M-tile, lane, swizzle row)
        uint32_t aoff[2], xorv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i3l = 2 * ib + e;
            const int mt = i3l >> 3, ln = i2b + 16 * (i3l & 7);
            aoff[e] = uint32_t(mt * MR_A_MT + ln * 32);
            xorv[e] = (uint32_t(ln) & 4u) << 2;
        }
        for (int64_t t = g.t_begin + blockIdx.x; t < g.t_end; t += gridDim.x) {
            const MrTile tl = mr_tile(g, t);
            const bool i2ok = tl.i2_0 + i2a < g.n2;
            for (int64_t j = 0; j < g.ncols; ++j) {
                mbar_wait(&ffull[fs], fph);
                const unsigned char* slot = sSlot + fs * g.slot_bytes;
                const int r2 = reinterpret_cast<const TcDesc*>(slot)->r2;
                const int r3 = reinterpret_cast<const TcDesc*>(slot)->r3;
                const float2* V = reinterpret_cast<const float2*>(slot + g.v_off) + (tl.i1 & 3);
                const float2* U2 = reinterpret_cast<const float2*>(slot + g.u2_off);
                const float2* U3 = reinterpret_cast<const float2*>(slot + g.u3_off);
                float4* W = sW + wb * MR_TI2 * MR_WLD;
                // phase A: W[i2, c] = sum_b V[i1, b, c] U2[i2, b]  -> (wr, wi, -wi, wr)
                if (ca < r3) {
                    uint64_t acc = 0;
                    const float2* vp = V + 4 * ca;  // V[(c + r3 b) * 4 + il]
                    const float2* up = U2 + i2a * (r2 | 1);
                    for (int b = 0; b < r2; ++b) cfma2v(acc, vp[4 * r3 * b], up[b]);
                    float2 w = f2_unpack(acc);
                    if (!i2ok) w = make_float2(0.f, 0.f);
                    W[i2a * MR_WLD + ca] = make_float4(w.x, w.y, -w.y, w.x);
                }
                named_bar_sync(1, MR_NPW * 32);  // W complete
                // phase B: T[i2, i3] = sum_c W[i2, c] U3[i3, c] for my two voxels
                uint64_t t0 = 0, t1 = 0;
                const float4* wp = W + i2b * MR_WLD;
                const float2* u3p = U3 + (2 * ib) * r3;
                for (int c = 0; c < r3; ++c) {
                    const float4 wv = wp[c];
                    cfma2(t0, wv, u3p[c]);
                    cfma2(t1, wv, u3p[r3 + c]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&fempty[fs]);  // slot (V, U2, U3) no longer read
                if (++fs == MR_JR) {
                    fs = 0;
                    fph ^= 1;
                }
                wb ^= 1;
                // i3 outside the grid contributes zero (U3 rows past n3 are
                // whatever follows in the arena)
                if (tl.i3_0 + 2 * ib >= g.n3) t0 = 0;
                if (tl.i3_0 + 2 * ib + 1 >= g.n3) t1 = 0;
                if (kpos == 0) mbar_wait(&empty[s], ph ^ 1u);
                unsigned char* st = sA + s * MR_A_STAGE;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float2 tv = f2_unpack(e ? t1 : t0);
                    const float hr = __uint_as_float(__float_as_uint(tv.x) & 0xFFFFE000u);
                    const float hi = __uint_as_float(__float_as_uint(tv.y) & 0xFFFFE000u);
                    float* a = reinterpret_cast<float*>(st + aoff[e] + ((kpos * 4u) ^ xorv[e]));
                    a[0] = hr;
                    a[MR_A_PLANE / 4] = tv.x - hr;
                    a[2 * MR_A_PLANE / 4] = hi;
                    a[3 * MR_A_PLANE / 4] = tv.y - hi;
                }
                if (++kpos == 8) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[s]);
                    kpos = 0;
                    if (++s == MR_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
            if (kpos != 0) {  // zero the tail K slots of the last stage and close it
                unsigned char* st = sA + s * MR_A_STAGE;
                for (uint32_t kq = kpos; kq < 8; ++kq)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        float* a = reinterpret_cast<float*>(st + aoff[e] + ((kq * 4u) ^ xorv[e]));
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) a[pl * MR_A_PLANE / 4] = 0.f;
                    }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                kpos = 0;
                if (++s == MR_NST) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp >= MR_FW0) {
        // ------------------------------------------ chain fold + epilogue
        const int quarter = warp & 3;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const uint32_t tC = tmem + lane_addr, tR = tmem + lane_addr + TC_RUN_COL;
        const int ln = quarter * 32 + lane;              // lane inside each M-tile
        const int i2l = ln & 15, i3s = ln >> 4;          // i3 = 8 mt + i3s
        const int64_t nv3 = int64_t(g.n1) * g.n2 * g.n3;
        const int nch = (g.nks + g.chain - 1) / g.chain;
        uint32_t gch = 0;
        for (int64_t t = g.t_begin + blockIdx.x; t < g.t_end; t += gridDim.x) {
            const MrTile tl = mr_tile(g, t);
            const int i2 = tl.i2_0 + i2l;
            for (int ch = 0; ch < nch; ++ch, ++gch) {
                mbar_wait(cfull, gch & 1);
                tc_fence_after();
                const bool last = ch == nch - 1;
                for (int mt = 0; mt < MR_NMT; ++mt) {
                    const uint32_t cb = uint32_t(mt * 2 * MR_P);
                    uint32_t cr[16], ci[16];
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        tmem_ld16(tC + cb + uint32_t(16 * half), cr);
                        tmem_ld16(tC + cb + uint32_t(MR_P + 16 * half), ci);
                        if (ch > 0) {
                            uint32_t rr[16], ri[16];
                            tmem_ld16(tR + cb + uint32_t(16 * half), rr);
                            tmem_ld16(tR + cb + uint32_t(MR_P + 16 * half), ri);
                            tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                cr[i] = __float_as_uint(__uint_as_float(cr[i]) + __uint_as_float(rr[i]));
                                ci[i] = __float_as_uint(__uint_as_float(ci[i]) + __uint_as_float(ri[i]));
                            }
                        } else {
                            tmem_ld_wait();
                        }
                        if (!last) {
                            tmem_st16(tR + cb + uint32_t(16 * half), cr);
                            tmem_st16(tR + cb + uint32_t(MR_P + 16 * half), ci);
                        } else {
                            const int i3 = tl.i3_0 + 8 * mt + i3s;
                            if (i2 < g.n2 && i3 < g.n3) {
                                float2* yp = y + int64_t(tl.k) * nv3 + tl.i1 + int64_t(g.n1) * (i2 + int64_t(g.n2) * i3);
#pragma unroll
                                for (int i = 0; i < 16; ++i) {
                                    const int c = 16 * half + i;
                                    if (c < p) yp[ldy * c] = make_float2(__uint_as_float(cr[i]), __uint_as_float(ci[i]));
                                }
                            }
                        }
                    }
                }
                if (!last) tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(cfree);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc(tmem, 512);
}

// X (m x p c64, column-major, p <= 32) -> 6 TF32 planes [pl][32][mp]
// (-Xi, Xr, Xi hi; the same lo), rows c >= p and columns j >= m zero.
__global__ void mrhs_split_x_kernel(const float2* __restrict__ x, int64_t ldx, int64_t m, int p, int64_t mp,
                                    float* __restrict__ planes) {
    const int64_t n = int64_t(MR_P) * mp;
    const int64_t plane = n;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e / mp);
        const int64_t j = e - int64_t(c) * mp;
        float2 v = make_float2(0.f, 0.f);
        if (c < p && j < m) v = x[j + ldx * c];
        const float rh = sm100::tf32_round(v.x), ih = sm100::tf32_round(v.y);
        const float rl = sm100::tf32_round(v.x - rh), il = sm100::tf32_round(v.y - ih);
        planes[e] = -ih;
        planes[plane + e] = rh;
        planes[2 * plane + e] = ih;
        planes[3 * plane + e] = -il;
        planes[4 * plane + e] = rl;
        planes[5 * plane + e] = il;
    }
}

}  // namespace tmb
