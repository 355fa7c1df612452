// Tensor-core (tcgen05, kind::tf32, 3xTF32 split) forward kernel, complex64.
//
// Forward of component k, for one output tile of ROWS = 128 voxel rows
// (TI1 x TI2 = 4 x 32 of (i1, i2)) times NMMA <= 128 voxels along mode 3:
//
//   Y[row, i3] = sum_j sum_r W_j[row, r] U3_j[i3, r],
//   W_j[row, r] = sum_b V_j[i1, b, r] U2_j[i2, b],  V_j = x_j (U1_j x_1 G_j),
//
// i.e. one GEMM with K = the packed (j, r) stream of component k
// (K = sum_j r3_j, no per-column padding) — the reference's stacked_forward
// (src/matvec.cpp:17-65) with reconstruct's three mode products
// (src/tensor.cpp:89-120,176-181) restricted to the tile.  The B operand
// (U3 of every column, concatenated along K) is pre-split at store creation
// into four fp32 planes {Re hi, Re lo, Im hi, Im lo} (hi = tf32(x),
// lo = tf32(x - hi)), laid out [plane][k][i3][K] and streamed by TMA
// (SWIZZLE_32B, 8 K per stage).  The A operand W is produced on the fly by 8
// producer warps (FFMA2 mode products) into the same four-plane split in
// shared memory (hi = W with the low 13 mantissa bits cleared, lo = W - hi),
// so no decompressed column is ever written anywhere.  Per 8-wide K step the
// MMA warp issues 12 tcgen05.mma (M=128, N=NMMA, K=8):
//   Yr += Ar.Br - Ai.Bi,  Yi += Ar.Bi + Ai.Br,  each product as
//   hi.hi + hi.lo + lo.hi (3xTF32) and the minus sign via the idesc negate-A bit.
//
// Accuracy: the tensor core's fp32 accumulate truncates, so one TMEM
// accumulator over the whole K stream (~45 000 terms per component at
// config 4) drifts toward zero linearly in K.  The K stream
// is therefore cut into chains of `chain` stages: each chain accumulates
// from zero in TMEM columns [0, 256) and is then folded (round-to-nearest
// fp32 adds) into a running sum at TMEM columns [256, 512) by 4 dedicated
// fold warps; the tile's last chain is added to the running sum on its way
// to y.  The error is then set by the chain length, not by K.
//
// Warp roles (512 threads, 1 CTA / SM, persistent over tiles):
//   warp 0      TMA producer of the B planes
//   warp 1      MMA issuer (one elected thread)
//   warp 2      factor loader: per column, bulk-copies {TDesc, G, U1 rows,
//               U2 rows} of the tile into a 2-deep shared-memory ring
//   warp 3      TMEM allocator
//   warps 4-11  A producers (mode-1 V, mode-2 W, hi/lo split)
//   warps 12-15 chain fold + epilogue (TMEM -> registers -> y)
// Pipelines: A/B stage ring (full: 1 TMA arrive+tx + 8 producer-warp
// arrivals; empty: tcgen05.commit), factor ring (full: bulk-copy tx; empty:
// 8 producer warps), chain (full: commit after the chain's last K step;
// free: 4 fold warps).
#pragma once

#include "tm_common.cuh"
#include "tm_sm100.cuh"

namespace tmb {

constexpr int TC_TI1 = 4, TC_TI2 = 32, TC_ROWS = 128;
constexpr int TC_NST_MAX = 4;   // A/B stages (8 K each)
constexpr int TC_JR = 2;        // factor-ring slots
constexpr int TC_THREADS = 512;
constexpr int TC_NPW = 8;       // producer warps
constexpr int TC_PW0 = 4;       // first producer warp
constexpr int TC_FW0 = 12;      // first fold / epilogue warp
constexpr int TC_NMAX = 128;    // i3 per tile (N per MMA)
constexpr int TC_RMAX = 16;     // rank bound of the tensor-core path
constexpr int TC_A_PLANE = TC_ROWS * 32;     // bytes (128 rows x 8 tf32)
constexpr int TC_A_STAGE = 4 * TC_A_PLANE;   // 16 KB
constexpr uint32_t TC_RUN_COL = 256;         // TMEM column of the running sum

struct TcGeom {
    int64_t ncols;
    int n1, n2, n3, q;
    int nt1, nt2, nt3;
    int nmma;       // N per MMA = i3 per tile (multiple of 16, <= 128)
    int p;          // right-hand sides
    int64_t ntiles;
    int rmax1, rmax2, rmax3;
    int slot_bytes;             // factor slot size (multiple of 128)
    int g_off, u1_off, u2_off;  // byte offsets in a slot (TDesc at 0)
    int b_stage;                // bytes of one B stage (4 planes x nmma x 32)
    int nst;                    // A/B stages in the ring (<= TC_NST_MAX)
    int chain;                  // K stages per TMEM accumulation chain
    int v_stride;               // float4 elements per V buffer
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sm100::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(sm100::smem_u32(bar))
        : "memory");
}

__host__ __device__ inline uint32_t round16(uint32_t b) { return (b + 15u) & ~15u; }

struct TcTile {
    int c, k, i1_0, i2_0, i3_0;
};

// Tile order: (i1, i2) fastest, then i3, component, right-hand side — the
// CTAs resident at one time share (k, i3-block) and so stream the same B
// planes through L2.
__device__ __forceinline__ TcTile tc_tile(const TcGeom& g, int64_t t) {
    const int64_t per_c = int64_t(g.q) * g.nt3 * g.nt2 * g.nt1;
    TcTile r;
    r.c = int(t / per_c);
    int64_t rem = t - int64_t(r.c) * per_c;
    const int64_t per_k = int64_t(g.nt3) * g.nt2 * g.nt1;
    r.k = int(rem / per_k);
    rem -= int64_t(r.k) * per_k;
    const int t3 = int(rem / (int64_t(g.nt2) * g.nt1));
    rem -= int64_t(t3) * g.nt2 * g.nt1;
    const int t2 = int(rem / g.nt1);
    const int t1 = int(rem - int64_t(t2) * g.nt1);
    r.i1_0 = t1 * TC_TI1;
    r.i2_0 = t2 * TC_TI2;
    r.i3_0 = t3 * g.nmma;
    return r;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap bmap, const TDesc* __restrict__ td,
                  const float2* __restrict__ arena, const int* __restrict__ kc, TcGeom g,
                  const float2* __restrict__ x, int64_t ldx, float2* __restrict__ y, int64_t ldy) {
    using namespace sm100;
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    // align to 1024 B by offsetting the shared array itself (keeps the
    // shared address space visible to the compiler: LDS/STS, not generic)
    unsigned char* sm = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
    const int nst = g.nst;
    unsigned char* sA = sm;
    unsigned char* sB = sA + nst * TC_A_STAGE;
    unsigned char* sSlot = sB + nst * g.b_stage;
    float4* sV = reinterpret_cast<float4*>(sSlot + TC_JR * g.slot_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * g.v_stride);
    uint64_t* full = bars;                 // [nst]
    uint64_t* empty = full + TC_NST_MAX;   // [nst]
    uint64_t* ffull = empty + TC_NST_MAX;  // [JR]
    uint64_t* fempty = ffull + TC_JR;      // [JR]
    uint64_t* cfull = fempty + TC_JR;      // 1
    uint64_t* cfree = cfull + 1;           // 1
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfree + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1 + TC_NPW);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < TC_JR; ++s) {
            mbar_init(&ffull[s], 1);
            mbar_init(&fempty[s], TC_NPW);
        }
        mbar_init(cfull, 1);
        mbar_init(cfree, 4);
        fence_mbar_init();
    }
    if (warp == 3) tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) tma_prefetch_desc(&bmap);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ B-plane TMA producer
        if (elect_one()) {
            uint32_t ks = 0;
            const int plane_bytes = g.b_stage / 4;
            for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                const TcTile tl = tc_tile(g, t);
                const int nks = (kc[tl.k] + 7) >> 3;
                for (int kk = 0; kk < nks; ++kk, ++ks) {
                    const uint32_t s = ks % nst, ph = (ks / nst) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], uint32_t(g.b_stage));
                    unsigned char* dst = sB + s * g.b_stage;
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl)
                        tma_load_3d(dst + pl * plane_bytes, &bmap, &full[s], kk * 8, tl.i3_0, pl * g.q + tl.k);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t id_pp = umma_idesc_tf32(TC_ROWS, g.nmma, false, false);
            const uint32_t id_np = umma_idesc_tf32(TC_ROWS, g.nmma, true, false);
            const int plane_b = g.b_stage / 4;
            const uint32_t yr = tmem, yi = tmem + TC_NMAX;
            uint32_t ks = 0, gch = 0;
            for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                const TcTile tl = tc_tile(g, t);
                const int nks = (kc[tl.k] + 7) >> 3;
                int cpos = 0;  // stage position inside the current chain
                for (int kk = 0; kk < nks; ++kk, ++ks) {
                    if (cpos == 0) {
                        mbar_wait(cfree, (gch & 1) ^ 1);  // the previous chain has been folded
                        tc_fence_after();
                    }
                    const uint32_t s = ks % nst, ph = (ks / nst) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + s * TC_A_STAGE);
                    const uint32_t b0 = smem_u32(sB + s * g.b_stage);
                    uint64_t A[4], B[4];
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) {
                        A[pl] = umma_smem_desc(a0 + pl * TC_A_PLANE, 256, 6);
                        B[pl] = umma_smem_desc(b0 + pl * plane_b, 256, 6);
                    }
                    const uint32_t acc = cpos > 0 ? 1u : 0u;
                    // planes: 0 = re hi, 1 = re lo, 2 = im hi, 3 = im lo
                    mma_tf32(yr, A[0], B[0], id_pp, acc);
                    mma_tf32(yr, A[0], B[1], id_pp, 1);
                    mma_tf32(yr, A[1], B[0], id_pp, 1);
                    mma_tf32(yr, A[2], B[2], id_np, 1);
                    mma_tf32(yr, A[2], B[3], id_np, 1);
                    mma_tf32(yr, A[3], B[2], id_np, 1);
                    mma_tf32(yi, A[0], B[2], id_pp, acc);
                    mma_tf32(yi, A[0], B[3], id_pp, 1);
                    mma_tf32(yi, A[1], B[2], id_pp, 1);
                    mma_tf32(yi, A[2], B[0], id_pp, 1);
                    mma_tf32(yi, A[2], B[1], id_pp, 1);
                    mma_tf32(yi, A[3], B[0], id_pp, 1);
                    mma_commit(&empty[s]);
                    if (++cpos == g.chain || kk == nks - 1) {
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
            uint32_t jc = 0;
            for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                const TcTile tl = tc_tile(g, t);
                const TDesc* tdk = td + int64_t(tl.k) * g.ncols;
                for (int64_t j = 0; j < g.ncols; ++j, ++jc) {
                    const uint32_t s = jc % TC_JR, ph = (jc / TC_JR) & 1;
                    mbar_wait(&fempty[s], ph ^ 1);
                    const TDesc d = tdk[j];
                    unsigned char* slot = sSlot + s * g.slot_bytes;
                    const uint32_t bg = round16(uint32_t(d.r1 * d.r2 * d.r3) * 8u);
                    const uint32_t b1 = uint32_t(TC_TI1 * d.r1) * 8u;
                    const uint32_t b2 = uint32_t(TC_TI2 * d.r2) * 8u;
                    mbar_arrive_expect_tx(&ffull[s], uint32_t(sizeof(TDesc)) + bg + b1 + b2);
                    bulk_g2s(slot, tdk + j, uint32_t(sizeof(TDesc)), &ffull[s]);
                    bulk_g2s(slot + g.g_off, arena + d.off_core, bg, &ffull[s]);
                    bulk_g2s(slot + g.u1_off, arena + d.off_u1 + int64_t(tl.i1_0) * d.r1, b1, &ffull[s]);
                    bulk_g2s(slot + g.u2_off, arena + d.off_u2 + int64_t(tl.i2_0) * d.r2, b2, &ffull[s]);
                }
            }
        }
    } else if (warp >= TC_PW0 && warp < TC_FW0) {
        // ------------------------------------------------------ A producers
        const int pt = threadIdx.x - TC_PW0 * 32;  // 0..255
        const int row = pt & (TC_ROWS - 1);
        const int h = pt >> 7;                      // c parity handled by this thread
        const int i1l = row & (TC_TI1 - 1), i2l = row / TC_TI1;
        uint32_t ks = 0, jc = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
            const TcTile tl = tc_tile(g, t);
            const bool row_ok = (tl.i1_0 + i1l < g.n1) && (tl.i2_0 + i2l < g.n2);
            const float2* xc = x + ldx * tl.c;
            uint32_t kpos = 0;  // K slot inside the current stage
            for (int64_t j = 0; j < g.ncols; ++j, ++jc) {
                const uint32_t s = jc % TC_JR, ph = (jc / TC_JR) & 1;
                const float2 xj = xc[j];
                mbar_wait(&ffull[s], ph);
                const unsigned char* slot = sSlot + s * g.slot_bytes;
                const TDesc d = *reinterpret_cast<const TDesc*>(slot);
                const float2* G = reinterpret_cast<const float2*>(slot + g.g_off);
                const float2* U1 = reinterpret_cast<const float2*>(slot + g.u1_off);
                const float2* U2 = reinterpret_cast<const float2*>(slot + g.u2_off);
                const int r1 = d.r1, r2 = d.r2, r3 = d.r3;
                float4* V = sV + (jc & 1) * g.v_stride;
                // mode 1 (+ x_j): V[(b + r2 c) * 4 + i1l] = x_j sum_a U1[i1l][a] G[a + r1 (b + r2 c)],
                // stored as (vr, vi, -vi, vr) for the FFMA2 mode-2 product
                const int nv = TC_TI1 * r2 * r3;
                for (int e = pt; e < nv; e += TC_NPW * 32) {
                    const int il = e & (TC_TI1 - 1), bc = e >> 2;
                    const float2* gp = G + r1 * bc;
                    const float2* up = U1 + il * r1;
                    float2 acc = make_float2(0.f, 0.f);
                    for (int a = 0; a < r1; ++a) cfma(acc, up[a], gp[a]);
                    const float2 v = cmul(acc, xj);
                    V[e] = make_float4(v.x, v.y, -v.y, v.x);
                }
                // my row of U2 into registers
                float2 u2[TC_RMAX];
#pragma unroll
                for (int b = 0; b < TC_RMAX; ++b) u2[b] = b < r2 ? U2[i2l * r2 + b] : make_float2(0.f, 0.f);
                named_bar_sync(1, TC_NPW * 32);  // V complete; the slot is no longer read
                __syncwarp();
                if (lane == 0) mbar_arrive(&fempty[s]);
                // mode 2 for c = 2u + h: W[row, c] = sum_b V[i1l, b, c] U2[i2l, b]
                uint64_t w[TC_RMAX / 2];
#pragma unroll
                for (int u = 0; u < TC_RMAX / 2; ++u) {
                    const int c = 2 * u + h;
                    w[u] = 0;
                    if (c < r3) {
                        const float4* vp = V + r2 * c * 4 + i1l;
#pragma unroll
                        for (int b = 0; b < TC_RMAX; ++b)
                            if (b < r2) cfma2(w[u], vp[b * 4], u2[b]);
                    }
                    if (!row_ok) w[u] = 0;
                }
                // scatter into the K stream (uniform stage bookkeeping)
#pragma unroll
                for (int c = 0; c < TC_RMAX; ++c) {
                    if (c < r3) {
                        const uint32_t st = ks % nst;
                        if (kpos == 0) mbar_wait(&empty[st], ((ks / nst) & 1) ^ 1);
                        if ((c & 1) == h) {
                            const float2 wv = f2_unpack(w[c >> 1]);
                            const float hr = __uint_as_float(__float_as_uint(wv.x) & 0xFFFFE000u);
                            const float hi = __uint_as_float(__float_as_uint(wv.y) & 0xFFFFE000u);
                            unsigned char* a = sA + st * TC_A_STAGE + sw_offset(row, kpos, 32);
                            *reinterpret_cast<float*>(a) = hr;
                            *reinterpret_cast<float*>(a + TC_A_PLANE) = wv.x - hr;
                            *reinterpret_cast<float*>(a + 2 * TC_A_PLANE) = hi;
                            *reinterpret_cast<float*>(a + 3 * TC_A_PLANE) = wv.y - hi;
                        }
                        if (++kpos == 8) {
                            fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&full[st]);
                            kpos = 0;
                            ++ks;
                        }
                    }
                }
            }
            if (kpos != 0) {  // zero the tail of the last stage and close it
                const uint32_t st = ks % nst;
                if (h == 0)
                    for (uint32_t kq = kpos; kq < 8; ++kq) {
                        unsigned char* a = sA + st * TC_A_STAGE + sw_offset(row, kq, 32);
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) *reinterpret_cast<float*>(a + pl * TC_A_PLANE) = 0.f;
                    }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[st]);
                kpos = 0;
                ++ks;
            }
        }
    } else if (warp >= TC_FW0) {
        // ------------------------------------------ chain fold + epilogue
        const int quarter = warp & 3;             // TMEM lane quarter
        const int erow = quarter * 32 + lane;     // TMEM lane = tile row
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const uint32_t tC = tmem + lane_addr, tR = tmem + lane_addr + TC_RUN_COL;
        const int64_t nv3 = int64_t(g.n1) * g.n2 * g.n3;
        uint32_t gch = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
            const TcTile tl = tc_tile(g, t);
            const int nks = (kc[tl.k] + 7) >> 3;
            const int nch = (nks + g.chain - 1) / g.chain;
            const int ei1 = tl.i1_0 + (erow & (TC_TI1 - 1)), ei2 = tl.i2_0 + erow / TC_TI1;
            const bool eok = ei1 < g.n1 && ei2 < g.n2;
            float2* yp = y + ldy * tl.c + int64_t(tl.k) * nv3 + ei1 + int64_t(g.n1) * ei2;
            const int64_t pl = int64_t(g.n1) * g.n2;
            for (int ch = 0; ch < nch; ++ch, ++gch) {
                mbar_wait(cfull, gch & 1);
                tc_fence_after();
                const bool last = ch == nch - 1;
                for (int cb = 0; cb < g.nmma; cb += 16) {
                    uint32_t cr[16], ci[16];
                    tmem_ld16(tC + uint32_t(cb), cr);
                    tmem_ld16(tC + uint32_t(TC_NMAX + cb), ci);
                    if (ch > 0) {
                        uint32_t rr[16], ri[16];
                        tmem_ld16(tR + uint32_t(cb), rr);
                        tmem_ld16(tR + uint32_t(TC_NMAX + cb), ri);
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
                        tmem_st16(tR + uint32_t(cb), cr);
                        tmem_st16(tR + uint32_t(TC_NMAX + cb), ci);
                    } else if (eok) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int i3 = tl.i3_0 + cb + i;
                            if (i3 < g.n3)
                                yp[pl * i3] = make_float2(__uint_as_float(cr[i]), __uint_as_float(ci[i]));
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

// ------------------------------------------------- store-side B planes (K6')
// planes[p][k][i3][K], K = kofs[k][j] + r:  p = 0 re hi, 1 re lo, 2 im hi, 3 im lo.
__global__ void build_bplanes_kernel(const TDesc* __restrict__ td, const float2* __restrict__ arena,
                                     const int* __restrict__ kofs, int64_t ncols, int q, int n3, int64_t kpad,
                                     float* __restrict__ planes) {
    const int64_t t = blockIdx.x;  // tensor index k*ncols + j
    const int k = int(t / ncols);
    const TDesc d = td[t];
    const int64_t k0 = kofs[t];
    const int64_t plane = int64_t(q) * n3 * kpad;
    for (int e = threadIdx.x; e < n3 * d.r3; e += blockDim.x) {
        const int i3 = e / d.r3, r = e - i3 * d.r3;
        const float2 u = arena[d.off_u3 + e];
        const float rh = sm100::tf32_round(u.x), ih = sm100::tf32_round(u.y);
        const int64_t o = (int64_t(k) * n3 + i3) * kpad + k0 + r;
        planes[o] = rh;
        planes[plane + o] = sm100::tf32_round(u.x - rh);
        planes[2 * plane + o] = ih;
        planes[3 * plane + o] = sm100::tf32_round(u.y - ih);
    }
}

}  // namespace tmb
