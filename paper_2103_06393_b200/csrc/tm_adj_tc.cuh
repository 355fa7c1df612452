// Tensor-core (tcgen05, kind::f16, 2-term fp16 split) adjoint kernel, complex64.
//
// The reference's stacked_adjoint (src/matvec.cpp:67-102) forms, per column
// j and component k, z_j += vec(T_jk)^H Phi_k.  With T_jk[row, i3] =
// sum_c W_j[row, c] U3_j[i3, c] (row = (i1, i2), W as in the forward) this is
//
//   z_j = sum_rows sum_c conj(W_j[row, c]) Q[row, (j, c)],
//   Q[row, (j, c)] = sum_i3 Phi[row, i3] conj(U3_j[i3, c]),
//
// i.e. one GEMM per 128-row tile, M = rows, K = i3 (all n3), N = the (j, c)
// slots of component k in chunks of 128 (whole columns per chunk, zero
// padded), followed by a per-column contraction with conj(W).  The complex
// product runs as one real GEMM of width 256:
//   [Qi | Qr] += Phir . [-U3i | U3r] + Phii . [U3r | U3i]
// with the B planes staged [-U3i][U3r][U3i] (hi and lo, i3-contiguous
// chunk-aligned copy built once per store) and the A planes the split of
// the Phi tile (built per call by adj_split_phi_kernel), both as scaled
// 2-term fp16 splits on tcgen05.mma.kind::f16 (K = 16 per MMA: half the
// MMAs and half the operand bytes of 3xTF32 at the same 22-bit operand
// precision; products hi.hi + hi.lo + lo.hi accumulate in fp32).  Both
// operands arrive by TMA; Q is accumulated in TMEM (two 256-column buffers,
// ping-pong over chunks).
//
// Warp roles (512 threads, 1 CTA / SM, persistent over row tiles):
//   warp 0      TMA producer of the A (Phi) and B (U3) planes
//   warp 1      MMA issuer
//   warp 2      factor loader (TcDesc, V rows, U2 rows per column)
//   warp 3      TMEM allocator
//   warps 4-11  consumers: per column, W = V x_2 U2 for the tile rows
//               (FFMA2), Q from TMEM, conj(W) . Q, warp-shuffle reduction
//               over the 32 rows of the warp, fixed-order sum over the 8
//               warps -> one partial z_j per (tile, component)
// A second kernel (adj_reduce_kernel) sums the partials in a fixed order,
// so results are bitwise reproducible.
#pragma once

#include <cuda_fp16.h>

#include "tm_common.cuh"
#include "tm_kernels_tc.cuh"
#include "tm_sm100.cuh"

namespace tmb {

// fp16 operand scaling of the adjoint GEMM.  Both operands are stored as a
// 2-term fp16 split (hi = fp16(v), lo = fp16(v - hi): 22 significant bits,
// the class of the 3xTF32 split) scaled by powers of two so their values sit
// inside fp16's normal range: U3 (orthonormal columns, |u| <= 1) by 2^12,
// Phi by 2^(14 - e) with max|Phi| < 2^e (measured per call).  Q in TMEM is
// then scaled by both factors, undone exactly on the fp32 partial sums.
constexpr float AJ_U3_SCALE = 4096.f;
__host__ __device__ inline float aj_phi_scale(float amax) {
    if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
    int e = 0;
    frexpf(amax, &e);  // amax < 2^e
    e = e < -100 ? -100 : (e > 100 ? 100 : e);
    return ldexpf(1.f, 14 - e);
}

constexpr int AJ_NST = 4;        // A/B stages (16 i3 each)
constexpr int AJ_NST2 = 5;       // stages of the CTA-pair kernel (half-size B stage)
constexpr int AJ_CH = 128;       // (j, c) slots per chunk
constexpr int AJ_APLANES = 4;    // Phi planes: re hi, re lo, im hi, im lo
constexpr int AJ_A_PLANE = TC_ROWS * 32;
constexpr int AJ_A_STAGE = AJ_APLANES * AJ_A_PLANE;       // 16 KB
constexpr int AJ_B_PLANE = AJ_CH * 32;
constexpr int AJ_B_STAGE = TC_BPLANES * AJ_B_PLANE;       // 24 KB
constexpr int AJ_MAXCOLS = 128;  // columns per chunk (r3 >= 1)
constexpr int AJ_NPW = 8;        // consumer warps (4 i1 rows x 2 c parities)
constexpr int AJ_NH = AJ_NPW / TC_TI1;
constexpr int AJ_THREADS = (TC_PW0 + AJ_NPW) * 32;

struct AjGeom {
    int64_t ncols;
    int n1, n2, n3, q;
    int nt1, nt2;
    int p;
    int64_t nrt;     // row tiles per component
    int64_t ntiles;  // p * q * nrt
    int nks;         // K steps (16 i3 each) per chunk
    int rmax2, rmax3;
    int slot_bytes, u2_off;
    int maxch;       // chunk stride of the chunk-start table
    int debug;       // diagnostics (TMB_TC_DEBUG & 4): consumers skip the mode-2 product
    int pair;        // 1: CTA-pair kernel (cta_group::2, M = 256 over two row tiles); tiles count pairs
    int split;       // work items per tile in this launch (chunk ranges; > 1 only for a final partial wave)
    int64_t tile0;   // first tile of this launch: item t is tile tile0 + t / split, part t % split
    int64_t t_begin, t_end;  // item range of this launch
};

struct AjTile {
    int c, k, i1_0, i2_0;
    int64_t rt;  // row tile inside the component
    int part;    // chunk range part (of g.split)
};

// Chunk range [n0, n1) of a work item over a tile of nc chunks.
__device__ __forceinline__ void aj_chunks(const AjGeom& g, const AjTile& tl, int nc, int& n0, int& n1) {
    n0 = int(int64_t(nc) * tl.part / g.split);
    n1 = int(int64_t(nc) * (tl.part + 1) / g.split);
}

__device__ __forceinline__ AjTile aj_tile(const AjGeom& g, int64_t item, uint32_t rank = 0) {
    AjTile r;
    const int64_t t = g.tile0 + item / g.split;
    r.part = int(item % g.split);
    const int64_t tpk = g.nrt >> g.pair;  // (pair) tiles per component
    const int64_t per_c = int64_t(g.q) * tpk;
    r.c = int(t / per_c);
    int64_t rem = t - int64_t(r.c) * per_c;
    r.k = int(rem / tpk);
    r.rt = ((rem - int64_t(r.k) * tpk) << g.pair) + rank;  // a pair tile = row tiles 2 pt, 2 pt + 1
    // i2 block fastest: the resident CTAs share the V rows of one i1 block
    const int t1 = int(r.rt / g.nt2), t2 = int(r.rt - int64_t(t1) * g.nt2);
    r.i1_0 = t1 * TC_TI1;
    r.i2_0 = t2 * TC_TI2;
    return r;
}

// One column of a chunk for the consumer thread (row = lane + 32 il, c parity
// h): W = V x_2 U2 (no x_j in the adjoint), Q[row, soff + c] from TMEM, and
// the partial sum_c conj(W) Q of this thread's row.
template <int NU>
__device__ __forceinline__ float2 aj_consume_column(const float2* __restrict__ V, const float2* __restrict__ U2,
                                                    int r2, int ld2, int r3, int h, int lane, uint32_t qaddr,
                                                    uint64_t* fempty_s) {
    using namespace sm100;
    uint64_t w[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) w[u] = 0;
    // V[(c + r3 b) * 4 + il], c = NH u + h.  The loop computes all NU values
    // unpredicated: for c = r3 (odd r3, h = 1) the load reads the next V entry
    // (at most 4 float2 past the V block, inside the slot) and the product is
    // dropped below.
    const float2* vp = V + 4 * h;
    const float2* up = U2 + lane * ld2;
    const int vstep = 4 * r3;
#pragma unroll 2
    for (int b = 0; b < r2; ++b) {
        const float2 ub = up[b];
#pragma unroll
        for (int u = 0; u < NU; ++u) cfma2v(w[u], vp[4 * AJ_NH * u], ub);
        vp += vstep;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(fempty_s);
    // Q columns: Qi at qaddr + s, Qr at qaddr + AJ_CH + s
    uint32_t qi[NU], qr[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        // (a slot past this column's last c reads slot 0 and is ignored: it
        // may lie past the end of the TMEM allocation)
        const uint32_t s = (u < NU - 1 || AJ_NH * u + h < r3) ? uint32_t(AJ_NH * u + h) : 0u;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(qi[u]) : "r"(qaddr + s));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(qr[u]) : "r"(qaddr + AJ_CH + s));
    }
    tmem_ld_wait();
    float ar = 0.f, ai = 0.f;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        if (u < NU - 1 || AJ_NH * u + h < r3) {
            const float2 wv = f2_unpack(w[u]);
            const float qre = __uint_as_float(qr[u]), qim = __uint_as_float(qi[u]);
            // conj(W) Q = (Wr Qr + Wi Qi) + i (Wr Qi - Wi Qr)
            ar = fmaf(wv.x, qre, fmaf(wv.y, qim, ar));
            ai = fmaf(wv.x, qim, fmaf(-wv.y, qre, ai));
        }
    }
    return make_float2(ar, ai);
}

// NSTX: A/B stage count override (0 = AJ_NST / AJ_NST2); 2 for stores whose
// rank-(r2, r3) factor slots leave no room for the default ring.
// BIG: stores with r3 > 16 (up to TC_RMAX = 32), a separate instantiation so
// the r3 <= 16 kernels keep their register budget.
template <bool PAIR, int NSTX = 0, bool BIG = false>
__global__ void __launch_bounds__(AJ_THREADS, 1)
    adj_tc_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                  const TcDesc* __restrict__ tcd, const float2* __restrict__ varena,
                  const float2* __restrict__ u2arena, const int* __restrict__ nch, const int* __restrict__ cstart,
                  AjGeom g, const float* __restrict__ phimax, float2* __restrict__ part) {
    using namespace sm100;
    extern __shared__ __align__(1024) unsigned char aj_smem_raw[];
    unsigned char* sm = aj_smem_raw + ((1024u - (smem_u32(aj_smem_raw) & 1023u)) & 1023u);
    // PAIR: the M = 256 MMA takes B rows [0, 128) of each N = 256 window from
    // the even CTA and [128, 256) from the odd one: the even CTA holds planes
    // (-U3i, U3r), the odd one (U3r, U3i), hi and lo — 4 planes per stage.
    constexpr int NST = NSTX ? NSTX : (PAIR ? AJ_NST2 : AJ_NST);
    constexpr int BSTAGE = PAIR ? 4 * AJ_B_PLANE : AJ_B_STAGE;
    unsigned char* sA = sm;
    unsigned char* sB = sA + NST * AJ_A_STAGE;
    unsigned char* sSlot = sB + NST * BSTAGE;
    float2* red = reinterpret_cast<float2*>(sSlot + TC_JR * g.slot_bytes);  // [2][AJ_MAXCOLS][8]
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * AJ_MAXCOLS * AJ_NPW);
    uint64_t* full = bars;                // [NST]
    uint64_t* empty = full + NST;         // [NST]
    uint64_t* ffull = empty + NST;        // [JR]
    uint64_t* fempty = ffull + TC_JR;     // [JR]
    uint64_t* qfull = fempty + TC_JR;     // [2]
    uint64_t* qfree = qfull + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qfree + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const int64_t tstart = g.t_begin + (PAIR ? (blockIdx.x >> 1) : blockIdx.x);
    const int64_t tstep = PAIR ? (gridDim.x >> 1) : gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < TC_JR; ++s) {
            mbar_init(&ffull[s], 1);
            mbar_init(&fempty[s], AJ_NPW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&qfull[s], 1);
            mbar_init(&qfree[s], AJ_NPW * (PAIR ? 2 : 1));  // PAIR: the peer's consumers too
        }
        fence_mbar_init();
    }
    if (warp == 3) {
        if (PAIR)
            tmem_alloc_pair(tmem_slot, 512);
        else
            tmem_alloc(tmem_slot, 512);
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&amap);
        tma_prefetch_desc(&bmap);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------- TMA producer
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const AjTile tl = aj_tile(g, t, rank);
                int n0, n1;
                aj_chunks(g, tl, nch[tl.k], n0, n1);
                const int arow = int(tl.rt * TC_ROWS);
                for (int n = n0; n < n1; ++n) {
                    for (int kk = 0; kk < g.nks; ++kk) {
                        mbar_wait_backoff(&empty[s], ph ^ 1, TC_BACKOFF_ADJ);
                        unsigned char* da = sA + s * AJ_A_STAGE;
                        unsigned char* db = sB + s * BSTAGE;
                        if (PAIR) {
                            // both CTAs' bytes complete on the even CTA's barrier
                            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2u * uint32_t(AJ_A_STAGE + BSTAGE));
                            const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
#pragma unroll
                            for (int pl = 0; pl < AJ_APLANES; ++pl)
                                tma_load_3d_pair(da + pl * AJ_A_PLANE, &amap, fb, kk * 16, arow,
                                                 (pl * g.p + tl.c) * g.q + tl.k);
                            // smem B slots (W1 hi, W2 hi, W1 lo, W2 lo) <- HBM planes rank + {0, 1} (+3 for lo)
#pragma unroll
                            for (int sl = 0; sl < 4; ++sl)
                                tma_load_3d_pair(db + sl * AJ_B_PLANE, &bmap, fb, kk * 16, n * AJ_CH,
                                                 (int(rank) + (sl & 1) + 3 * (sl >> 1)) * g.q + tl.k);
                        } else {
                            mbar_arrive_expect_tx(&full[s], uint32_t(AJ_A_STAGE + AJ_B_STAGE));
#pragma unroll
                            for (int pl = 0; pl < AJ_APLANES; ++pl)
                                tma_load_3d(da + pl * AJ_A_PLANE, &amap, &full[s], kk * 16, arow,
                                            (pl * g.p + tl.c) * g.q + tl.k);
#pragma unroll
                            for (int pl = 0; pl < TC_BPLANES; ++pl)
                                tma_load_3d(db + pl * AJ_B_PLANE, &bmap, &full[s], kk * 16, n * AJ_CH,
                                            pl * g.q + tl.k);
                        }
                        if (++s == NST) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        if ((!PAIR || rank == 0) && elect_one()) {
            const uint32_t idesc = umma_idesc_f16(TC_ROWS * (PAIR ? 2 : 1), 2 * AJ_CH, false, false);
            uint32_t s = 0, ph = 0, nq = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const AjTile tl = aj_tile(g, t, rank);
                int n0, n1;
                aj_chunks(g, tl, nch[tl.k], n0, n1);
                for (int n = n0; n < n1; ++n, ++nq) {
                    const uint32_t qb = nq & 1, qph = (nq >> 1) & 1;
                    mbar_wait(&qfree[qb], qph ^ 1);  // consumers are done with this buffer
                    tc_fence_after();
                    const uint32_t qd = tmem + qb * 256u;
                    for (int kk = 0; kk < g.nks; ++kk) {
                        mbar_wait(&full[s], ph);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + s * AJ_A_STAGE);
                        const uint32_t b0 = smem_u32(sB + s * BSTAGE);
                        uint64_t A[4];
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) A[pl] = umma_smem_desc(a0 + pl * AJ_A_PLANE, 256, 6);
                        // B windows: [-U3i|U3r] at plane 0 / 3 (hi / lo), [U3r|U3i] at plane 1 / 4
                        // (PAIR: smem slots 0 / 2 and 1 / 3 of each CTA, half a window each)
                        const uint64_t B2h = umma_smem_desc(b0 + 0 * AJ_B_PLANE, 256, 6);
                        const uint64_t B1h = umma_smem_desc(b0 + 1 * AJ_B_PLANE, 256, 6);
                        const uint64_t B2l = umma_smem_desc(b0 + (PAIR ? 2 : 3) * AJ_B_PLANE, 256, 6);
                        const uint64_t B1l = umma_smem_desc(b0 + (PAIR ? 3 : 4) * AJ_B_PLANE, 256, 6);
                        const uint32_t acc = kk > 0 ? 1u : 0u;
                        // [Qi | Qr] += Phir . [-U3i | U3r] + Phii . [U3r | U3i]
#define MMA(...) (PAIR ? mma_f16_pair(__VA_ARGS__) : mma_f16(__VA_ARGS__))
#define COMMIT(b) (PAIR ? mma_commit_pair(b) : mma_commit(b))
                        MMA(qd, A[0], B2h, idesc, acc);
                        MMA(qd, A[0], B2l, idesc, 1);
                        MMA(qd, A[1], B2h, idesc, 1);
                        MMA(qd, A[2], B1h, idesc, 1);
                        MMA(qd, A[2], B1l, idesc, 1);
                        MMA(qd, A[3], B1h, idesc, 1);
                        COMMIT(&empty[s]);
                        if (++s == NST) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                    COMMIT(&qfull[qb]);
#undef MMA
#undef COMMIT
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---------------------------------------------------- factor loader
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const AjTile tl = aj_tile(g, t, rank);
                const TcDesc* tdk = tcd + int64_t(tl.k) * g.ncols;
                int n0, n1;
                aj_chunks(g, tl, nch[tl.k], n0, n1);
                const int* cs = cstart + int64_t(tl.k) * (g.maxch + 1);
                for (int64_t j = cs[n0]; j < cs[n1]; ++j) {
                    mbar_wait_backoff(&fempty[s], ph ^ 1, TC_BACKOFF_ADJ);
                    const TcDesc d = tdk[j];
                    unsigned char* slot = sSlot + s * g.slot_bytes;
                    const uint32_t r23 = uint32_t(d.r2 * d.r3);
                    const uint32_t ld2 = uint32_t(d.r2 | 1);
                    const uint32_t bv = round16(uint32_t(TC_TI1) * r23 * 8u);
                    const uint32_t b2 = uint32_t(TC_TI2) * ld2 * 8u;
                    mbar_arrive_expect_tx(&ffull[s], uint32_t(sizeof(TcDesc)) + bv + b2);
                    bulk_g2s(slot, tdk + j, uint32_t(sizeof(TcDesc)), &ffull[s]);
                    bulk_g2s(slot + TC_SLOT_V, varena + d.off_v + int64_t(tl.i1_0) * r23, bv, &ffull[s]);
                    bulk_g2s(slot + g.u2_off, u2arena + d.off_u2 + int64_t(tl.i2_0) * ld2, b2, &ffull[s]);
                    if (++s == TC_JR) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp >= TC_PW0 && warp < TC_PW0 + AJ_NPW) {
        // -------------------------------------------------------- consumers
        const int pw = warp - TC_PW0;
        const int i1l = pw & (TC_TI1 - 1), h = pw / TC_TI1;
        const int ctid = threadIdx.x - TC_PW0 * 32;  // 0..255
        const uint32_t lane_addr = uint32_t(i1l * 32) << 16;
        uint32_t fs = 0, fph = 0, nq = 0;
        for (int64_t t = tstart; t < g.t_end; t += tstep) {
            const AjTile tl = aj_tile(g, t, rank);
            int n0, n1;
            aj_chunks(g, tl, nch[tl.k], n0, n1);
            const int* cs = cstart + int64_t(tl.k) * (g.maxch + 1);
            // exact power of two: undoes the (rhs, component) Phi scale and the U3 scale
            const float inv_scale = 1.f / (aj_phi_scale(phimax[int64_t(tl.c) * g.q + tl.k]) * AJ_U3_SCALE);
            for (int n = n0; n < n1; ++n, ++nq) {
                const uint32_t qb = nq & 1, qph = (nq >> 1) & 1;
                const int j0 = cs[n], j1 = cs[n + 1];
                float2* rb = red + (nq & 1) * AJ_MAXCOLS * AJ_NPW;
                mbar_wait(&qfull[qb], qph);
                tc_fence_after();
                const uint32_t qbase = tmem + lane_addr + qb * 256u;
                for (int j = j0; j < j1; ++j) {
                    mbar_wait(&ffull[fs], fph);
                    const unsigned char* slot = sSlot + fs * g.slot_bytes;
                    const TcDesc* dd = reinterpret_cast<const TcDesc*>(slot);
                    const int r2 = dd->r2, r3 = dd->r3, soff = dd->pad0;
                    const float2* V = reinterpret_cast<const float2*>(slot + TC_SLOT_V) + i1l;
                    const float2* U2 = reinterpret_cast<const float2*>(slot + g.u2_off);
                    float2 a;
#define AJ_COL(NU) \
    a = aj_consume_column<NU>(V, U2, (g.debug & 4) ? 0 : r2, r2 | 1, r3, h, lane, qbase + uint32_t(soff), &fempty[fs])
                    if constexpr (BIG) {
                        switch ((r3 + AJ_NH - 1) / AJ_NH) {
                            case 1: AJ_COL(1); break;
                            case 2: AJ_COL(2); break;
                            case 3: AJ_COL(3); break;
                            case 4: AJ_COL(4); break;
                            case 5: AJ_COL(5); break;
                            case 6: AJ_COL(6); break;
                            case 7: AJ_COL(7); break;
                            case 8: AJ_COL(8); break;
                            case 9: AJ_COL(9); break;
                            case 10: AJ_COL(10); break;
                            case 11: AJ_COL(11); break;
                            case 12: AJ_COL(12); break;
                            case 13: AJ_COL(13); break;
                            case 14: AJ_COL(14); break;
                            case 15: AJ_COL(15); break;
                            default: AJ_COL(16); break;
                        }
                    } else {
                        switch ((r3 + AJ_NH - 1) / AJ_NH) {
                            case 1: AJ_COL(1); break;
                            case 2: AJ_COL(2); break;
                            case 3: AJ_COL(3); break;
                            case 4: AJ_COL(4); break;
                            case 5: AJ_COL(5); break;
                            case 6: AJ_COL(6); break;
                            case 7: AJ_COL(7); break;
                            default: AJ_COL(8); break;
                        }
                    }
#undef AJ_COL
                    if (++fs == TC_JR) {
                        fs = 0;
                        fph ^= 1;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
                        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
                    }
                    if (lane == 0) rb[(j - j0) * AJ_NPW + pw] = a;
                }
                // Q buffer no longer read by this warp
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_cluster(mapa_shared(smem_u32(&qfree[qb]), 0));
                    else
                        mbar_arrive(&qfree[qb]);
                }
                named_bar_sync(1, AJ_NPW * 32);  // all partials of the chunk are in rb
                for (int jj = ctid; jj < j1 - j0; jj += AJ_NPW * 32) {
                    float sx = 0.f, sy = 0.f;
#pragma unroll
                    for (int w = 0; w < AJ_NPW; ++w) {
                        sx += rb[jj * AJ_NPW + w].x;
                        sy += rb[jj * AJ_NPW + w].y;
                    }
                    part[((int64_t(tl.c) * g.ncols + j0 + jj) * g.q + tl.k) * g.nrt + tl.rt] =
                        make_float2(sx * inv_scale, sy * inv_scale);
                }
                // rb (this parity) is rewritten two chunks later, after the
                // next chunk's named barrier: no second barrier needed
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 3) {
        if (PAIR)
            tmem_dealloc_pair(tmem, 512);
        else
            tmem_dealloc(tmem, 512);
    }
}

// max |Re|, |Im| of each (right-hand side, component) block of Phi — the
// fp16 scale of its planes — by an order-free atomicMax on the bit
// patterns of non-negative floats.  blockIdx.y = block index - b0.
__global__ void absmax_kernel(const float2* __restrict__ phi, int64_t ldphi, int64_t nv, int q, int64_t b0,
                              float* __restrict__ out) {
    const int64_t b = b0 + blockIdx.y;
    const int64_t c = b / q, k = b - c * q;
    const float2* src = phi + ldphi * c + k * nv;
    float m = 0.f;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nv; e += int64_t(gridDim.x) * blockDim.x) {
        const float2 v = src[e];
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(out + b), __float_as_uint(m));
}

// max |Phi| of component k for every right-hand side c of the pass (out[c q +
// k], the per-component form of absmax_kernel used when Phi arrives from the
// host component by component).
__global__ void absmax_comp_kernel(const float2* __restrict__ phi, int64_t ldphi, int64_t nv, int q, int k,
                                   float* __restrict__ out) {
    const int64_t c = blockIdx.y;
    const float2* src = phi + ldphi * c + int64_t(k) * nv;
    float m = 0.f;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nv; e += int64_t(gridDim.x) * blockDim.x) {
        const float2 v = src[e];
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(out + c * q + k), __float_as_uint(m));
}

// Phi (c64, [c][k n_v + v]) -> scaled 2-term fp16 planes [pl][c][k][row-tile
// order][n3p] (n3p = n3 rounded up to 8 for the TMA row pitch), pl = re hi,
// re lo, im hi, im lo; tile rows are (i2 + 32 i1) of the (TI1 x TI2) row
// tiles, rows outside the grid are zero.  One block per (row tile, 32 i3,
// k, c), transposed through shared memory so both the read
// (voxel-contiguous) and the write (i3-contiguous) are coalesced.
__global__ void __launch_bounds__(256) adj_split_phi_kernel(const float2* __restrict__ phi, int64_t ldphi, int n1,
                                                            int n2, int n3, int n3p, int q, int p, int nt2,
                                                            int64_t nrt, int64_t b0, const float* __restrict__ phimax,
                                                            __half* __restrict__ planes) {
    __shared__ float2 tile[TC_ROWS][33];
    const int64_t rt = blockIdx.x;
    const int i3b = blockIdx.y * 32;
    const int64_t b = b0 + blockIdx.z;  // (rhs, component) block
    const int k = int(b % q), c = int(b / q);
    const int t1 = int(rt / nt2), t2 = int(rt - int64_t(t1) * nt2);  // as aj_tile
    const int64_t nv = int64_t(n1) * n2 * n3;
    const float2* src = phi + ldphi * c + int64_t(k) * nv;
    const float sc = aj_phi_scale(phimax[b]);
    for (int e = threadIdx.x; e < TC_ROWS * 32; e += 256) {
        const int vr = e & (TC_ROWS - 1), i3l = e >> 7;
        const int i1l = vr & 3, i2l = vr >> 2;
        const int i1 = t1 * TC_TI1 + i1l, i2 = t2 * TC_TI2 + i2l, i3 = i3b + i3l;
        float2 v = make_float2(0.f, 0.f);
        if (i1 < n1 && i2 < n2 && i3 < n3) v = src[i1 + int64_t(n1) * (i2 + int64_t(n2) * i3)];
        tile[i2l + 32 * i1l][i3l] = make_float2(v.x * sc, v.y * sc);
    }
    __syncthreads();
    const int64_t R = nrt * TC_ROWS;
    const int64_t plane = int64_t(p) * q * R * n3p;
    for (int e = threadIdx.x; e < TC_ROWS * 32; e += 256) {
        const int i3l = e & 31, row = e >> 5;
        const int i3 = i3b + i3l;
        if (i3 >= n3p) continue;
        const float2 v = tile[row][i3l];
        const __half rh = __float2half_rn(v.x), ih = __float2half_rn(v.y);
        const int64_t o = ((int64_t(c) * q + k) * R + rt * TC_ROWS + row) * n3p + i3;
        planes[o] = rh;
        planes[plane + o] = __float2half_rn(v.x - __half2float(rh));
        planes[2 * plane + o] = ih;
        planes[3 * plane + o] = __float2half_rn(v.y - __half2float(ih));
    }
}

// U3 planes for the adjoint: [pl][k][slot][n3p] fp16 (i3-contiguous), slot
// = chunk * 128 + offset of the (j, c) pair inside its chunk; values
// normalised by 2^-e3 (factor_scale_kernel) and scaled by AJ_U3_SCALE, 2-term fp16 split, in the 6-plane order
// (-U3i, U3r, U3i hi; the same lo): the windows [-U3i|U3r] and [U3r|U3i].
__global__ void build_adj_bplanes_kernel(const TDesc* __restrict__ td, const float2* __restrict__ arena,
                                         const int* __restrict__ aslot, int64_t ncols, int q, int n3, int n3p,
                                         int64_t nslots, const TcDesc* __restrict__ tcd, __half* __restrict__ planes) {
    const int64_t t = blockIdx.x;
    const int k = int(t / ncols);
    const TDesc d = td[t];
    const int sc = -fexp_e3(tcd[t].fexp);  // normalised U3 (|u| <= 1), exact
    const int64_t s0 = aslot[t];
    const int64_t plane = int64_t(q) * nslots * n3p;
    for (int e = threadIdx.x; e < n3 * d.r3; e += blockDim.x) {
        const int i3 = e / d.r3, r = e - i3 * d.r3;
        const float2 u0 = arena[d.off_u3 + e];
        const float2 u = make_float2(ldexpf(u0.x, sc) * AJ_U3_SCALE, ldexpf(u0.y, sc) * AJ_U3_SCALE);
        const __half rh = __float2half_rn(u.x), ih = __float2half_rn(u.y);
        const __half rl = __float2half_rn(u.x - __half2float(rh)), il = __float2half_rn(u.y - __half2float(ih));
        const int64_t o = (int64_t(k) * nslots + s0 + r) * n3p + i3;
        planes[o] = __hneg(ih);
        planes[plane + o] = rh;
        planes[2 * plane + o] = ih;
        planes[3 * plane + o] = __hneg(il);
        planes[4 * plane + o] = rl;
        planes[5 * plane + o] = il;
    }
}

// ------------------------------------------------ adjoint as one GEMM (W arena)
// For stores with the transposed W arena (build_warena): G = conj(W)^T Phi on
// the forward arena kernel (fwd_tc_kernel<..., WA, ADJ>), then z from G here.
//
// Phi as the GEMM's K-major B operand: [plane][k][n = i3 p + c][row] fp16,
// rows tile-major (the arena's order) and contiguous, scaled per component by
// fp16_scale(max over the component's right-hand sides of max(|re|, |im|))
// (absmax_kernel's per-(rhs, component) maxima), split hi / lo.  One block per
// (row tile, n, k); thread t -> (i1 = i1_0 + t % 4, i2 = i2_0 + t / 4), so four
// threads read 32 contiguous bytes of Phi.
__global__ void adjg_split_phi_kernel(const float2* __restrict__ phi, int64_t ldphi, int n1, int n2, int n3, int p,
                                      int q, int nt2, int64_t R, int64_t nt, const float* __restrict__ phimax,
                                      __half* __restrict__ planes, int k0) {
    using namespace sm100;
    const int tile = int(blockIdx.x);
    const int64_t n = blockIdx.y;
    const int k = k0 + int(blockIdx.z);  // components [k0, k0 + gridDim.z)
    const int i3 = int(n / p), c = int(n - int64_t(i3) * p);
    const int t1 = tile / nt2, t2 = tile - t1 * nt2;
    const int t = int(threadIdx.x);
    const int i1 = t1 * TC_TI1 + (t & 3), i2 = t2 * TC_TI2 + (t >> 2);
    // the component's scale: max over the pass's right-hand sides, reduced by the block
    // (one load per thread instead of p)
    __shared__ float wmx[TC_ROWS / 32];
    float m = 0.f;
    for (int cc = t; cc < p; cc += TC_ROWS) m = fmaxf(m, phimax[int64_t(cc) * q + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((t & 31) == 0) wmx[t >> 5] = m;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < TC_ROWS / 32; ++w) m = fmaxf(m, wmx[w]);
    const float sc = fp16_scale(m);
    float2 v = make_float2(0.f, 0.f);
    if (i1 < n1 && i2 < n2) {
        const int64_t nv = int64_t(n1) * n2 * n3;
        v = phi[ldphi * c + int64_t(k) * nv + i1 + int64_t(n1) * (i2 + int64_t(n2) * i3)];
    }
    uint32_t hi, lo;
    f16_split2(f2_pack(v.x * sc, v.y * sc), hi, lo);
    const int64_t pl = int64_t(q) * nt * R;
    unsigned short* o = reinterpret_cast<unsigned short*>(planes) + (int64_t(k) * nt + n) * R + int64_t(tile) * TC_ROWS +
                        (t & 3) * TC_TI2 + (t >> 2);
    // the B plane order of the forward kernel: Re hi, Im hi, Re lo, Im lo
    o[0] = static_cast<unsigned short>(hi);
    o[pl] = static_cast<unsigned short>(hi >> 16);
    o[2 * pl] = static_cast<unsigned short>(lo);
    o[3 * pl] = static_cast<unsigned short>(lo >> 16);
}

// z[j, c] = sum_k inv_k sum_r sum_i3 conj(U3n_jk[i3, r]) G[k][i3 p + c][kofs_jk + r]
// (U3n = U3 2^-e3 undoes the arena's normalisation W 2^e3; inv_k the W and
// Phi scales).  One block per column j; thread (c, i3 group) with the r3
// slots innermost (contiguous in G); the i3 groups are summed in a fixed
// order: bitwise reproducible.
// kmax[k] = max over the pass's right-hand sides c of phimax[c q + k] (the
// component's Phi scale, read by adjg_contract_kernel).
__global__ void phimax_k_kernel(const float* __restrict__ phimax, int p, int q, float* __restrict__ kmax) {
    for (int k = int(threadIdx.x); k < q; k += int(blockDim.x)) {
        float m = 0.f;
        for (int c = 0; c < p; ++c) m = fmaxf(m, phimax[int64_t(c) * q + k]);
        kmax[k] = m;
    }
}

__global__ void adjg_contract_kernel(const float2* __restrict__ G, int64_t gslots, int64_t nt, int p, int q,
                                     int64_t ncols, int n3, const TcDesc* __restrict__ tcd,
                                     const float2* __restrict__ arena, const int* __restrict__ kofs,
                                     const float* __restrict__ kmax, float wsc, float2* __restrict__ z,
                                     int64_t ldz) {
    __shared__ float2 red[256];
    const int64_t j = blockIdx.x;
    const int tid = int(threadIdx.x);
    for (int c0 = 0; c0 < p; c0 += 256) {
        const int pc = min(p - c0, 256), ng = 256 / pc;
        const int c = c0 + tid % pc, gi = tid / pc;
        float ar = 0.f, ai = 0.f;
        if (gi < ng) {
            for (int k = 0; k < q; ++k) {
                const float m = kmax[k];
                const int64_t t = int64_t(k) * ncols + j;
                const TcDesc d = tcd[t];
                const float sk = ldexpf(1.f, -fexp_e3(d.fexp)) / (wsc * fp16_scale(m));
                const float2* u3 = arena + d.off_u3;  // n3 x r3, row-major
                const float2* gk = G + int64_t(k) * nt * gslots + kofs[t];
                float kr = 0.f, ki = 0.f;
                for (int i3 = gi; i3 < n3; i3 += ng) {
                    const float2* gr = gk + (int64_t(i3) * p + c) * gslots;
                    for (int r = 0; r < d.r3; ++r) {
                        const float2 u = u3[i3 * d.r3 + r], gv = gr[r];
                        kr += u.x * gv.x + u.y * gv.y;  // conj(u) gv
                        ki += u.x * gv.y - u.y * gv.x;
                    }
                }
                ar += kr * sk;
                ai += ki * sk;
            }
        }
        red[tid] = make_float2(ar, ai);
        __syncthreads();
        if (tid < pc) {
            float sr = 0.f, si = 0.f;
            for (int g2 = 0; g2 < ng; ++g2) {
                sr += red[g2 * pc + tid].x;
                si += red[g2 * pc + tid].y;
            }
            z[j + ldz * (c0 + tid)] = make_float2(sr, si);
        }
        __syncthreads();
    }
}

}  // namespace tmb
