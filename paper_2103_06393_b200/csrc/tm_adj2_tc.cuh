// Tensor-core adjoint for groups of NR = 2 or 4 right-hand sides (p >= 2), complex64.
//
// The single-RHS adjoint (tm_adj_tc.cuh) recomputes its consumers' mode-2
// product W = V x_2 U2 for every right-hand side.  Here one CTA takes a row
// tile of NR right-hand sides c0 .. c0 + NR - 1: per chunk of CH = 128 / NR
// slots of the (j, c) stream the MMA warp builds Q for each,
//   [Qi|Qr]_r = Phi_r . [-U3i|U3r] + ...  (N = 2 CH, 6 kind::f16 MMAs per r
//   and 16 i3; TMEM buffer qb: columns qb 256 + r 2 CH + [Qi CH | Qr CH]),
// and each consumer thread forms W[row, c] once per column and contracts it
// with every Q_r — the reference's stacked_adjoint (src/matvec.cpp:67-102)
// with the projection form of SURVEY §8 (conj(T) . Phi = conj(W) . (Phi
// conj(U3))).  The CH-slot chunks use their own packing of the adjoint U3
// planes (tm_capi.cu: ensure_adj_pack), whole columns per chunk; TcDesc.pad1
// (CH 64) / pad2 (CH 32) is a column's slot inside its chunk.  Everything
// else (Phi planes, partials, adj_reduce_kernel, split final waves) is the
// single-RHS path's.  NR = 4 halves the W work again but its N = 64 MMAs
// read A (4 KB) per 2 KB of B, so the MMA side, not the consumers, bounds it
// (DESIGN.md §6).
#pragma once

#include "tm_adj_tc.cuh"

namespace tmb {

// NR right-hand sides per CTA (2 or 4): chunks of 128 / NR slots, so the
// TMEM holds [Qi|Qr] of every right-hand side twice (ping-pong).
template <int NR>
struct A2 {
    static constexpr int CH = 128 / NR;                         // (j, c) slots per chunk
    static constexpr int NST = NR == 4 ? 2 : 3;                 // A/B stages (16 i3 each)
    static constexpr int A_STAGE = NR * AJ_A_STAGE;             // Phi planes of the NR right-hand sides
    static constexpr int B_PLANE = CH * 32;
    static constexpr int B_STAGE = TC_BPLANES * B_PLANE;
    static constexpr int RED = 2 * NR * CH * AJ_NPW;            // float2 partial buffer [buf][rhs][col][warp]
};

// Tile of a pass over right-hand-side groups: item -> (group cp, component k,
// row tile rt), i2 block fastest as in aj_tile.
template <int NR>
__device__ __forceinline__ AjTile aj2_tile(const AjGeom& g, int64_t item, uint32_t rank = 0) {
    AjTile r;
    const int64_t t = g.tile0 + item / g.split;
    r.part = int(item % g.split);
    const int64_t tpk = g.nrt >> g.pair;  // (pair) tiles per component
    const int64_t per_c = int64_t(g.q) * tpk;
    const int64_t cp = t / per_c;
    r.c = int(NR * cp);
    int64_t rem = t - cp * per_c;
    r.k = int(rem / tpk);
    r.rt = ((rem - int64_t(r.k) * tpk) << g.pair) + rank;  // a pair tile = row tiles 2 pt, 2 pt + 1
    const int t1 = int(r.rt / g.nt2), t2 = int(r.rt - int64_t(t1) * g.nt2);
    r.i1_0 = t1 * TC_TI1;
    r.i2_0 = t2 * TC_TI2;
    return r;
}

// One column for the consumer thread: W once, then sum_c conj(W) Q_r for the
// NR right-hand sides (Q_r: Qi at qaddr + r 2 CH + s, Qr at + CH).
template <int NU, int NR>
__device__ __forceinline__ void aj2_consume_column(const float2* __restrict__ V, const float2* __restrict__ U2,
                                                   int r2, int ld2, int r3, int h, int lane, uint32_t qaddr,
                                                   uint64_t* fempty_s, float2 (&a)[NR]) {
    constexpr int CH = A2<NR>::CH;
    using namespace sm100;
    uint64_t w[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) w[u] = 0;
    const float2* vp = V + 4 * h;  // V[(c + r3 b) * 4 + il], c = NH u + h (as aj_consume_column)
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
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
        uint32_t qi[NU], qr[NU];
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const uint32_t s = (u < NU - 1 || AJ_NH * u + h < r3) ? uint32_t(AJ_NH * u + h) : 0u;
            const uint32_t q0 = qaddr + uint32_t(rr * 2 * CH) + s;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(qi[u]) : "r"(q0));
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(qr[u]) : "r"(q0 + CH));
        }
        tmem_ld_wait();
        float ar = 0.f, ai = 0.f;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            if (u < NU - 1 || AJ_NH * u + h < r3) {
                const float2 wv = f2_unpack(w[u]);
                const float qre = __uint_as_float(qr[u]), qim = __uint_as_float(qi[u]);
                ar = fmaf(wv.x, qre, fmaf(wv.y, qim, ar));
                ai = fmaf(wv.x, qim, fmaf(-wv.y, qre, ai));
            }
        }
        a[rr] = make_float2(ar, ai);
    }
}

// PAIR: CTA pairs (cta_group::2, M = 256 over two row tiles) as in
// adj_tc_kernel: each N = 2 CH window [-U3i | U3r] / [U3r | U3i] takes its
// first CH rows from the even CTA and the rest from the odd one, so a CTA
// stages 4 of the 6 U3 planes' halves and reads half of B per MMA.
template <int NR, bool PAIR, bool BIG = false>  // BIG: r3 > 16 (see adj_tc_kernel)
__global__ void __launch_bounds__(AJ_THREADS, 1)
    adj_tc2_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                   const TcDesc* __restrict__ tcd, const float2* __restrict__ varena,
                   const float2* __restrict__ u2arena, const int* __restrict__ nch, const int* __restrict__ cstart,
                   AjGeom g, const float* __restrict__ phimax, float2* __restrict__ part) {
    using namespace sm100;
    using P = A2<NR>;
    constexpr int A2_CH = P::CH, A2_NST = P::NST, A2_A_STAGE = P::A_STAGE, A2_B_PLANE = P::B_PLANE,
                  A2_B_STAGE = PAIR ? 4 * P::B_PLANE : P::B_STAGE;
    extern __shared__ __align__(1024) unsigned char a2_smem_raw[];
    unsigned char* sm = a2_smem_raw + ((1024u - (smem_u32(a2_smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = sm;
    unsigned char* sB = sA + A2_NST * A2_A_STAGE;
    unsigned char* sSlot = sB + A2_NST * A2_B_STAGE;
    float2* red = reinterpret_cast<float2*>(sSlot + TC_JR * g.slot_bytes);  // [2 buf][NR rhs][A2_CH cols][8]
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + P::RED);
    uint64_t* full = bars;                 // [NST]
    uint64_t* empty = full + A2_NST;       // [NST]
    uint64_t* ffull = empty + A2_NST;      // [JR]
    uint64_t* fempty = ffull + TC_JR;      // [JR]
    uint64_t* qfull = fempty + TC_JR;      // [2]
    uint64_t* qfree = qfull + 2;           // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qfree + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const int64_t tstart = g.t_begin + (PAIR ? (blockIdx.x >> 1) : blockIdx.x);
    const int64_t tstep = PAIR ? (gridDim.x >> 1) : gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < A2_NST; ++s) {
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
                const AjTile tl = aj2_tile<NR>(g, t, rank);
                int n0, n1;
                aj_chunks(g, tl, nch[tl.k], n0, n1);
                const int arow = int(tl.rt * TC_ROWS);
                for (int n = n0; n < n1; ++n) {
                    for (int kk = 0; kk < g.nks; ++kk) {
                        mbar_wait_backoff(&empty[s], ph ^ 1, TC_BACKOFF_ADJ);
                        unsigned char* da = sA + s * A2_A_STAGE;
                        unsigned char* db = sB + s * A2_B_STAGE;
                        if (PAIR) {
                            // both CTAs' bytes complete on the even CTA's barrier
                            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2u * uint32_t(A2_A_STAGE + A2_B_STAGE));
                            const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
#pragma unroll
                            for (int rr = 0; rr < NR; ++rr)
#pragma unroll
                                for (int pl = 0; pl < AJ_APLANES; ++pl)
                                    tma_load_3d_pair(da + (rr * AJ_APLANES + pl) * AJ_A_PLANE, &amap, fb, kk * 16,
                                                     arow, (pl * g.p + tl.c + rr) * g.q + tl.k);
                            // smem B slots (W1 hi, W2 hi, W1 lo, W2 lo) <- planes rank + {0, 1} (+3 for lo)
#pragma unroll
                            for (int sl = 0; sl < 4; ++sl)
                                tma_load_3d_pair(db + sl * A2_B_PLANE, &bmap, fb, kk * 16, n * A2_CH,
                                                 (int(rank) + (sl & 1) + 3 * (sl >> 1)) * g.q + tl.k);
                        } else {
                            mbar_arrive_expect_tx(&full[s], uint32_t(A2_A_STAGE + A2_B_STAGE));
#pragma unroll
                            for (int rr = 0; rr < NR; ++rr)
#pragma unroll
                                for (int pl = 0; pl < AJ_APLANES; ++pl)
                                    tma_load_3d(da + (rr * AJ_APLANES + pl) * AJ_A_PLANE, &amap, &full[s], kk * 16,
                                                arow, (pl * g.p + tl.c + rr) * g.q + tl.k);
#pragma unroll
                            for (int pl = 0; pl < TC_BPLANES; ++pl)
                                tma_load_3d(db + pl * A2_B_PLANE, &bmap, &full[s], kk * 16, n * A2_CH,
                                            pl * g.q + tl.k);
                        }
                        if (++s == A2_NST) {
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
            const uint32_t idesc = umma_idesc_f16(TC_ROWS * (PAIR ? 2 : 1), 2 * A2_CH, false, false);
            uint32_t s = 0, ph = 0, nq = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const AjTile tl = aj2_tile<NR>(g, t, rank);
                int n0, n1;
                aj_chunks(g, tl, nch[tl.k], n0, n1);
                for (int n = n0; n < n1; ++n, ++nq) {
                    const uint32_t qb = nq & 1, qph = (nq >> 1) & 1;
                    mbar_wait(&qfree[qb], qph ^ 1);
                    tc_fence_after();
                    for (int kk = 0; kk < g.nks; ++kk) {
                        mbar_wait(&full[s], ph);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + s * A2_A_STAGE);
                        const uint32_t b0 = smem_u32(sB + s * A2_B_STAGE);
                        // B windows: [-U3i|U3r] at plane 0 / 3 (hi / lo), [U3r|U3i] at plane 1 / 4
                        // (PAIR: smem slots 0 / 2 and 1 / 3 of each CTA, half a window each)
                        const uint64_t B2h = umma_smem_desc(b0 + 0 * A2_B_PLANE, 256, 6);
                        const uint64_t B1h = umma_smem_desc(b0 + 1 * A2_B_PLANE, 256, 6);
                        const uint64_t B2l = umma_smem_desc(b0 + (PAIR ? 2 : 3) * A2_B_PLANE, 256, 6);
                        const uint64_t B1l = umma_smem_desc(b0 + (PAIR ? 3 : 4) * A2_B_PLANE, 256, 6);
                        const uint32_t acc = kk > 0 ? 1u : 0u;
#pragma unroll
                        for (int rr = 0; rr < NR; ++rr) {
                            uint64_t A[4];
#pragma unroll
                            for (int pl = 0; pl < 4; ++pl)
                                A[pl] = umma_smem_desc(a0 + (rr * AJ_APLANES + pl) * AJ_A_PLANE, 256, 6);
                            const uint32_t qd = tmem + qb * 256u + uint32_t(rr * 2 * A2_CH);
#define MMA(...) (PAIR ? mma_f16_pair(__VA_ARGS__) : mma_f16(__VA_ARGS__))
                            MMA(qd, A[0], B2h, idesc, acc);
                            MMA(qd, A[0], B2l, idesc, 1);
                            MMA(qd, A[1], B2h, idesc, 1);
                            MMA(qd, A[2], B1h, idesc, 1);
                            MMA(qd, A[2], B1l, idesc, 1);
                            MMA(qd, A[3], B1h, idesc, 1);
#undef MMA
                        }
                        if (PAIR)
                            mma_commit_pair(&empty[s]);
                        else
                            mma_commit(&empty[s]);
                        if (++s == A2_NST) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                    if (PAIR)
                        mma_commit_pair(&qfull[qb]);
                    else
                        mma_commit(&qfull[qb]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---------------------------------------------------- factor loader
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const AjTile tl = aj2_tile<NR>(g, t, rank);
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
            const AjTile tl = aj2_tile<NR>(g, t, rank);
            int n0, n1;
            aj_chunks(g, tl, nch[tl.k], n0, n1);
            const int* cs = cstart + int64_t(tl.k) * (g.maxch + 1);
            float inv_scale[NR];
#pragma unroll
            for (int rr = 0; rr < NR; ++rr)
                inv_scale[rr] = 1.f / (aj_phi_scale(phimax[int64_t(tl.c + rr) * g.q + tl.k]) * AJ_U3_SCALE);
            for (int n = n0; n < n1; ++n, ++nq) {
                const uint32_t qb = nq & 1, qph = (nq >> 1) & 1;
                const int j0 = cs[n], j1 = cs[n + 1];
                float2* rb = red + (nq & 1) * NR * A2_CH * AJ_NPW;  // [rhs][col][warp]
                mbar_wait(&qfull[qb], qph);
                tc_fence_after();
                const uint32_t qbase = tmem + lane_addr + qb * 256u;
                for (int j = j0; j < j1; ++j) {
                    mbar_wait(&ffull[fs], fph);
                    const unsigned char* slot = sSlot + fs * g.slot_bytes;
                    const TcDesc* dd = reinterpret_cast<const TcDesc*>(slot);
                    // slot inside the chunk: pad1 for 64-slot chunks, pad2 for 32-slot chunks
                    const int r2 = dd->r2, r3 = dd->r3, soff = NR == 2 ? dd->pad1 : dd->pad2;
                    const float2* V = reinterpret_cast<const float2*>(slot + TC_SLOT_V) + i1l;
                    const float2* U2 = reinterpret_cast<const float2*>(slot + g.u2_off);
                    float2 a[NR];
#define A2_COL(NU) \
    aj2_consume_column<NU, NR>(V, U2, (g.debug & 4) ? 0 : r2, r2 | 1, r3, h, lane, qbase + uint32_t(soff), &fempty[fs], a)
                    if constexpr (BIG) {
                        switch ((r3 + AJ_NH - 1) / AJ_NH) {
                            case 1: A2_COL(1); break;
                            case 2: A2_COL(2); break;
                            case 3: A2_COL(3); break;
                            case 4: A2_COL(4); break;
                            case 5: A2_COL(5); break;
                            case 6: A2_COL(6); break;
                            case 7: A2_COL(7); break;
                            case 8: A2_COL(8); break;
                            case 9: A2_COL(9); break;
                            case 10: A2_COL(10); break;
                            case 11: A2_COL(11); break;
                            case 12: A2_COL(12); break;
                            case 13: A2_COL(13); break;
                            case 14: A2_COL(14); break;
                            case 15: A2_COL(15); break;
                            default: A2_COL(16); break;
                        }
                    } else {
                        switch ((r3 + AJ_NH - 1) / AJ_NH) {
                            case 1: A2_COL(1); break;
                            case 2: A2_COL(2); break;
                            case 3: A2_COL(3); break;
                            case 4: A2_COL(4); break;
                            case 5: A2_COL(5); break;
                            case 6: A2_COL(6); break;
                            case 7: A2_COL(7); break;
                            default: A2_COL(8); break;
                        }
                    }
#undef A2_COL
                    if (++fs == TC_JR) {
                        fs = 0;
                        fph ^= 1;
                    }
#pragma unroll
                    for (int rr = 0; rr < NR; ++rr) {
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            a[rr].x += __shfl_xor_sync(0xffffffffu, a[rr].x, o);
                            a[rr].y += __shfl_xor_sync(0xffffffffu, a[rr].y, o);
                        }
                        if (lane == 0) rb[(rr * A2_CH + (j - j0)) * AJ_NPW + pw] = a[rr];
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_cluster(mapa_shared(smem_u32(&qfree[qb]), 0));
                    else
                        mbar_arrive(&qfree[qb]);
                }
                named_bar_sync(1, AJ_NPW * 32);  // all partials of the chunk are in rb
                for (int e = ctid; e < NR * (j1 - j0); e += AJ_NPW * 32) {
                    const int rr = e / (j1 - j0), jj = e - rr * (j1 - j0);
                    float sx = 0.f, sy = 0.f;
#pragma unroll
                    for (int w = 0; w < AJ_NPW; ++w) {
                        sx += rb[(rr * A2_CH + jj) * AJ_NPW + w].x;
                        sy += rb[(rr * A2_CH + jj) * AJ_NPW + w].y;
                    }
                    part[((int64_t(tl.c + rr) * g.ncols + j0 + jj) * g.q + tl.k) * g.nrt + tl.rt] =
                        make_float2(sx * inv_scale[rr], sy * inv_scale[rr]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // the peer no longer arrives on this CTA's barriers / uses the pair's TMEM
    if (warp == 3) {
        if (PAIR)
            tmem_dealloc_pair(tmem, 512);
        else
            tmem_dealloc(tmem, 512);
    }
}

}  // namespace tmb
