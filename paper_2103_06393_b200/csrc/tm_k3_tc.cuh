// Batched multi-RHS forward at (near) algorithmic cost ("K3"), complex64,
// for large right-hand-side counts (config 5: p = 32).
//
// The x-in-B forward (tm_kernels_tc.cuh) multiplies every W element into the
// N space i3 x p: r3 * p tensor MACs per voxel and column against the
// reference's r3 + p (reconstruct's mode 3 and the rank-1 update,
// src/matvec.cpp:43-49).  K3 decompresses each column ONCE per tile instead:
//
//   T_j[row, i3] = sum_c W_j[row, c] U3_j[i3, c]      (CUDA cores, fp32)
//   Y[row, i3, :] += sum_j T_j[row, i3] X[j, :]        (tcgen05, K = columns)
//
// Tile = 128 rows (4 i1 x 32 i2) x 4 i3 x up to 32 right-hand sides.  Per
// column the producer warps form W = V x_2 U2 (V = U1 x_1 G from the store's
// V arena) and T for the tile's 4 i3, and write T as a scaled 2-term fp16
// split (re hi, re lo, im hi, im lo) into the A operand of GEMM2: four
// M = 128 blocks (one per i3), K = 16 consecutive columns per stage.  B is
// X (m x p) as fp16 split planes [Xr | Xi] and [-Xi | Xr] (N = 64: the p = 32
// right-hand sides' real and imaginary parts), streamed by TMA.  Per stage the
// MMA thread issues 6 tcgen05.mma.kind::f16 (M = 128, N = 64, K = 16) per i3
// block:  [Yr | Yi] += Tr [Xr | Xi] + Ti [-Xi | Xr],  each as hi.hi + hi.lo
// + lo.hi.  Accumulation is chained (`chain` stages per TMEM chain, folded
// into a per-CTA running sum in L2 by 4 fold warps, as the x-in-B forward),
// so the tensor core's truncating fp32 accumulate does not drift with m.
//
// Warp roles (512 threads, 1 CTA / SM, persistent over tiles):
//   warp 0      TMA producer of the X planes (B)
//   warp 1      MMA issuer
//   warp 2      factor loader: per column {TcDesc, V rows, U2 rows, U3 rows}
//   warp 3      TMEM allocator (256 columns: 4 i3 x [Yr | Yi] x 32)
//   warps 4-11  producers: W, T, fp16 split -> A stage
//   warps 12-15 chain fold + epilogue
#pragma once

#include <cuda_fp16.h>

#include "tm_common.cuh"
#include "tm_kernels_tc.cuh"
#include "tm_sm100.cuh"

namespace tmb {

constexpr int K3_NI3 = 4;                        // i3 per tile (one M = 128 block each)
constexpr int K3_P = 32;                         // right-hand sides per pass (N = 2 K3_P)
constexpr int K3_NST = 2;                        // A/B stages (16 columns each)
constexpr int K3_A_PLANE = TC_ROWS * 32;         // one plane of one i3 block: 128 rows x 16 fp16
constexpr int K3_A_BLOCK = 4 * K3_A_PLANE;       // re hi, re lo, im hi, im lo
constexpr int K3_A_STAGE = K3_NI3 * K3_A_BLOCK;  // 64 KB
constexpr int K3_B_PLANE = 2 * K3_P * 32;        // 64 rows x 16 fp16
constexpr int K3_B_STAGE = 4 * K3_B_PLANE;       // [Xr|Xi] hi, [-Xi|Xr] hi, [Xr|Xi] lo, [-Xi|Xr] lo
constexpr int K3_YCOLS = K3_NI3 * 2 * K3_P;      // TMEM columns of the accumulator
constexpr int K3_THREADS = 16 * 32;

struct K3Geom {
    int64_t ncols;
    int n1, n2, n3, q;
    int nt1, nt2, nt3;
    int p;             // right-hand sides of this pass (<= K3_P)
    int64_t ntiles;
    int rmax2, rmax3;
    int slot_bytes, u2_off, u3_off;
    int nks;           // K stages per tile = ceil(ncols / 16)
    int chain;         // K stages per TMEM accumulation chain
    int jr;            // factor-ring slots (as many as shared memory allows, <= K3_JR_MAX): a
                       // column is little work, so the ring must cover the bulk-copy latency
    float sa;          // fp16 scale of T (power of two)
};
constexpr int K3_JR_MAX = 12;

struct K3Tile {
    int k, i1_0, i2_0, i3_0;
};

// Tile order: i3 block fastest (the tiles resident together share the V / U2
// rows of their (i1, i2) block), then i2 block, i1 block, component.
__host__ __device__ inline K3Tile k3_tile(const K3Geom& g, int64_t t) {
    K3Tile r;
    const int64_t per_k = int64_t(g.nt1) * g.nt2 * g.nt3;
    r.k = int(t / per_k);
    int64_t rem = t - int64_t(r.k) * per_k;
    const int t1 = int(rem / (int64_t(g.nt2) * g.nt3));
    rem -= int64_t(t1) * g.nt2 * g.nt3;
    const int t2 = int(rem / g.nt3);
    const int t3 = int(rem - int64_t(t2) * g.nt3);
    r.i1_0 = t1 * TC_TI1;
    r.i2_0 = t2 * TC_TI2;
    r.i3_0 = t3 * K3_NI3;
    return r;
}

// One column for one producer thread: row = (t >> 1) of the tile, c parity h.
// W[row, c] for c = h, h + 2, ... (NU values), the partial T over those c for
// the tile's 4 i3, the pair's sum (shuffle), then the two i3 l = 2h, 2h + 1 of
// this thread written as a scaled fp16 split into K slot `ks` of stage `st`.
template <int NU>
__device__ __forceinline__ void k3_produce_column(const float2* __restrict__ V, const float2* __restrict__ U2,
                                                  const float2* __restrict__ U3, int r2, int ld2, int r3, int h,
                                                  int i1l, int i2, float tsc, int nvalid, unsigned char* st,
                                                  uint32_t rowbase, uint32_t xorv, uint32_t ks,
                                                  uint64_t* fempty_s, int lane) {
    using namespace sm100;
    uint64_t w[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) w[u] = 0;
    // V[(c + r3 b) * 4 + i1l] with c = h + 2u; for c >= r3 (odd r3, h = 1, last
    // u) the load reads the next V entry (inside the slot) and is dropped below
    const float2* vp = V + 4 * h + i1l;
    const float2* up = U2 + i2 * ld2;
    const int vstep = 4 * r3;
#pragma unroll 2
    for (int b = 0; b < r2; ++b) {
        const float2 ub = up[b];
#pragma unroll
        for (int u = 0; u < NU; ++u) cfma2v(w[u], vp[8 * u], ub);
        vp += vstep;
    }
    // T partials over this thread's c, for the 4 i3 of the tile
    uint64_t tp[K3_NI3];
#pragma unroll
    for (int l = 0; l < K3_NI3; ++l) {
        tp[l] = 0;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const int c = h + 2 * u;
            if (u < NU - 1 || c < r3) cfma2v(tp[l], f2_unpack(w[u]), U3[l * r3 + c]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(fempty_s);  // this warp no longer reads the slot
    // the pair (lanes 2k, 2k + 1: same row, c parities 0 / 1) sums its halves
#pragma unroll
    for (int l = 0; l < K3_NI3; ++l) {
        float2 v = f2_unpack(tp[l]);
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
        tp[l] = f2_pack(v.x * tsc, v.y * tsc);
    }
    // this thread writes i3 l = 2h, 2h + 1 (zero past the grid's n3)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int l = 2 * h + e;
        const uint64_t tv = (l < nvalid) ? (h ? tp[2 + e] : tp[e]) : 0ull;
        uint32_t hi, lo;
        f16_split2(tv, hi, lo);
        unsigned short* a =
            reinterpret_cast<unsigned short*>(st + l * K3_A_BLOCK + rowbase + ((ks * 2u) ^ xorv));
        a[0] = static_cast<unsigned short>(hi);                           // re hi
        a[K3_A_PLANE / 2] = static_cast<unsigned short>(lo);              // re lo
        a[2 * K3_A_PLANE / 2] = static_cast<unsigned short>(hi >> 16);    // im hi
        a[3 * K3_A_PLANE / 2] = static_cast<unsigned short>(lo >> 16);    // im lo
    }
}

__global__ void __launch_bounds__(K3_THREADS, 1)
    fwd_k3_kernel(const __grid_constant__ CUtensorMap xmap, const TcDesc* __restrict__ tcd,
                  const float2* __restrict__ varena, const float2* __restrict__ u2arena,
                  const float2* __restrict__ arena, K3Geom g, float2* __restrict__ y, int64_t ldy,
                  float* __restrict__ rsum, const float* __restrict__ xmax) {
    using namespace sm100;
    extern __shared__ __align__(1024) unsigned char k3_smem_raw[];
    unsigned char* sm = k3_smem_raw + ((1024u - (smem_u32(k3_smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = sm;
    unsigned char* sB = sA + K3_NST * K3_A_STAGE;
    unsigned char* sSlot = sB + K3_NST * K3_B_STAGE;
    const uint32_t jr = uint32_t(g.jr);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sSlot + jr * g.slot_bytes);
    uint64_t* full = bars;              // [K3_NST]
    uint64_t* empty = full + K3_NST;    // [K3_NST]
    uint64_t* ffull = empty + K3_NST;   // [jr]
    uint64_t* fempty = ffull + K3_JR_MAX;  // [jr]
    uint64_t* cfull = fempty + K3_JR_MAX;  // 1
    uint64_t* cfree = cfull + 1;        // 1
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfree + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < K3_NST; ++s) {
            mbar_init(&full[s], 1 + 8);
            mbar_init(&empty[s], 1);
        }
        for (uint32_t s = 0; s < jr; ++s) {
            mbar_init(&ffull[s], 1);
            mbar_init(&fempty[s], 8);
        }
        mbar_init(cfull, 1);
        mbar_init(cfree, 4);
        fence_mbar_init();
    }
    // A stages start as zeros: K slots past the last column of a tile multiply
    // the zero-padded X rows and must be finite
    for (int i = threadIdx.x; i < K3_NST * K3_A_STAGE / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sA)[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    if (warp == 3) tmem_alloc(tmem_slot, K3_YCOLS);
    if (warp == 0 && lane == 0) tma_prefetch_desc(&xmap);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t tstart = blockIdx.x, tstep = gridDim.x;

    if (warp == 0) {
        // ------------------------------------------------ X-plane TMA producer
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.ntiles; t += tstep)
                for (int kk = 0; kk < g.nks; ++kk) {
                    mbar_wait_backoff(&empty[s], ph ^ 1, 128);
                    mbar_arrive_expect_tx(&full[s], uint32_t(K3_B_STAGE));
                    unsigned char* dst = sB + s * K3_B_STAGE;
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) tma_load_3d(dst + pl * K3_B_PLANE, &xmap, &full[s], kk * 16, 0, pl);
                    if (++s == K3_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t id = umma_idesc_f16(TC_ROWS, 2 * K3_P, false, false);
            uint32_t s = 0, ph = 0, gch = 0;
            for (int64_t t = tstart; t < g.ntiles; t += tstep) {
                int cpos = 0;
                for (int kk = 0; kk < g.nks; ++kk) {
                    if (cpos == 0) {
                        mbar_wait(cfree, (gch & 1) ^ 1);  // the previous chain has been folded
                        tc_fence_after();
                    }
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + s * K3_A_STAGE);
                    const uint32_t b0 = smem_u32(sB + s * K3_B_STAGE);
                    const uint64_t Bah = umma_smem_desc(b0, 256, 6);
                    const uint64_t Bbh = umma_smem_desc(b0 + K3_B_PLANE, 256, 6);
                    const uint64_t Bal = umma_smem_desc(b0 + 2 * K3_B_PLANE, 256, 6);
                    const uint64_t Bbl = umma_smem_desc(b0 + 3 * K3_B_PLANE, 256, 6);
                    const uint32_t acc = cpos > 0 ? 1u : 0u;
#pragma unroll
                    for (int l = 0; l < K3_NI3; ++l) {
                        const uint32_t ab = a0 + l * K3_A_BLOCK;
                        const uint64_t Arh = umma_smem_desc(ab, 256, 6);
                        const uint64_t Arl = umma_smem_desc(ab + K3_A_PLANE, 256, 6);
                        const uint64_t Aih = umma_smem_desc(ab + 2 * K3_A_PLANE, 256, 6);
                        const uint64_t Ail = umma_smem_desc(ab + 3 * K3_A_PLANE, 256, 6);
                        const uint32_t d = tmem + uint32_t(l * 2 * K3_P);
                        // [Yr | Yi] += Tr [Xr | Xi] + Ti [-Xi | Xr], each as hi.hi + hi.lo + lo.hi
                        mma_f16(d, Arh, Bah, id, acc);
                        mma_f16(d, Arh, Bal, id, 1);
                        mma_f16(d, Arl, Bah, id, 1);
                        mma_f16(d, Aih, Bbh, id, 1);
                        mma_f16(d, Aih, Bbl, id, 1);
                        mma_f16(d, Ail, Bbh, id, 1);
                    }
                    mma_commit(&empty[s]);
                    if (++s == K3_NST) {
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
            for (int64_t t = tstart; t < g.ntiles; t += tstep) {
                const K3Tile tl = k3_tile(g, t);
                const TcDesc* tdk = tcd + int64_t(tl.k) * g.ncols;
                for (int64_t j = 0; j < g.ncols; ++j) {
                    mbar_wait_backoff(&fempty[s], ph ^ 1, 128);
                    const TcDesc d = tdk[j];
                    unsigned char* slot = sSlot + s * g.slot_bytes;
                    const uint32_t r23 = uint32_t(d.r2 * d.r3);
                    const uint32_t ld2 = uint32_t(d.r2 | 1);
                    const uint32_t bv = round16(uint32_t(TC_TI1) * r23 * 8u);
                    const uint32_t b2 = uint32_t(TC_TI2) * ld2 * 8u;
                    const uint32_t b3 = uint32_t(K3_NI3) * uint32_t(d.r3) * 8u;  // multiple of 16
                    mbar_arrive_expect_tx(&ffull[s], uint32_t(sizeof(TcDesc)) + bv + b2 + b3);
                    bulk_g2s(slot, tdk + j, uint32_t(sizeof(TcDesc)), &ffull[s]);
                    bulk_g2s(slot + TC_SLOT_V, varena + d.off_v + int64_t(tl.i1_0) * r23, bv, &ffull[s]);
                    bulk_g2s(slot + g.u2_off, u2arena + d.off_u2 + int64_t(tl.i2_0) * ld2, b2, &ffull[s]);
                    bulk_g2s(slot + g.u3_off, arena + d.off_u3 + int64_t(tl.i3_0) * d.r3, b3, &ffull[s]);
                    if (++s == jr) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp >= TC_PW0 && warp < TC_PW0 + 8) {
        // ------------------------------------------------------- producers
        const int pt = threadIdx.x - TC_PW0 * 32;  // 0..255
        const int row = pt >> 1, h = pt & 1;       // tile row = i2 + 32 i1 (= TMEM lane)
        const int i1l = row >> 5, i2 = row & 31;
        const uint32_t rowbase = uint32_t(row) * 32u, xorv = (uint32_t(row) & 4u) << 2;
        uint32_t fs = 0, fph = 0, s = 0, ph = 0;
        for (int64_t t = tstart; t < g.ntiles; t += tstep) {
            const K3Tile tl = k3_tile(g, t);
            const int nvalid = min(K3_NI3, g.n3 - tl.i3_0);
            for (int64_t j = 0; j < g.ncols; ++j) {
                const uint32_t ks = uint32_t(j & 15);
                if (ks == 0) mbar_wait(&empty[s], ph ^ 1u);
                mbar_wait(&ffull[fs], fph);
                const unsigned char* slot = sSlot + fs * g.slot_bytes;
                const TcDesc* dd = reinterpret_cast<const TcDesc*>(slot);
                const int r2 = dd->r2, r3 = dd->r3;
                // T = (W_n . U3) 2^-e3: W_n carries the store's factor normalisation
                const float tsc = ldexpf(g.sa, -fexp_e3(dd->fexp));
                const float2* V = reinterpret_cast<const float2*>(slot + TC_SLOT_V);
                const float2* U2 = reinterpret_cast<const float2*>(slot + g.u2_off);
                const float2* U3 = reinterpret_cast<const float2*>(slot + g.u3_off);
                unsigned char* st = sA + s * K3_A_STAGE;
#define K3_COL(NU) \
    k3_produce_column<NU>(V, U2, U3, r2, r2 | 1, r3, h, i1l, i2, tsc, nvalid, st, rowbase, xorv, ks, &fempty[fs], lane)
                switch ((r3 + 1) >> 1) {
                    case 1: K3_COL(1); break;
                    case 2: K3_COL(2); break;
                    case 3: K3_COL(3); break;
                    case 4: K3_COL(4); break;
                    case 5: K3_COL(5); break;
                    case 6: K3_COL(6); break;
                    case 7: K3_COL(7); break;
                    default: K3_COL(8); break;
                }
#undef K3_COL
                if (++fs == jr) {
                    fs = 0;
                    fph ^= 1;
                }
                if (ks == 15 || j == g.ncols - 1) {  // stage complete (a tile's last one may be partial)
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[s]);
                    if (++s == K3_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp >= TC_PW0 + 8) {
        // ------------------------------------------ chain fold + epilogue
        // Running sum of the tile: rsum[blockIdx.x][col / 4][row] as float4
        // (4 consecutive TMEM columns), L2-resident; the first chain stores,
        // later chains add (red.global.add, round-to-nearest), the last chain
        // reads it back and writes y.
        const int quarter = warp & 3;
        const uint32_t tC = tmem + (uint32_t(quarter * 32) << 16);
        const int row = lane + 32 * quarter;
        float4* rs = reinterpret_cast<float4*>(rsum) + int64_t(blockIdx.x) * (K3_YCOLS / 4) * TC_ROWS + row;
        const int64_t nv3 = int64_t(g.n1) * g.n2 * g.n3;
        const int nch = (g.nks + g.chain - 1) / g.chain;
        const float inv = 1.f / (g.sa * fp16_scale(*xmax));  // exact power of two (T scale x X scale)
        uint32_t gch = 0;
        for (int64_t t = tstart; t < g.ntiles; t += tstep) {
            const K3Tile tl = k3_tile(g, t);
            const int ei1 = tl.i1_0 + quarter, ei2 = tl.i2_0 + lane;
            const bool eok = ei1 < g.n1 && ei2 < g.n2;
            for (int ch = 0; ch < nch; ++ch, ++gch) {
                mbar_wait_backoff(cfull, gch & 1, 256);
                tc_fence_after();
                const bool last = ch == nch - 1;
                for (int l = 0; l < K3_NI3; ++l)
                    for (int cb = 0; cb < K3_P; cb += 16) {
                        uint32_t cr[16], ci[16];
                        const int col = l * 2 * K3_P + cb;  // Yr of rhs cb.. at col, Yi at col + K3_P
                        tmem_ld16(tC + uint32_t(col), cr);
                        tmem_ld16(tC + uint32_t(col + K3_P), ci);
                        tmem_ld_wait();
                        float4* rr = rs + int64_t(col / 4) * TC_ROWS;
                        float4* ri = rs + int64_t((col + K3_P) / 4) * TC_ROWS;
                        if (!last) {
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const float4 vr = make_float4(__uint_as_float(cr[4 * m]), __uint_as_float(cr[4 * m + 1]),
                                                              __uint_as_float(cr[4 * m + 2]),
                                                              __uint_as_float(cr[4 * m + 3]));
                                const float4 vi = make_float4(__uint_as_float(ci[4 * m]), __uint_as_float(ci[4 * m + 1]),
                                                              __uint_as_float(ci[4 * m + 2]),
                                                              __uint_as_float(ci[4 * m + 3]));
                                float4* a = rr + int64_t(m) * TC_ROWS;
                                float4* b = ri + int64_t(m) * TC_ROWS;
                                if (ch == 0) {
                                    *a = vr;
                                    *b = vi;
                                } else {
                                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(vr.x),
                                                 "f"(vr.y), "f"(vr.z), "f"(vr.w)
                                                 : "memory");
                                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(b), "f"(vi.x),
                                                 "f"(vi.y), "f"(vi.z), "f"(vi.w)
                                                 : "memory");
                                }
                            }
                        } else if (eok && tl.i3_0 + l < g.n3) {
                            float2* yp = y + int64_t(tl.k) * nv3 + ei1 + int64_t(g.n1) * (ei2 + int64_t(g.n2) * (tl.i3_0 + l));
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
                                if (ch > 0) {
                                    ar = rr[int64_t(m) * TC_ROWS];
                                    ai = ri[int64_t(m) * TC_ROWS];
                                }
                                const float re[4] = {__uint_as_float(cr[4 * m]) + ar.x, __uint_as_float(cr[4 * m + 1]) + ar.y,
                                                     __uint_as_float(cr[4 * m + 2]) + ar.z,
                                                     __uint_as_float(cr[4 * m + 3]) + ar.w};
                                const float im[4] = {__uint_as_float(ci[4 * m]) + ai.x, __uint_as_float(ci[4 * m + 1]) + ai.y,
                                                     __uint_as_float(ci[4 * m + 2]) + ai.z,
                                                     __uint_as_float(ci[4 * m + 3]) + ai.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const int c = cb + 4 * m + e;
                                    if (c < g.p) yp[ldy * c] = make_float2(re[e] * inv, im[e] * inv);
                                }
                            }
                        }
                    }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(cfree);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc(tmem, K3_YCOLS);
}

// X planes of a pass (B of GEMM2): [4][2 K3_P rows n][kpad columns j] fp16,
// plane 0 = [Xr | Xi] hi, 1 = [-Xi | Xr] hi, 2 / 3 the same lo; row n < K3_P
// is right-hand side n's first half of the pair, n >= K3_P the second; rows
// of right-hand sides >= p and columns >= m are zero.  sb = fp16_scale(max|x|).
__global__ void k3_xplanes_kernel(const float2* __restrict__ x, int64_t ldx, int64_t ncols, int p, int64_t kpad,
                                  const float* __restrict__ xmax, __half* __restrict__ planes) {
    const float sb = fp16_scale(*xmax);
    const int64_t plane = int64_t(2 * K3_P) * kpad;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(K3_P) * kpad;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e / kpad);
        const int64_t j = e - int64_t(c) * kpad;
        float2 v = make_float2(0.f, 0.f);
        if (c < p && j < ncols) {
            v = x[j + ldx * c];
            v.x *= sb;
            v.y *= sb;
        }
        const __half rh = __float2half_rn(v.x), ih = __float2half_rn(v.y);
        const __half rl = __float2half_rn(v.x - __half2float(rh)), il = __float2half_rn(v.y - __half2float(ih));
        const int64_t o1 = int64_t(c) * kpad + j, o2 = int64_t(c + K3_P) * kpad + j;
        planes[o1] = rh;                      // [Xr | Xi] hi
        planes[o2] = ih;
        planes[plane + o1] = __hneg(ih);      // [-Xi | Xr] hi
        planes[plane + o2] = rh;
        planes[2 * plane + o1] = rl;          // lo
        planes[2 * plane + o2] = il;
        planes[3 * plane + o1] = __hneg(il);
        planes[3 * plane + o2] = rl;
    }
}

}  // namespace tmb
