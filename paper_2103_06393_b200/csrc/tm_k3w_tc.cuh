// Batched multi-RHS forward on the W arena ("K3W"), complex64, for large
// right-hand-side counts (config 5: p = 32) of stores whose W arena exists.
//
// The x-in-B forward (tm_kernels_tc.cuh) multiplies every W element into the
// N space i3 x p: r3 * p tensor MACs per voxel and column against the
// reference's r3 + p (reconstruct's mode 3 and the rank-1 update,
// src/matvec.cpp:43-49; 5.4x at config 5).  K3W decompresses each column
// ONCE per tile instead, at the algorithmic cost, with both contractions on
// the tensor cores:
//
//   GEMM1  T_j[row, i3] = sum_r W_j[row, r] U3_j[i3, r]   (K = slots, N = 16)
//   GEMM2  Y[row, i3, :] += sum_j T_j[row, i3] X[j, :]     (K = columns)
//
// Slot stream.  K3W runs on its own copy of the W arena's fp16-split A planes
// (pre-swizzled 16 KB blocks [k][row tile][stage], built once per store):
// columns are packed back to back except that at most two columns overlap a
// K16 stage (a column that would be the third starts the next stage).  Half 0
// of a stage is its first column, which ends in the stage (it may have
// started in the previous one: a straddler), half 1 the second, which may
// continue into the next stage as that stage's half 0; the converters add
// the two partials.
// GEMM1 per stage: A1 = the stage's W planes (one bulk copy), B1 = a
// per-store block-diagonal table ([k][stage][i3 block], 4 fp16 planes of
// 16 n x 16 slots: n = half c x 8 + i3 x 2 + (Tr, Ti) for the column of half
// c; U3 2^-e3 x 2^12 as the fp16 split; bulk-copied) — 4 tcgen05.mma
// (M = 128): D1 = Wr B1a + Wi B1b as hi.hi + hi.lo + lo.hi, the hi planes of
// W against [B hi ; B lo] in one N = 32 MMA each (the hi.lo terms land in
// columns 16-31), into one of 8 TMEM buffers of 32 columns.  Converter warps
// read D1 (tcgen05.ld), scale and split T, and store it 4 columns at a time
// into the A operand of GEMM2 at K position j % 16 (4 M = 128 blocks, one per
// i3 of the tile).  GEMM2: B = X as fp16-split planes [Xr | Xi], [-Xi | Xr]
// (N = 64) by TMA, 6 tcgen05.mma per i3 block per 16 columns, [Yr | Yi] +=
// Tr [Xr | Xi] + Ti [-Xi | Xr]; chained accumulation folded into a per-CTA
// L2 running sum.  The MMA thread issues the GEMM1s of GEMM2 stage kk + 1
// before GEMM2 kk (the tensor pipe runs in order), so the converters fill one
// A stage while GEMM2 runs on the other.
//
// Warp roles (512 threads, 1 CTA / SM, persistent over tiles):
//   warp 0      TMA producer of the X planes (B of GEMM2)
//   warp 1      MMA issuer (GEMM1 per stage, GEMM2 per 16 columns)
//   warp 2      loader of the W stages (A1 and B1 blocks by bulk copy)
//   warp 3      TMEM allocator (512 columns: GEMM2 accumulator 256, D1 8 x 32)
//   warps 4-11  converters (D1 -> A2): lane quarter w & 3, i3 pair (w - 4) >> 2
//   warps 12-15 chain fold + epilogue
#pragma once

#include <cuda_fp16.h>

#include "tm_common.cuh"
#include "tm_kernels_tc.cuh"
#include "tm_sm100.cuh"

namespace tmb {

constexpr int K3_NI3 = 4;                        // i3 per tile (one M = 128 block each)
constexpr int K3_P = 32;                         // right-hand sides per pass (N = 2 K3_P)
constexpr int K3_NST = 2;                        // A/B stages of GEMM2 (16 columns each)
constexpr int K3_A_PLANE = TC_ROWS * 32;         // one plane of one i3 block: 128 rows x 16 fp16
constexpr int K3_A_BLOCK = 4 * K3_A_PLANE;       // re hi, re lo, im hi, im lo
constexpr int K3_A_STAGE = K3_NI3 * K3_A_BLOCK;  // 64 KB
constexpr int K3_B_PLANE = 2 * K3_P * 32;        // 64 rows x 16 fp16
constexpr int K3_B_STAGE = 4 * K3_B_PLANE;       // [Xr|Xi] hi, [-Xi|Xr] hi, [Xr|Xi] lo, [-Xi|Xr] lo
constexpr int K3_YCOLS = K3_NI3 * 2 * K3_P;      // TMEM columns of the GEMM2 accumulator
constexpr int K3_ND1 = 8;                        // D1 (GEMM1 output) TMEM buffers of 32 columns (hi and lo halves)
constexpr int K3_TCOLS = 512;                    // TMEM allocation
constexpr int K3_CI = 2;                         // i3 per converter warp (1: 16 converter warps, measured slower)
constexpr int K3_NCW = 4 * (K3_NI3 / K3_CI);     // converter warps (TMEM lane quarter x i3 group)
constexpr int K3_THREADS = (8 + K3_NCW) * 32;
// W stage: A1 = 4 planes [128 rows][16 slots] fp16 (SW32), then B1 = 4 planes [16 n][16 slots] fp16 (SW32)
constexpr int K3_B1_PLANE = 16 * 32;
constexpr int K3_B1_BYTES = 4 * K3_B1_PLANE;     // 2 KB
constexpr int K3_W_B1 = 4 * K3_A_PLANE;
constexpr int K3_W_STAGE = (K3_W_B1 + K3_B1_BYTES + 1023) / 1024 * 1024;
constexpr int K3_NWS = 4;                        // W stages

struct K3Geom {
    int64_t ncols;
    int n1, n2, n3, q;
    int nt1, nt2, nt3;
    int p;             // right-hand sides of this pass (<= K3_P)
    int64_t ntiles;    // tiles of this launch: tile0 .. tile0 + ntiles - 1
    int64_t tile0;
    int nks;           // GEMM2 K stages per tile = ceil(ncols / 16)
    int chain;         // K stages per TMEM accumulation chain
    float tsc;         // power of two taking D1 (W-arena x U3 units) into fp16 range
    float wsc;         // the W arena's scale x the B1 scale (the epilogue undoes wsc x tsc x sb)
};

struct K3Tile {
    int k, i1_0, i2_0, i3_0;
};

// Tile order: i3 block fastest (the tiles resident together stream the same
// W planes of their row tile through L2), then i2 block, i1 block, component.
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

__device__ __forceinline__ void mbar_arrive_n(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(sm100::smem_u32(bar)), "r"(n) : "memory");
}

__global__ void __launch_bounds__(K3_THREADS, 1)
    fwd_k3w_kernel(const __grid_constant__ CUtensorMap xmap, const unsigned char* __restrict__ patab,
                   const __half* __restrict__ b1tab, const int* __restrict__ kc,
                   const uint32_t* __restrict__ sflag, int64_t nstg, const int* __restrict__ gend, K3Geom g, float2* __restrict__ y, int64_t ldy,
                   float* __restrict__ rsum, const float* __restrict__ xmax) {
    using namespace sm100;
    extern __shared__ __align__(1024) unsigned char k3_smem_raw[];
    unsigned char* sm = k3_smem_raw + ((1024u - (smem_u32(k3_smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = sm;
    unsigned char* sB = sA + K3_NST * K3_A_STAGE;
    unsigned char* sW = sB + K3_NST * K3_B_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sW + K3_NWS * K3_W_STAGE);
    uint64_t* full = bars;              // [K3_NST]  A2 / X stage of GEMM2
    uint64_t* empty = full + K3_NST;    // [K3_NST]
    uint64_t* wfull = empty + K3_NST;   // [K3_NWS]  W stage of GEMM1
    uint64_t* wempty = wfull + K3_NWS;  // [K3_NWS]
    uint64_t* dfull = wempty + K3_NWS;  // [K3_ND1]  D1 buffers
    uint64_t* dempty = dfull + K3_ND1;  // [K3_ND1]
    uint64_t* cfull = dempty + K3_ND1;  // 1
    uint64_t* cfree = cfull + 1;        // 1
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfree + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < K3_NST; ++s) {
            mbar_init(&full[s], 1 + K3_NCW * 16);  // X TMA + every converter warp per column of the stage
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < K3_NWS; ++s) {
            mbar_init(&wfull[s], 1);
            mbar_init(&wempty[s], 1);
        }
        for (int s = 0; s < K3_ND1; ++s) {
            mbar_init(&dfull[s], 1);
            mbar_init(&dempty[s], K3_NCW);  // the stage's converter warps
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
    if (warp == 3) tmem_alloc(tmem_slot, K3_TCOLS);
    if (warp == 0 && lane == 0) tma_prefetch_desc(&xmap);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tD1 = tmem + uint32_t(K3_YCOLS);
    const int64_t tstart = blockIdx.x, tstep = gridDim.x;

    if (warp == 0) {
        // ------------------------------------------------ X-plane TMA producer
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.ntiles; t += tstep)
                for (int kk = 0; kk < g.nks; ++kk) {
                    mbar_wait_backoff(&empty[s], ph ^ 1, 512);
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
            const uint32_t id2 = umma_idesc_f16(TC_ROWS, 2 * K3_P, false, false);
            const uint32_t id1 = umma_idesc_f16(TC_ROWS, 16, false, false);
            const uint32_t id1w = umma_idesc_f16(TC_ROWS, 32, false, false);
            uint32_t s = 0, ph = 0, gch = 0;
            uint32_t sg = 0;  // W stages issued (all tiles): W ring slot sg % K3_NWS, D1 buffer sg % K3_ND1
            const uint64_t wdesc0 = umma_smem_desc(smem_u32(sW), 256, 6);
            const uint64_t adesc0 = umma_smem_desc(smem_u32(sA), 256, 6);
            const uint64_t bdesc0 = umma_smem_desc(smem_u32(sB), 256, 6);
            for (int64_t t = tstart; t < g.ntiles; t += tstep) {
                const K3Tile tl = k3_tile(g, g.tile0 + t);
                // gend[k][kk]: W stages up to the last one holding a column of GEMM2 stage kk
                const int* ge = gend + int64_t(tl.k) * g.nks;
                int snext = 0;
                // GEMM1 of the W stages [snext, lim)
                auto gemm1_until = [&](int lim) {
                    while (snext < lim) {
                        const uint32_t ws = sg % K3_NWS, wph = (sg / K3_NWS) & 1u;
                        const uint32_t db = sg % K3_ND1, dph = (sg / K3_ND1) & 1u;
                        mbar_wait(&wfull[ws], wph);
                        mbar_wait(&dempty[db], dph ^ 1u);
                        tc_fence_after();
                        // descriptors: the start-address field is addr >> 4 (< 2^14 for shared
                        // memory), so an offset is a plain add to the slot's base descriptor
                        const uint64_t Arh = wdesc0 + uint64_t(ws) * (K3_W_STAGE >> 4);
                        const uint64_t Arl = Arh + (K3_A_PLANE >> 4);
                        const uint64_t Aih = Arh + (2 * K3_A_PLANE >> 4);
                        const uint64_t Ail = Arh + (3 * K3_A_PLANE >> 4);
                        const uint64_t Bah = Arh + (K3_W_B1 >> 4);
                        const uint64_t Bbh = Bah + (2 * K3_B1_PLANE >> 4);
                        const uint32_t d = tD1 + db * 32u;
                        // D1 = Wr B1a + Wi B1b (Tr = Wr U3r - Wi U3i, Ti = Wr U3i + Wi U3r in B1's
                        // columns): the hi planes of A meet [B hi ; B lo] in one N = 32 MMA (columns
                        // 16-31 take the hi.lo terms; the converters add the halves), so each A
                        // plane is read once
                        mma_f16(d, Arh, Bah, id1w, 0);
                        mma_f16(d, Arl, Bah, id1, 1);
                        mma_f16(d, Aih, Bbh, id1w, 1);
                        mma_f16(d, Ail, Bbh, id1, 1);
                        mma_commit(&wempty[ws]);
                        mma_commit(&dfull[db]);
                        ++snext;
                        ++sg;
                    }
                };
                int cpos = 0;
                const int last = g.nks - 1;
                int gnext = ge[min(1, last)];  // gend one GEMM2 stage ahead, loaded a stage early
                for (int kk = 0; kk < g.nks; ++kk) {
                    const int need = gnext;
                    gnext = ge[min(kk + 2, last)];
                    // GEMM1 of every W stage holding a column of GEMM2 stages kk and kk + 1,
                    // issued before GEMM2 kk: the tensor pipe runs in order, so the converters
                    // fill stage kk + 1 while GEMM2 kk executes (the A ring holds two stages)
                    gemm1_until(need);
                    if (cpos == 0) {
                        mbar_wait(cfree, (gch & 1) ^ 1);  // the previous chain has been folded
                        tc_fence_after();
                    }
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t Bah = bdesc0 + uint64_t(s) * (K3_B_STAGE >> 4);
                    const uint64_t Bbh = Bah + (K3_B_PLANE >> 4);
                    const uint64_t Bal = Bah + (2 * K3_B_PLANE >> 4);
                    const uint64_t Bbl = Bah + (3 * K3_B_PLANE >> 4);
                    const uint32_t acc = cpos > 0 ? 1u : 0u;
#pragma unroll
                    for (int l = 0; l < K3_NI3; ++l) {
                        const uint64_t Arh = adesc0 + uint64_t(s) * (K3_A_STAGE >> 4) + uint64_t(l) * (K3_A_BLOCK >> 4);
                        const uint64_t Arl = Arh + (K3_A_PLANE >> 4);
                        const uint64_t Aih = Arh + (2 * K3_A_PLANE >> 4);
                        const uint64_t Ail = Arh + (3 * K3_A_PLANE >> 4);
                        const uint32_t d = tmem + uint32_t(l * 2 * K3_P);
                        // [Yr | Yi] += Tr [Xr | Xi] + Ti [-Xi | Xr], each as hi.hi + hi.lo + lo.hi
                        mma_f16(d, Arh, Bah, id2, acc);
                        mma_f16(d, Arh, Bal, id2, 1);
                        mma_f16(d, Arl, Bah, id2, 1);
                        mma_f16(d, Aih, Bbh, id2, 1);
                        mma_f16(d, Aih, Bbl, id2, 1);
                        mma_f16(d, Ail, Bbh, id2, 1);
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
        // ------------------------------------------------ W-stage loader
        if (elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.ntiles; t += tstep) {
                const K3Tile tl = k3_tile(g, g.tile0 + t);
                const int nws = (kc[tl.k] + 15) >> 4;
                const int rt = (tl.i1_0 / TC_TI1) * g.nt2 + tl.i2_0 / TC_TI2;  // row tile
                const unsigned char* pa = patab + (int64_t(tl.k) * g.nt1 * g.nt2 + rt) * nstg * (4 * K3_A_PLANE);
                const __half* b1 = b1tab + ((int64_t(tl.k) * nstg) * g.nt3 + tl.i3_0 / K3_NI3) * (K3_B1_BYTES / 2);
                for (int kk = 0; kk < nws; ++kk) {
                    mbar_wait_backoff(&wempty[s], ph ^ 1, 128);
                    mbar_arrive_expect_tx(&wfull[s], uint32_t(4 * K3_A_PLANE + K3_B1_BYTES));
                    unsigned char* dst = sW + s * K3_W_STAGE;
                    bulk_g2s(dst, pa + int64_t(kk) * (4 * K3_A_PLANE), uint32_t(4 * K3_A_PLANE), &wfull[s]);
                    bulk_g2s(dst + K3_W_B1, b1 + int64_t(kk) * g.nt3 * (K3_B1_BYTES / 2), uint32_t(K3_B1_BYTES),
                             &wfull[s]);
                    if (++s == K3_NWS) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp >= TC_PW0 && warp < TC_PW0 + K3_NCW) {
        // ------------------------------------------------------- converters
        // every converter warp takes every W stage: warp w reads TMEM lane quarter
        // w & 3 (row = i2 + 32 i1 of the tile) and converts the i3 pair 2 grp,
        // 2 grp + 1 (grp = (w - 4) >> 2); completed columns are buffered in
        // registers and stored 4 K positions at a time (one 64-bit store per
        // i3 and plane)
        const int grp = (warp - TC_PW0) >> 2, quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t rowbase = uint32_t(row) * 32u, xorv = (uint32_t(row) & 4u) << 2;
        const uint32_t lane_addr = (uint32_t(quarter * 32) << 16) + uint32_t(2 * K3_CI * grp);
        const float tsc = g.tsc;
        uint32_t sg = 0;       // W stages of all tiles so far
        uint32_t tseq = 0;     // tiles so far: GEMM2 stage sequence = tseq nks + j / 16
        // [i3 of the pair][plane]: a shift register of the last 4 columns' fp16 values
        // (ba: the older two, bb: the newer two; a new column enters at the top of bb)
        uint32_t ba[K3_CI][4], bb[K3_CI][4];
#pragma unroll
        for (int l = 0; l < K3_CI; ++l)
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) ba[l][pl] = bb[l][pl] = 0u;
        for (int64_t t = tstart; t < g.ntiles; t += tstep, ++tseq) {
            const K3Tile tl = k3_tile(g, g.tile0 + t);
            const int nws = (kc[tl.k] + 15) >> 4;
            const uint32_t* fl = sflag + int64_t(tl.k) * nstg;
            int j = 0;           // next column to complete
            uint32_t fnext = fl[0];
            // D1 of stage kk is loaded while stage kk - 1 is converted (software pipelining);
            // this warp's columns: half c at 8 c + 2 K3_CI grp + (2 l + part), the hi.lo terms
            // at + 16; cur = [half 0 | half 1 | half 0 hi.lo | half 1 hi.lo], NW words each
            constexpr int NW = 2 * K3_CI;
            uint32_t cur[4 * NW];
            auto load_d1 = [&](uint32_t sgx) {
                const uint32_t dbx = sgx % K3_ND1;
                mbar_wait(&dfull[dbx], (sgx / K3_ND1) & 1u);
                tc_fence_after();
                const uint32_t ta = tD1 + lane_addr + dbx * 32u;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {  // columns + 0, 8, 16, 24
                    if constexpr (NW == 4)
                        tmem_ld4(ta + 8u * q4, *reinterpret_cast<uint32_t(*)[4]>(&cur[NW * q4]));
                    else
                        tmem_ld2(ta + 8u * q4, *reinterpret_cast<uint32_t(*)[2]>(&cur[NW * q4]));
                }
            };
            load_d1(sg);
            float t1prev[NW] = {};  // the previous stage's half 1 (a straddler's head)
            for (int kk = 0; kk < nws; ++kk, ++sg) {
                const uint32_t f = fnext;
                if (kk + 1 < nws) fnext = fl[kk + 1];
                tmem_ld_wait_regs(cur);
                float t0[NW], t1[NW];
#pragma unroll
                for (int e = 0; e < NW; ++e) {
                    t0[e] = __uint_as_float(cur[e]) + __uint_as_float(cur[2 * NW + e]);
                    t1[e] = __uint_as_float(cur[NW + e]) + __uint_as_float(cur[3 * NW + e]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&dempty[sg % K3_ND1]);
                if (kk + 1 < nws) load_d1(sg + 1);
                if (f & 4u) {
                    // half 0 continues the previous stage's half 1 (a column straddling the boundary)
#pragma unroll
                    for (int e = 0; e < NW; ++e) t0[e] += t1prev[e];
                }
#pragma unroll
                for (int e = 0; e < NW; ++e) t1prev[e] = t1[e];
                const int nc = 1 + ((f & 3u) == 3u ? 1 : 0);  // columns ending here: half 0, half 1 if it ends
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (c >= nc) break;
                    const float* tv = c ? t1 : t0;
                    const uint32_t ks = uint32_t(j) & 15u, sub = ks & 3u;
#pragma unroll
                    for (int l = 0; l < K3_CI; ++l) {
                        uint32_t hi, lo;
                        f16_split2(f2_pack(tv[2 * l] * tsc, tv[2 * l + 1] * tsc), hi, lo);
                        // shift in: (ba, bb) <- (ba.hi16 bb.lo16, bb.hi16 new)
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) ba[l][pl] = __byte_perm(ba[l][pl], bb[l][pl], 0x5432);
                        bb[l][0] = __byte_perm(bb[l][0], hi, 0x5432);  // re hi
                        bb[l][1] = __byte_perm(bb[l][1], lo, 0x5432);  // re lo
                        bb[l][2] = __byte_perm(bb[l][2], hi, 0x7632);  // im hi
                        bb[l][3] = __byte_perm(bb[l][3], lo, 0x7632);  // im lo
                    }
                    const bool last = j == int(g.ncols) - 1;
                    if (sub == 3u || last) {
                        // flush K positions ks & ~3 .. ks into the GEMM2 stage of column j
                        const uint32_t aseq = tseq * uint32_t(g.nks) + uint32_t(j >> 4);
                        const uint32_t as = aseq % K3_NST, aph = (aseq / K3_NST) & 1u;
                        mbar_wait(&empty[as], aph ^ 1u);
                        unsigned char* st = sA + as * K3_A_STAGE + rowbase + (((ks & ~3u) * 2u) ^ xorv);
                        // the register holds columns (ks & ~3) .. ks in its top sub + 1 positions
                        const uint32_t drop = 16u * (3u - sub);
#pragma unroll
                        for (int l = 0; l < K3_CI; ++l)
#pragma unroll
                            for (int pl = 0; pl < 4; ++pl) {
                                uint64_t v64 = (uint64_t(bb[l][pl]) << 32) | ba[l][pl];
                                if (drop) v64 >>= drop;  // a tile's last, partial group
                                *reinterpret_cast<uint64_t*>(st + (K3_CI * grp + l) * K3_A_BLOCK + pl * K3_A_PLANE) = v64;
                            }
                        fence_proxy_async_smem();
                        __syncwarp();
                        // a tile's last column also stands in for the missing columns of its stage
                        if (lane == 0) mbar_arrive_n(&full[as], last ? 16u - (ks & ~3u) : 4u);
                    }
                    ++j;
                }
            }
        }
    } else if (warp >= TC_PW0 + K3_NCW) {
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
        // exact power of two (W-arena scale x T scale x X scale)
        const float inv = 1.f / (g.wsc * g.tsc * fp16_scale(*xmax));
        uint32_t gch = 0;
        for (int64_t t = tstart; t < g.ntiles; t += tstep) {
            const K3Tile tl = k3_tile(g, g.tile0 + t);
            const int ei1 = tl.i1_0 + quarter, ei2 = tl.i2_0 + lane;
            const bool eok = ei1 < g.n1 && ei2 < g.n2;
            for (int ch = 0; ch < nch; ++ch, ++gch) {
                mbar_wait_backoff(cfull, gch & 1, 1024);
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
                            float2* yp = y + int64_t(tl.k) * nv3 + ei1 +
                                         int64_t(g.n1) * (ei2 + int64_t(g.n2) * (tl.i3_0 + l));
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
                                if (ch > 0) {
                                    ar = rr[int64_t(m) * TC_ROWS];
                                    ai = ri[int64_t(m) * TC_ROWS];
                                }
                                const float re[4] = {__uint_as_float(cr[4 * m]) + ar.x,
                                                     __uint_as_float(cr[4 * m + 1]) + ar.y,
                                                     __uint_as_float(cr[4 * m + 2]) + ar.z,
                                                     __uint_as_float(cr[4 * m + 3]) + ar.w};
                                const float im[4] = {__uint_as_float(ci[4 * m]) + ai.x,
                                                     __uint_as_float(ci[4 * m + 1]) + ai.y,
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
    if (warp == 3) tmem_dealloc(tmem, K3_TCOLS);
}

// X planes of a pass (B of GEMM2): [4][2 K3_P rows n][kpad columns j] fp16,
// plane 0 = [Xr | Xi] hi, 1 = [-Xi | Xr] hi, 2 / 3 the same lo; row n < K3_P
// is right-hand side n's real-part row, n >= K3_P its imaginary-part row;
// rows of right-hand sides >= p and columns >= m are zero.  sb =
// fp16_scale(max|x|).
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

// Per-store tables of K3W (built on first use, tm_capi.cu ensure_k3w) on
// K3W's padded slot stream (column j of component k at slot poff[t], t = k m
// + j, taking 8 slots if r3 <= 8 else 16; a stage holds one or two columns):
//   pa[k][row tile][stage][plane][128 rows x 32 B] — the W arena's four fp16
//     planes on K3W's slot stream, each (row tile, stage) block one
//     contiguous 16 KB A operand, pre-swizzled for SW32 K-major (byte row 32
//     + ((slot 2) ^ ((row & 4) << 2))), loaded by one bulk copy
//     (build_k3w_pa_kernel; padding zero by the caller's memset);
//   b1[k][stage][i3 block][4 planes][16 n][16 slots] — GEMM1's B operand,
//     pre-swizzled for SW32 K-major (byte n 32 + ((slot 2) ^ ((n & 4) << 2))):
//     n = c 8 + l 2 + part for the column of half c (stage desc sd: the
//     tensor of half 0 / half 1, -1 if none; a column's slot r sits at stage
//     slot poff - 16 stage + r, so a straddler's slots are split between the
//     two stages' tables), i3 = 4 block + l, part 0 = Tr, 1 = Ti; planes B1a
//     hi / lo, B1b hi / lo with (B1a, B1b) = (U3r, -U3i) for Tr and (U3i,
//     U3r) for Ti, U3 = U3_t[i3, r] 2^-e3 2^12 (build_k3w_b1_kernel).
__global__ void build_k3w_pa_kernel(const TDesc* __restrict__ td, const int* __restrict__ kofs,
                                    const int* __restrict__ poff, int64_t ncols, int q, const __half* __restrict__ wa,
                                    int64_t rows_pad, int64_t kpad, int64_t nstg, unsigned char* __restrict__ pa) {
    const int64_t t = blockIdx.x;
    const int k = int(t / ncols);
    const int r3 = td[t].r3;
    const int64_t k0 = kofs[t], p0 = poff[t];
    const int64_t plane = int64_t(q) * rows_pad * kpad, nrt = rows_pad / TC_ROWS;
    for (int64_t e = threadIdx.x; e < rows_pad * r3; e += blockDim.x) {
        const int64_t row = e / r3;
        const int r = int(e - row * r3);
        const int64_t src = (int64_t(k) * rows_pad + row) * kpad + k0 + r;
        const int64_t slot = p0 + r, rt = row / TC_ROWS;
        const uint32_t rr = uint32_t(row % TC_ROWS), sl = uint32_t(slot % 16);
        unsigned char* blk = pa + ((int64_t(k) * nrt + rt) * nstg + slot / 16) * (4 * K3_A_PLANE);
        const uint32_t off = rr * 32u + ((sl * 2u) ^ ((rr & 4u) << 2));
#pragma unroll
        for (int pl = 0; pl < 4; ++pl)
            *reinterpret_cast<__half*>(blk + pl * K3_A_PLANE + off) = wa[pl * plane + src];
    }
}

__global__ void build_k3w_b1_kernel(const TDesc* __restrict__ td, const TcDesc* __restrict__ tcd,
                                    const float2* __restrict__ arena, const int2* __restrict__ sd,
                                    const int* __restrict__ poff, int n3, int nt3, int64_t nstg,
                                    __half* __restrict__ b1) {
    const int64_t blk = blockIdx.x;  // (k stage) nt3 + i3 block
    const int ib = int(blk % nt3);
    const int64_t ks = blk / nt3;    // k nstg + stage
    const int n = threadIdx.x >> 4, slot = threadIdx.x & 15;
    const int c = n >> 3, l = (n >> 1) & 3, part = n & 1;
    const int2 d2 = sd[ks];
    const int t = c ? d2.y : d2.x;
    float a = 0.f, b = 0.f;
    if (t >= 0) {
        const int64_t st0 = (ks % nstg) * 16;
        const int r = slot + int(st0) - poff[t];  // the column's slot index
        const int i3 = ib * K3_NI3 + l;
        const TDesc d = td[t];
        if (r >= 0 && r < d.r3 && i3 < n3) {
            const float2 u = arena[d.off_u3 + int64_t(i3) * d.r3 + r];
            const float sc = ldexpf(TC_U3_SCALE, -fexp_e3(tcd[t].fexp));
            a = (part ? u.y : u.x) * sc;
            b = (part ? u.x : -u.y) * sc;
        }
    }
    const __half ah = __float2half_rn(a), bh = __float2half_rn(b);
    const __half al = __float2half_rn(a - __half2float(ah)), bl = __float2half_rn(b - __half2float(bh));
    unsigned char* o = reinterpret_cast<unsigned char*>(b1 + blk * (K3_B1_BYTES / 2));
    const uint32_t off = uint32_t(n) * 32u + ((uint32_t(slot) * 2u) ^ ((uint32_t(n) & 4u) << 2));
    *reinterpret_cast<__half*>(o + off) = ah;
    *reinterpret_cast<__half*>(o + K3_B1_PLANE + off) = al;
    *reinterpret_cast<__half*>(o + 2 * K3_B1_PLANE + off) = bh;
    *reinterpret_cast<__half*>(o + 3 * K3_B1_PLANE + off) = bl;
}

}  // namespace tmb
