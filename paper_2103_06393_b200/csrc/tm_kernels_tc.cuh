// Tensor-core (tcgen05, kind::f16, 2-term fp16 split) forward kernel, complex64.
//
// Forward of component k, for one output tile of ROWS = 128 voxel rows
// (TI1 x TI2 = 4 x 32 of (i1, i2)) times up to 2 x 128 rows of the N space
// n = i3 * p + c (voxels along mode 3 times the right-hand sides of the pass):
//
//   Y[row, n] = sum_j sum_r W_j[row, r] B_j[n, r],
//   W_j[row, r] = sum_b V_j[i1, b, r] U2_j[i2, b],   V_j = U1_j x_1 G_j,
//   B_j[i3 p + c, r] = x[j, c] U3_j[i3, r],
//
// i.e. one GEMM with K = the packed (j, r) stream of component k
// (K = sum_j r3_j, no per-column padding) — the reference's stacked_forward
// (src/matvec.cpp:17-65) with reconstruct's mode products (src/tensor.cpp:
// 89-120,176-181) restricted to the tile and the rank-1 updates folded into
// B.  B is built per call (build_xb_kernel) as a scaled 2-term fp16 split
// in four planes {Re hi, Im hi, Re lo, Im lo} [plane][k][n][K] and streamed
// by TMA (SWIZZLE_32B, 16 K per stage).  The mode-1 products V_j are formed
// once per store (build_v_kernel).  The A operand W is produced on the fly
// by 8 producer warps (FFMA2 mode-2 products, scaled into fp16 range) into
// the same four-plane split in shared memory, so no decompressed column is
// ever written anywhere; with p > 1 one W serves every right-hand side.
// Per 16-wide K step the MMA warp issues 12 tcgen05.mma of N = 256:
//   Yr += Ar.Br - Ai.Bi,  Yi += Ar.Bi + Ai.Br,  each product as
//   hi.hi + hi.lo + lo.hi and the minus sign via the idesc negate-A bit.
// PAIR: clusters of 2 CTAs run M = 256 cta_group::2 MMAs over two i1
// blocks, each CTA holding half of the tile's N rows of B.
//
// Accuracy: the tensor core's fp32 accumulate truncates, so one TMEM
// accumulator over the whole K stream (~45 000 terms per component at
// config 4) drifts toward zero linearly in K.  The K stream
// is therefore cut into chains of `chain` stages: each chain accumulates
// from zero in TMEM and is then folded (round-to-nearest fp32 adds) by 4
// dedicated fold warps into a running sum held in a per-CTA scratch in
// global memory (L2-resident, [i3][row] so the fold is coalesced; the CTA
// owns its tile, so the fold is deterministic); the tile's last chain is
// added to the running sum on its way to y.  The error is then set by the
// chain length, not by K.  All 512 TMEM columns hold [Yr|Yi] of the 256-row
// N span, so each produced W element feeds 256 columns of MMA work.
//
// Warp roles (512 threads, 1 CTA / SM, persistent over tiles):
//   warp 0      TMA producer of the B planes
//   warp 1      MMA issuer (one elected thread; the even CTA of a pair)
//   warp 2      factor loader: per column, bulk-copies {TcDesc, V rows,
//               U2 rows} of the tile into a 3-deep shared-memory ring
//   warp 3      TMEM allocator
//   warps 4-11  A producers (mode-2 W, scale, hi/lo split)
//   warps 12-15 chain fold + epilogue (TMEM -> registers -> y)
// Pipelines: A/B stage ring (full: 1 TMA arrive+tx + the producer-warp
// arrivals of both CTAs; empty: tcgen05.commit), factor ring (full:
// bulk-copy tx; empty: 8 producer warps), chain (full: commit after the
// chain's last K step; free: the fold warps of both CTAs).
#pragma once

#include <cuda_fp16.h>

#include "tm_common.cuh"
#include "tm_sm100.cuh"

namespace tmb {

// fp16 operand scaling (see also tm_adj_tc.cuh): operands are stored as a
// 2-term fp16 split (hi = fp16(v), lo = fp16(v - hi): 22 significant bits)
// of values scaled by powers of two into fp16's normal range — U3
// (orthonormal columns, |u| <= 1) by 2^12, data-dependent operands by
// 2^(14 - e) where 2^e bounds their magnitude (fp16_scale).  The products
// hi.hi + hi.lo + lo.hi run on tcgen05.mma.kind::f16 (K = 16) with fp32
// accumulation; the scale is undone exactly on the fp32 results.
constexpr float TC_U3_SCALE = 4096.f;
__host__ __device__ inline float fp16_scale(float amax) {
    if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
    int e = 0;
    frexpf(amax, &e);  // amax < 2^e
    e = e < -100 ? -100 : (e > 100 ? 100 : e);
    return ldexpf(1.f, 14 - e);
}

constexpr int TC_TI1 = 4, TC_TI2 = 32, TC_ROWS = 128;
// Back-off (ns between barrier polls) of the warp roles that wait off the
// critical path — the B-plane TMA warp, the factor loader and the chain fold —
// so that their polling takes fewer issue slots from the producer / consumer
// warps sharing their SM sub-partitions.
#ifndef TC_BACKOFF_TMA
#define TC_BACKOFF_TMA 128
#endif
#ifndef TC_BACKOFF_LD
#define TC_BACKOFF_LD 128
#endif
#ifndef TC_BACKOFF_FOLD
#define TC_BACKOFF_FOLD 256
#endif
#ifndef TC_BACKOFF_ADJ
#define TC_BACKOFF_ADJ 64
#endif
constexpr int TC_NST_MAX = 6;   // A/B stages (16 K each; as many as shared memory allows)
constexpr int TC_JR = 3;        // factor-ring slots
constexpr int TC_NR = 2;        // tile rows per producer lane (rows i2a + 8 e, e < TC_NR)
constexpr int TC_NPW = 16 / TC_NR;  // producer warps: 4 i1 rows x (4 / TC_NR) blocks of 8 TC_NR i2
constexpr int TC_NH = 4;        // c partition across lanes: c = 4 u + (lane & 3)
constexpr int TC_PW0 = 4;       // first producer warp
constexpr int TC_FW0 = TC_PW0 + TC_NPW;   // first fold / epilogue warp
constexpr int TC_THREADS = (TC_FW0 + 4) * 32;
constexpr int TC_NMAX = 128;    // i3 per tile (N per MMA)
constexpr int TC_RMAX = 32;     // rank bound of the tensor-core path (forward: up to 3 A stages per column)
constexpr int TC_A_PLANE = TC_ROWS * 32;     // bytes (128 rows x 16 fp16 = one K16 stage)
constexpr int TC_A_STAGE = 4 * TC_A_PLANE;   // 16 KB
constexpr uint32_t TC_RUN_COL = 256;         // TMEM column of the running sum
constexpr int TC_SLOT_V = 128;               // byte offset of the V block in a factor slot
constexpr int TC_BPLANES = 6;                // adjoint B planes in HBM: [-U3i, U3r, U3i] x {hi, lo}
constexpr int TC_FPLANES = 4;                // forward B planes: [Br, Bi] x {hi, lo}

// Per-tensor descriptor of the tensor-core forward (component-major like
// TDesc).  off_v: float2 offset of the tensor's mode-1 product
// V = U1 x_1 G in the V arena, laid out [i1/4][c + r3 b][i1 % 4] (c innermost:
// the four consecutive c of one producer warp's lanes are bank-conflict
// free for every r2); off_u2:
// float2 offset of the tensor's U2 copy in the U2 arena, n2 rounded up to
// TI2 rows (zero rows past n2) with an odd row stride r2 | 1 (conflict-free
// 32-lane row loads); pad0: the (j, c) slot of the column inside its
// adjoint chunk.
struct TcDesc {
    int64_t off_v;
    int64_t off_u2;
    int64_t off_u3;  // float2 offset of U3t (n3 x r3 row-major) in the store arena
    int32_t r2, r3, pad0, pad1, pad2;
    int32_t fexp;    // factor normalisation exponents (factor_scale_kernel): e2 in bits 0-7, e3 in 8-15 (signed)
};
__host__ __device__ inline int fexp_e2(int32_t f) { return int(int8_t(f & 0xff)); }
__host__ __device__ inline int fexp_e3(int32_t f) { return int(int8_t((f >> 8) & 0xff)); }
static_assert(sizeof(TcDesc) % 16 == 0, "TcDesc is bulk-copied (16-byte granularity)");

struct TcGeom {
    int64_t ncols;
    int n1, n2, n3, q;
    int nt1, nt2, nt3;
    int nmma;       // i3 per half tile = N of the narrow MMAs (multiple of 16, <= 128)
    int nh3;        // i3 halves per tile (1 or 2): a tile spans nh3 * nmma voxels along mode 3
    int p;          // right-hand sides of this pass (B rows n = i3 * p + c)
    int nt;         // B rows = n3 * p: the N space the tiles span (nt3 tiles of nmma * nh3 rows)
    float wsc;      // fp16 scale of W (power of two from the store's max vbound)
    int64_t ntiles;
    int rmax2, rmax3;
    int slot_bytes;             // factor slot size (multiple of 128)
    int u2_off;                 // byte offset of the U2 rows in a slot
    int b_stage;                // bytes of one B stage (4 planes x nmma x 32)
    int nst;                    // A/B stages in the ring (3..TC_NST_MAX)
    int chain;                  // K stages per TMEM accumulation chain
    int debug;                  // diagnostics (TMB_TC_DEBUG): 1 = no mode-2 work, 2 = no B loads
    int pair;                   // 1: CTA-pair kernel (cta_group::2, M = 256), nt1 counts pairs of i1 blocks
    int64_t gslots;             // ADJ: slots per component in the G buffer ([k][n][slot])
    unsigned long long* prof;   // diagnostics (TMB_TC_DEBUG & 8, builds with -DTMB_TC_PROFILE): per-role wait cycles
    int split;                  // work items per tile in this launch (column ranges; > 1 only in a final
                                // partial wave, whose items write partial tiles to ypart)
    int64_t tile0;              // first tile of the launch: item t = tile tile0 + t / split, part t % split
    float2* ypart;              // split > 1: [item][rank][span][128 rows] partial results (scaled)
    int64_t t_begin, t_end;     // tile range of this launch (one wave: see run_forward_tc)
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sm100::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(sm100::smem_u32(bar))
        : "memory");
}

__host__ __device__ inline uint32_t round16(uint32_t b) { return (b + 15u) & ~15u; }

// Barrier wait, timed into `acc` (cycles) when the wait profile is on.  The
// profile is compiled in only with -DTMB_TC_PROFILE (then TMB_TC_DEBUG=8
// prints it): even disabled, the timing branches cost several percent in
// the producer warps (measured).
#ifdef TMB_TC_PROFILE
#define TC_TWAIT(on, acc, call)                  \
    do {                                         \
        if (on) {                                \
            const long long t0_ = clock64();     \
            call;                                \
            (acc) += uint64_t(clock64() - t0_);  \
        } else {                                 \
            call;                                \
        }                                        \
    } while (0)
#else
#define TC_TWAIT(on, acc, call) \
    do {                        \
        call;                   \
    } while (0)
#endif

struct TcTile {
    int c, k, i1_0, i2_0, i3_0;
    int part;  // column-range part of the tile (of g.split)
};

// Tile order: i3 block fastest, then i2 block, then i1 block, component,
// right-hand side.  The CTAs resident at one time then share the V rows
// of their i1 block (read by all n2/TI2 x n3/NMMA tiles of that block —
// re-reading them from HBM per tile would cost ~200 GB per config-4
// forward) and stream the same B planes of component k through L2.
__host__ __device__ inline TcTile tc_tile(const TcGeom& g, int64_t item, uint32_t rank = 0) {
    const int64_t t = g.tile0 + item / g.split;
    TcTile r;
    r.part = int(item % g.split);
    r.c = 0;  // the right-hand sides live in the N space (B rows n = i3 * p + c)
    int64_t rem = t;
    const int64_t per_k = int64_t(g.nt3) * g.nt2 * g.nt1;
    r.k = int(rem / per_k);
    rem -= int64_t(r.k) * per_k;
    const int t1 = int(rem / (int64_t(g.nt2) * g.nt3));
    rem -= int64_t(t1) * g.nt2 * g.nt3;
    const int t2 = int(rem / g.nt3);
    const int t3 = int(rem - int64_t(t2) * g.nt3);
    r.i1_0 = (t1 * (1 + g.pair) + int(rank)) * TC_TI1;  // a pair tile spans 2 i1 blocks, one per CTA
    r.i2_0 = t2 * TC_TI2;
    r.i3_0 = t3 * g.nmma * g.nh3;
    return r;
}

// Column range [j0, j1) of a work item and its packed-K range [ka, kb) in
// the component's K stream (kofs: component-major K offsets, kc: K per
// component); the item runs stages [ka / 16, ceil(kb / 16)).  WA (the
// W-arena forward): parts are cut at stage boundaries instead (j0 / j1 unused).
template <bool WA = false>
__device__ __forceinline__ void tc_range(const TcGeom& g, const TcTile& tl, const int* __restrict__ kofs,
                                         const int* __restrict__ kc, int& j0, int& j1, uint32_t& ka, uint32_t& kb) {
    if (WA && g.split > 1) {
        const uint32_t kk = uint32_t(kc[tl.k]), ns = (kk + 15u) >> 4;
        const uint32_t s0 = uint32_t(uint64_t(ns) * tl.part / g.split);
        const uint32_t s1 = uint32_t(uint64_t(ns) * (tl.part + 1) / g.split);
        j0 = j1 = 0;
        ka = s0 * 16u;
        kb = s1 == ns ? kk : s1 * 16u;
        return;
    }
    if (g.split == 1) {  // the common case: the whole column stream
        j0 = 0;
        j1 = int(g.ncols);
        ka = 0u;
        kb = uint32_t(kc[tl.k]);
        return;
    }
    j0 = int(g.ncols * tl.part / g.split);
    j1 = int(g.ncols * (tl.part + 1) / g.split);
    ka = j0 == 0 ? 0u : uint32_t(kofs[int64_t(tl.k) * g.ncols + j0]);
    kb = j1 == int(g.ncols) ? uint32_t(kc[tl.k]) : uint32_t(kofs[int64_t(tl.k) * g.ncols + j1]);
}

// Producer-side state of the A stage ring: the current (open) stage's ring
// slot and phase, and the next free K position inside it.
struct ARing {
    uint32_t st, ph, kpos;
};

// Ring slot / phase `i` stages ahead of the current one (i < nst).
__device__ __forceinline__ void ring_ahead(const ARing& r, uint32_t i, uint32_t nst, uint32_t& s, uint32_t& ph) {
    s = r.st + i;
    ph = r.ph;
    if (s >= nst) {
        s -= nst;
        ph ^= 1u;
    }
}

// One column of one tile for the producer thread: two tile rows (i2a, i2a + 8
// of the warp's i1) and the c values c = 4u + hq.  Mode 2:
// W[row, c] = x_j sum_b V[i1, b, c] U2[i2, b] (FFMA2, V shared by the two
// rows, U2 by the NU values of c), then the scaled fp16 hi/lo split of W
// into its K slots of the A ring.  A warp's 2-byte plane stores cover 8 rows
// x 4 consecutive K slots (8 bytes of each 32-byte K-major row, swizzled):
// conflict-free, one wavefront.  NU = ceil(r3/4) <= 8 (r3 <= TC_RMAX = 32).
template <int NU, bool PAIR>
__device__ __forceinline__ void tc_produce_column(const float2* __restrict__ V, const float2* __restrict__ U2, int r2,
                                                  int ld2, int r3, int hq, int i2a, float wsc, uint64_t* fempty_s,
                                                  uint64_t* empty, uint64_t* full, unsigned char* sA,
                                                  const uint32_t (&rowbase)[TC_NR], const uint32_t (&xorv)[TC_NR],
                                                  int lane, uint32_t nst, ARing& ring) {
    using namespace sm100;
    uint64_t w[TC_NR][NU];
#pragma unroll
    for (int e = 0; e < TC_NR; ++e)
#pragma unroll
        for (int u = 0; u < NU; ++u) w[e][u] = 0;
    // V[(c + r3 b) * 4 + il]: c = 4u + hq  ->  stride 16 float2 per u, 4 r3 per b.
    // Every lane computes all NU values: for c >= r3 the loads read
    // neighbouring V entries (or the slot's U2 rows past the V block — at
    // most 12 float2 beyond it, inside the slot) and the products are never
    // stored, so the inner loop carries no predicates.
    const float2* vp = V + 4 * hq;
    const int vstep = 4 * r3;
    const float2* pu[TC_NR];
#pragma unroll
    for (int e = 0; e < TC_NR; ++e) pu[e] = U2 + (i2a + 8 * e) * ld2;
#pragma unroll 4
    for (int b = 0; b < r2; ++b) {
        float2 ue[TC_NR];
#pragma unroll
        for (int e = 0; e < TC_NR; ++e) ue[e] = *pu[e]++;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const float2 v = vp[16 * u];
#pragma unroll
            for (int e = 0; e < TC_NR; ++e) cfma2v(w[e][u], v, ue[e]);
        }
        vp += vstep;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(fempty_s);  // this warp no longer reads the slot
    // W x wsc (x_j lives in the B operand: build_xb_kernel)
    const uint64_t sc2 = f2_pack(wsc, wsc);
#pragma unroll
    for (int e = 0; e < TC_NR; ++e)
#pragma unroll
        for (int u = 0; u < NU; ++u) asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(w[e][u]) : "l"(sc2));
    // wait for every stage (16 K) this column opens: kpos + r3 <= 15 + 32,
    // so at most three (two while r3 <= 16); the ring holds nst >= 3 stages
    const uint32_t kend = ring.kpos + uint32_t(r3);
    if (ring.kpos == 0) mbar_wait(&empty[ring.st], ring.ph ^ 1u);
    uint32_t s1, ph1, s2, ph2;
    ring_ahead(ring, 1, nst, s1, ph1);
    ring_ahead(ring, 2, nst, s2, ph2);
    if (kend > 16) mbar_wait(&empty[s1], ph1 ^ 1u);
    if (NU > 4 && kend > 32) mbar_wait(&empty[s2], ph2 ^ 1u);
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int c = TC_NH * u + hq;
        if (u < NU - 1 || c < r3) {
            const uint32_t K = ring.kpos + uint32_t(c);
            const uint32_t s = K < 16 ? ring.st : (NU <= 4 || K < 32 ? s1 : s2);
            unsigned char* st = sA + s * TC_A_STAGE;
#pragma unroll
            for (int e = 0; e < TC_NR; ++e) {
                uint32_t hi, lo;
                f16_split2(w[e][u], hi, lo);
                unsigned short* a = reinterpret_cast<unsigned short*>(st + rowbase[e] + (((K & 15u) * 2u) ^ xorv[e]));
                a[0] = static_cast<unsigned short>(hi);                      // Re hi
                a[TC_A_PLANE / 2] = static_cast<unsigned short>(lo);         // Re lo
                a[2 * TC_A_PLANE / 2] = static_cast<unsigned short>(hi >> 16);  // Im hi
                a[3 * TC_A_PLANE / 2] = static_cast<unsigned short>(lo >> 16);  // Im lo
            }
        }
    }
    if (kend >= 16) {  // the current stage is complete (and with r3 > 16 maybe the next one too)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            if (PAIR) {
                mbar_arrive_cluster(mapa_shared(smem_u32(&full[ring.st]), 0));  // the even CTA issues the MMAs
                if (NU > 4 && kend >= 32) mbar_arrive_cluster(mapa_shared(smem_u32(&full[s1]), 0));
            } else {
                mbar_arrive(&full[ring.st]);
                if (NU > 4 && kend >= 32) mbar_arrive(&full[s1]);
            }
        }
        if (NU > 4 && kend >= 32) {
            ring.st = s2;
            ring.ph = ph2;
        } else {
            ring.st = s1;
            ring.ph = ph1;
        }
    }
    ring.kpos = kend & 15u;
}

// BIG: stores with r3 > 16 (up to TC_RMAX = 32); the default instantiation
// keeps the r3 <= 16 dispatch (fewer registers, smaller code).
// WA: the A operand W = V x_2 U2 comes precomputed from the store's W arena
// by TMA (build_warena_kernel; stores whose W fits the memory budget) — no
// producer warps, no factor ring; the tile's K range is cut at stage
// boundaries for split items (a column's r3 slots may straddle parts: the
// sum over K is linear).
// ADJ (with WA): the adjoint of a W-arena store as one GEMM, G = conj(W)^T Phi
// (M = the packed (j, r3) slots of a component, N = (i3, c), K = rows): A =
// the transposed arena, B = Phi as row-contiguous fp16 planes, the MMA signs
// of a conjugated A, and the epilogue writes raw G (adjg_contract_kernel
// finishes z).  The tile map reuses the forward's with nt2 = 1: "i1 block" =
// slot tile.
template <bool PAIR, bool BIG = false, bool WA = false, bool ADJ = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap bmap, const __grid_constant__ CUtensorMap amap,
                  const TcDesc* __restrict__ tcd,
                  const float2* __restrict__ varena, const float2* __restrict__ u2arena, const int* __restrict__ kc,
                  const int* __restrict__ kofs, TcGeom g, const float2* __restrict__ x, int64_t ldx, float2* __restrict__ y, int64_t ldy,
                  float2* __restrict__ rsum, const float* __restrict__ wmax) {
    using namespace sm100;
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    // align to 1024 B by offsetting the shared array itself (keeps the
    // shared address space visible to the compiler: LDS/STS, not generic)
    unsigned char* sm = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
    const uint32_t nst = uint32_t(g.nst);
    unsigned char* sA = sm;
    unsigned char* sB = sA + nst * TC_A_STAGE;
    unsigned char* sSlot = sB + nst * g.b_stage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sSlot + (WA ? 0 : TC_JR * g.slot_bytes));  // WA: no factor ring
    uint64_t* full = bars;                 // [nst]
    uint64_t* empty = full + TC_NST_MAX;   // [nst]
    uint64_t* ffull = empty + TC_NST_MAX;  // [JR]
    uint64_t* fempty = ffull + TC_JR;      // [JR]
    uint64_t* cfull = fempty + TC_JR;      // 1
    uint64_t* cfree = cfull + 1;           // 1
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfree + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // CTA pairs (PAIR): both CTAs walk the same pair tiles; rank 0 issues the
    // cta_group::2 MMAs, so its full / cfree barriers count the peer's
    // producer and fold warps too (remote arrivals), and its commits
    // multicast to the empty / cfull barriers of both CTAs.
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const int64_t tstart = g.t_begin + (PAIR ? (blockIdx.x >> 1) : blockIdx.x);
    const int64_t tstep = PAIR ? (gridDim.x >> 1) : gridDim.x;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < nst; ++s) {
            mbar_init(&full[s], WA ? 1 : 1 + TC_NPW * (PAIR ? 2 : 1));
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < TC_JR; ++s) {
            mbar_init(&ffull[s], 1);
            mbar_init(&fempty[s], TC_NPW);
        }
        mbar_init(cfull, 1);
        mbar_init(cfree, 4 * (PAIR ? 2 : 1));
        fence_mbar_init();
    }
    if (warp == 3) {
        if (PAIR)
            tmem_alloc_pair(tmem_slot, 512);
        else
            tmem_alloc(tmem_slot, 512);
    }
    if (warp == 0 && lane == 0) tma_prefetch_desc(&bmap);
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // barriers of both CTAs initialised before any remote arrival
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // wait profile (g.prof): per role, cycles spent in barrier waits
    [[maybe_unused]] uint64_t t_w = 0, t_w2 = 0;
    [[maybe_unused]] bool rec = false;
#ifdef TMB_TC_PROFILE
    const long long t_role = clock64();
#endif

    if (warp == 0) {
        // ------------------------------------------------ B-plane TMA producer
        if (elect_one()) {
            rec = true;
            uint32_t s = 0, ph = 0;
            const int plane_bytes = g.nmma * 32;
            // WA: the tile's A rows in the W arena (tile-major: [i1 / 4][i2 / 32][128 rows])
            constexpr uint32_t a_bytes = WA ? uint32_t(TC_A_STAGE) : 0u;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const TcTile tl = tc_tile(g, t, rank);
                int j0, j1;
                uint32_t ka, kb;
                tc_range<WA>(g, tl, kofs, kc, j0, j1, ka, kb);
                const int arow = ((tl.i1_0 / TC_TI1) * g.nt2 + tl.i2_0 / TC_TI2) * TC_ROWS;
                for (int kk = int(ka >> 4); kk < int((kb + 15) >> 4); ++kk) {
                    TC_TWAIT(g.prof, t_w, (mbar_wait_backoff(&empty[s], ph ^ 1, TC_BACKOFF_TMA)));
                    if constexpr (WA) {  // A: this CTA's 128 rows x 16 K of the 4 W planes
                        unsigned char* da = sA + s * TC_A_STAGE;
                        if (PAIR) {
                            const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
#pragma unroll
                            for (int pl = 0; pl < 4; ++pl)
                                tma_load_3d_pair(da + pl * TC_A_PLANE, &amap, fb, kk * 16, arow, pl * g.q + tl.k);
                        } else {
#pragma unroll
                            for (int pl = 0; pl < 4; ++pl)
                                tma_load_3d(da + pl * TC_A_PLANE, &amap, &full[s], kk * 16, arow, pl * g.q + tl.k);
                        }
                    }
                    if (PAIR) {
                        // each CTA loads its half of the i3 span (B rows [rank nmma, +nmma) of the
                        // M = 256 MMA); the bytes of both halves complete on rank 0's barrier
                        if (rank == 0) {
                            if (g.debug & 2)
                                mbar_arrive(&full[s]);
                            else
                                mbar_arrive_expect_tx(&full[s], 2u * (uint32_t(g.b_stage) + a_bytes));
                        }
                        if (!(g.debug & 2)) {
                            unsigned char* dst = sB + s * g.b_stage;
                            const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
#pragma unroll
                            for (int pl = 0; pl < TC_FPLANES; ++pl)
                                tma_load_3d_pair(dst + pl * plane_bytes, &bmap, fb, kk * 16,
                                                 tl.i3_0 + int(rank) * g.nmma, pl * g.q + tl.k);
                        }
                    } else if (g.debug & 2) {
                        mbar_arrive(&full[s]);
                    } else {
                        mbar_arrive_expect_tx(&full[s], uint32_t(g.b_stage) + a_bytes);
                        unsigned char* dst = sB + s * g.b_stage;
                        // smem plane pl = (Br hi, Bi hi, Br lo, Bi lo) holds both halves of the
                        // tile's N rows contiguously ([pl][hh][nmma rows])
                        for (int hh = 0; hh < g.nh3; ++hh)
#pragma unroll
                            for (int pl = 0; pl < TC_FPLANES; ++pl)
                                tma_load_3d(dst + (pl * g.nh3 + hh) * plane_bytes, &bmap, &full[s], kk * 16,
                                            tl.i3_0 + hh * g.nmma, pl * g.q + tl.k);
                    }
                    if (++s == nst) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        if ((!PAIR || rank == 0) && elect_one()) {
            rec = true;
            // complex product over the tile's span = nh3 * NMMA voxels along i3
            // (TMEM: Yr at [0, span), Yi at [span, 2 span)), four real products
            // of full width N = span, each as hi.hi + hi.lo + lo.hi:
            //   Yr += Ar.U3r,  Yr -= Ai.U3i (negate-A bit),  Yi += Ar.U3i,  Yi += Ai.U3r
            const int span = g.nmma * g.nh3;
            const uint32_t id_p = umma_idesc_f16(TC_ROWS * (PAIR ? 2 : 1), span, false, false);
            const uint32_t id_n = umma_idesc_f16(TC_ROWS * (PAIR ? 2 : 1), span, true, false);
            // Yr += Ar Br -/+ Ai Bi, Yi += Ar Bi +/- Ai Br: the lower signs for the adjoint
            // GEMM's conjugated A (ADJ)
            const uint32_t id_aibi = ADJ ? id_p : id_n, id_aibr = ADJ ? id_n : id_p;
            const int plane_b = (PAIR ? span / 2 : span) * 32;  // one smem B plane (this CTA's i3 rows)
            uint32_t s = 0, ph = 0, gch = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const TcTile tl = tc_tile(g, t, rank);
                int j0, j1;
                uint32_t ka, kb;
                tc_range<WA>(g, tl, kofs, kc, j0, j1, ka, kb);
                const int nks = int((kb + 15) >> 4) - int(ka >> 4);
                int cpos = 0;  // stage position inside the current chain
                for (int kk = 0; kk < nks; ++kk) {
                    if (cpos == 0) {
                        TC_TWAIT(g.prof, t_w, (mbar_wait(cfree, (gch & 1) ^ 1)));  // previous chain folded
                        tc_fence_after();
                    }
                    TC_TWAIT(g.prof, t_w2, (mbar_wait(&full[s], ph)));
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + s * TC_A_STAGE);
                    const uint32_t b0 = smem_u32(sB + s * g.b_stage);
                    // A planes: 0 = re hi, 1 = re lo, 2 = im hi, 3 = im lo
                    uint64_t A[4];
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) A[pl] = umma_smem_desc(a0 + pl * TC_A_PLANE, 256, 6);
                    const uint32_t acc = cpos > 0 ? 1u : 0u;
                    const uint64_t Brh = umma_smem_desc(b0 + 0 * plane_b, 256, 6);
                    const uint64_t Bih = umma_smem_desc(b0 + 1 * plane_b, 256, 6);
                    const uint64_t Brl = umma_smem_desc(b0 + 2 * plane_b, 256, 6);
                    const uint64_t Bil = umma_smem_desc(b0 + 3 * plane_b, 256, 6);
                    const uint32_t yr = tmem, yi = tmem + uint32_t(span);
#define MMA(...) (PAIR ? mma_f16_pair(__VA_ARGS__) : mma_f16(__VA_ARGS__))
#define COMMIT(b) (PAIR ? mma_commit_pair(b) : mma_commit(b))
                    MMA(yr, A[0], Brh, id_p, acc);
                    MMA(yr, A[0], Brl, id_p, 1);
                    MMA(yr, A[1], Brh, id_p, 1);
                    MMA(yr, A[2], Bih, id_aibi, 1);
                    MMA(yr, A[2], Bil, id_aibi, 1);
                    MMA(yr, A[3], Bih, id_aibi, 1);
                    MMA(yi, A[0], Bih, id_p, acc);
                    MMA(yi, A[0], Bil, id_p, 1);
                    MMA(yi, A[1], Bih, id_p, 1);
                    MMA(yi, A[2], Brh, id_aibr, 1);
                    MMA(yi, A[2], Brl, id_aibr, 1);
                    MMA(yi, A[3], Brh, id_aibr, 1);
                    COMMIT(&empty[s]);
                    if (++s == nst) {
                        s = 0;
                        ph ^= 1;
                    }
                    if (++cpos == g.chain || kk == nks - 1) {
                        COMMIT(cfull);
                        cpos = 0;
                        ++gch;
                    }
                }
            }
        }
#undef MMA
#undef COMMIT
        __syncwarp();
    } else if (warp == 2 && !WA) {
        // ---------------------------------------------------- factor loader
        if (elect_one()) {
            rec = true;
            uint32_t s = 0, ph = 0;
            for (int64_t t = tstart; t < g.t_end; t += tstep) {
                const TcTile tl = tc_tile(g, t, rank);
                const TcDesc* tdk = tcd + int64_t(tl.k) * g.ncols;
                int j0, j1;
                uint32_t ka, kb;
                tc_range(g, tl, kofs, kc, j0, j1, ka, kb);
                for (int j = j0; j < j1; ++j) {
                    TC_TWAIT(g.prof, t_w, (mbar_wait_backoff(&fempty[s], ph ^ 1, TC_BACKOFF_LD)));
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
    } else if (!WA && warp >= TC_PW0 && warp < TC_FW0) {
        static_assert(TC_NH * 8 >= TC_RMAX, "producer switch covers ceil(TC_RMAX / TC_NH)");
        // ------------------------------------------------------ A producers
        // warp pw: i1 = pw / (4 / NR) (warp-uniform), rows i2 in a block of 8 NR;
        // lane: row lane rl in [0, 8) (rows i2a = block base + rl, + 8 e for
        // e < NR) and c = 4u + hq.  Each quad of lanes is 2 row lanes x 2 hq, so a
        // quad's V and U2 loads touch 2 addresses each: one shared-memory
        // wavefront per LDS.64 for both (lanes of a quad on 4 distinct
        // addresses cost two; tools/smem_probe.cu).
        // tile row = i2 + 32 i1 (= TMEM lane of the accumulator)
        rec = lane == 0;
        const int pw = warp - TC_PW0;
        const int rl = 2 * ((lane >> 2) & 3) + (lane & 1);
        constexpr int wpi = 4 / TC_NR;  // producer warps per i1 row of the tile
        const int i1l = pw / wpi, hq = 2 * (lane >> 4) + ((lane >> 1) & 1);
        const int i2a = 8 * TC_NR * (pw % wpi) + rl;
        uint32_t rowbase[TC_NR], xorv[TC_NR];
#pragma unroll
        for (int e = 0; e < TC_NR; ++e) {
            const uint32_t row = uint32_t(i2a + 8 * e + 32 * i1l);
            rowbase[e] = row * 32u;
            xorv[e] = (row & 4u) << 2;
        }
        ARing ring{0, 0, 0};
        uint32_t fs = 0, fph = 0;
        for (int64_t t = tstart; t < g.t_end; t += tstep) {
            const TcTile tl = tc_tile(g, t, rank);
            int j0, j1;
            uint32_t ka, kb;
            tc_range(g, tl, kofs, kc, j0, j1, ka, kb);
            if (ka & 15u) {
                // a column-range item starting inside a stage: its first K slots belong to
                // the previous part's columns and are zero here
                ring.kpos = ka & 15u;
                TC_TWAIT(g.prof != nullptr, t_w2, (mbar_wait(&empty[ring.st], ring.ph ^ 1u)));
                unsigned char* st = sA + ring.st * TC_A_STAGE;
                for (uint32_t kq = uint32_t(hq); kq < ring.kpos; kq += 4)
#pragma unroll
                    for (int e = 0; e < TC_NR; ++e) {
                        __half* a = reinterpret_cast<__half*>(st + rowbase[e] + ((kq * 2u) ^ xorv[e]));
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) a[pl * TC_A_PLANE / 2] = __float2half_rn(0.f);
                    }
            }
            // (r2, r3) of the next column are prefetched from the global descriptor table one
            // column ahead, so the NU dispatch does not wait on the slot's descriptor
            const int2* rk = reinterpret_cast<const int2*>(&tcd[int64_t(tl.k) * g.ncols].r2);
            constexpr int kDescStride = int(sizeof(TcDesc) / sizeof(int2));
            int2 rn = j0 < j1 ? __ldg(rk + int64_t(j0) * kDescStride) : make_int2(0, 0);
            for (int j = j0; j < j1; ++j) {
                const int r2 = rn.x, r3 = rn.y;
                if (j + 1 < j1) rn = __ldg(rk + int64_t(j + 1) * kDescStride);
                TC_TWAIT(g.prof, t_w, (mbar_wait(&ffull[fs], fph)));
                const unsigned char* slot = sSlot + fs * g.slot_bytes;
                const float2* V = reinterpret_cast<const float2*>(slot + TC_SLOT_V) + i1l;
                const float2* U2 = reinterpret_cast<const float2*>(slot + g.u2_off);
#define TC_COL(NU)                                                                                             \
    tc_produce_column<NU, PAIR>(V, U2, (g.debug & 1) ? 0 : r2, r2 | 1, r3, hq, i2a, g.wsc, &fempty[fs], empty, full, sA, \
                          rowbase, xorv, lane, nst, ring)
                if constexpr (BIG) {
                    switch ((r3 + TC_NH - 1) / TC_NH) {
                        case 1: TC_COL(1); break;
                        case 2: TC_COL(2); break;
                        case 3: TC_COL(3); break;
                        case 4: TC_COL(4); break;
                        case 5: TC_COL(5); break;
                        case 6: TC_COL(6); break;
                        case 7: TC_COL(7); break;
                        default: TC_COL(8); break;
                    }
                } else {
                    switch ((r3 + TC_NH - 1) / TC_NH) {
                        case 1: TC_COL(1); break;
                        case 2: TC_COL(2); break;
                        case 3: TC_COL(3); break;
                        default: TC_COL(4); break;
                    }
                }
#undef TC_COL
                if (++fs == TC_JR) {
                    fs = 0;
                    fph ^= 1;
                }
            }
            if (ring.kpos != 0) {  // zero the tail of the last stage and close it
                unsigned char* st = sA + ring.st * TC_A_STAGE;
                for (uint32_t kq = ring.kpos + uint32_t(hq); kq < 16; kq += 4)
#pragma unroll
                    for (int e = 0; e < TC_NR; ++e) {
                        __half* a = reinterpret_cast<__half*>(st + rowbase[e] + ((kq * 2u) ^ xorv[e]));
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) a[pl * TC_A_PLANE / 2] = __float2half_rn(0.f);
                    }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_cluster(mapa_shared(smem_u32(&full[ring.st]), 0));
                    else
                        mbar_arrive(&full[ring.st]);
                }
                ring_ahead(ring, 1, nst, ring.st, ring.ph);
                ring.kpos = 0;
            }
        }
    } else if (warp >= TC_FW0) {
        // ------------------------------------------ chain fold + epilogue
        // The running sum of the tile lives in this CTA's private scratch
        // rsum[blockIdx.x][i3 / 2][row] as float4 (re, im of i3 and i3 + 1;
        // L2-resident, a warp's 32 rows are one coalesced 512-byte access).
        // The fold is fire-and-forget so the accumulator is released as soon
        // as TMEM has been read: the first chain of a tile stores, later
        // chains add with red.global.add.v4.f32 (round-to-nearest; every
        // element is only ever touched by this thread, in program order, so
        // the sum is deterministic), and the last chain reads the running sum
        // back and writes y.
        rec = lane == 0;
        const int quarter = warp & 3;             // TMEM lane quarter = i1 of the tile
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const uint32_t tC = tmem + lane_addr;
        const int row = lane + 32 * quarter;      // row = i2 + 32 i1
        const int span = g.nmma * g.nh3;
        float4* rs = reinterpret_cast<float4*>(rsum) + int64_t(blockIdx.x) * (span / 2) * TC_ROWS + row;
        const int64_t nv3 = int64_t(g.n1) * g.n2 * g.n3;
        // exact power of two (W scale x B scale); the adjoint GEMM writes raw G
        const float inv = ADJ ? 1.f : 1.f / (g.wsc * fp16_scale(*wmax));
        uint32_t gch = 0;
        for (int64_t t = tstart; t < g.t_end; t += tstep) {
            const TcTile tl = tc_tile(g, t, rank);
            int j0, j1;
            uint32_t ka, kb;
            tc_range<WA>(g, tl, kofs, kc, j0, j1, ka, kb);
            const int nks = int((kb + 15) >> 4) - int(ka >> 4);
            const int nch = (nks + g.chain - 1) / g.chain;
            const int ei1 = tl.i1_0 + quarter, ei2 = tl.i2_0 + lane;
            // split items write their partial tile to ypart ([item][rank][i3][row]); the wave's
            // reduce kernel sums the parts into y in a fixed order
            const bool part_out = g.split > 1;
            const bool eok = ADJ || part_out || (ei1 < g.n1 && ei2 < g.n2);
            float2* yp = part_out ? g.ypart + ((t * (1 + g.pair) + int64_t(rank)) * span) * TC_ROWS + row
                         : ADJ    ? y + int64_t(tl.k) * g.nt * g.gslots + int64_t(tl.i1_0 / TC_TI1) * TC_ROWS + row
                                  : y + int64_t(tl.k) * nv3 + ei1 + int64_t(g.n1) * ei2;
            const int64_t pl = int64_t(g.n1) * g.n2;
            // output of tile column nl (N row n = i3_0 + nl = i3 * p + c)
            auto put = [&](int nl, float2 v) {
                if (part_out) {
                    yp[int64_t(TC_ROWS) * nl] = v;
                    return;
                }
                if (ADJ) {  // G[k][n][slot]: a warp's 32 slots are contiguous
                    const int n = tl.i3_0 + nl;
                    if (n < g.nt) yp[int64_t(n) * g.gslots] = v;
                    return;
                }
                const int n = tl.i3_0 + nl;
                if (n >= g.nt) return;
                int i3 = n, c = 0;
                if (g.p > 1) {
                    i3 = n / g.p;
                    c = n - i3 * g.p;
                }
                yp[ldy * c + pl * i3] = v;
            };
            if (WA && nch == 0) {
                // an empty K range (a split item of the W-arena forward with fewer
                // K stages than parts): its partial tile is zero
                if (part_out)
                    for (int nl = 0; nl < span; ++nl) put(nl, make_float2(0.f, 0.f));
                continue;
            }
            for (int ch = 0; ch < nch; ++ch, ++gch) {
                TC_TWAIT(g.prof, t_w, (mbar_wait_backoff(cfull, gch & 1, TC_BACKOFF_FOLD)));
                tc_fence_after();
                const bool last = ch == nch - 1;
                for (int hh = 0; hh < g.nh3; ++hh)
                    for (int cb = 0; cb < g.nmma; cb += 16) {
                        uint32_t cr[16], ci[16];
                        const int i3l = hh * g.nmma + cb;  // even; Yr at column i3l, Yi at span + i3l
                        tmem_ld16(tC + uint32_t(i3l), cr);
                        tmem_ld16(tC + uint32_t(span + i3l), ci);
                        tmem_ld_wait();
                        float4* rp = rs + int64_t(i3l / 2) * TC_ROWS;
                        if (!last) {
#pragma unroll
                            for (int m = 0; m < 8; ++m) {
                                float4* a = rp + int64_t(m) * TC_ROWS;
                                const float4 v = make_float4(__uint_as_float(cr[2 * m]), __uint_as_float(ci[2 * m]),
                                                             __uint_as_float(cr[2 * m + 1]),
                                                             __uint_as_float(ci[2 * m + 1]));
                                if (ch == 0)
                                    *a = v;
                                else
                                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(v.x),
                                                 "f"(v.y), "f"(v.z), "f"(v.w)
                                                 : "memory");
                            }
                        } else {
                            float4 r[8];
                            if (ch > 0) {
#pragma unroll
                                for (int m = 0; m < 8; ++m) r[m] = rp[int64_t(m) * TC_ROWS];
                            } else {
#pragma unroll
                                for (int m = 0; m < 8; ++m) r[m] = make_float4(0.f, 0.f, 0.f, 0.f);
                            }
                            if (eok) {
#pragma unroll
                                for (int m = 0; m < 8; ++m) {
                                    put(i3l + 2 * m, make_float2((__uint_as_float(cr[2 * m]) + r[m].x) * inv,
                                                                 (__uint_as_float(ci[2 * m]) + r[m].y) * inv));
                                    put(i3l + 2 * m + 1, make_float2((__uint_as_float(cr[2 * m + 1]) + r[m].z) * inv,
                                                                     (__uint_as_float(ci[2 * m + 1]) + r[m].w) * inv));
                                }
                            }
                        }
                    }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_cluster(mapa_shared(smem_u32(cfree), 0));
                    else
                        mbar_arrive(cfree);
                }
            }
        }
    }
#ifdef TMB_TC_PROFILE
    if (g.prof && rec) {
        const int role = warp < 3 ? warp : (warp < TC_FW0 ? 3 : 4);
        atomicAdd(g.prof + 3 * role, static_cast<unsigned long long>(clock64() - t_role));
        atomicAdd(g.prof + 3 * role + 1, static_cast<unsigned long long>(t_w));
        atomicAdd(g.prof + 3 * role + 2, static_cast<unsigned long long>(t_w2));

    }
#endif
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

// max |x[j, c]| over the columns and right-hand sides of a pass (the fp16
// scale of the B operand), by an order-free atomicMax on float bit patterns.
__global__ void xmax_kernel(const float2* __restrict__ x, int64_t ldx, int64_t ncols, int64_t p, float* __restrict__ out) {
    float m = 0.f;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < ncols * p; e += int64_t(gridDim.x) * blockDim.x) {
        const float2 v = x[(e % ncols) + ldx * (e / ncols)];
        m = fmaxf(m, sqrtf(v.x * v.x + v.y * v.y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(out), __float_as_uint(m));
}

// The forward's B operand for a pass of p right-hand sides:
// B[k][n = i3 p + c][K = kofs[k][j] + r] = sb x[j, c] U3_j[i3, r] as a 2-term
// fp16 split in 4 planes [Re hi, Im hi, Re lo, Im lo][q][nt][kpad] (sb =
// fp16_scale(max |x|); U3 normalised by 2^-e3 so |U3| <= 1, factor_scale_kernel).  x_j rides in B so the producers' A
// operand is x-free and, with p > 1, W = V x_2 U2 is produced once for all
// right-hand sides (they share the tile's N space).  One block per tensor.
__global__ void build_xb_kernel(const TDesc* __restrict__ td, const float2* __restrict__ arena,
                                const int* __restrict__ kofs, const float2* __restrict__ x, int64_t ldx, int p,
                                int64_t ncols, int q, int n3, int64_t nt, int64_t kpad, const float* __restrict__ xmax,
                                const TcDesc* __restrict__ tcd, __half* __restrict__ planes, int64_t t0 = 0) {
    const int64_t t = t0 + blockIdx.x;  // tensor index k*ncols + j (t0: first tensor of a component range)
    const int k = int(t / ncols);
    const int64_t j = t - int64_t(k) * ncols;
    const TDesc d = td[t];
    const int e3 = fexp_e3(tcd[t].fexp);
    const int64_t k0 = kofs[t];
    const int64_t plane = int64_t(q) * nt * kpad;
    const float sb = fp16_scale(*xmax);
    for (int e = threadIdx.x; e < n3 * d.r3 * p; e += blockDim.x) {
        const int c = e / (n3 * d.r3);
        const int rem = e - c * (n3 * d.r3);
        const int i3 = rem / d.r3, r = rem - i3 * d.r3;
        const float2 u0 = arena[d.off_u3 + rem];
        const float2 u = make_float2(ldexpf(u0.x, -e3), ldexpf(u0.y, -e3));  // normalised U3 (|u| <= 1), exact
        const float2 xv = x[j + ldx * c];
        const float br = (xv.x * u.x - xv.y * u.y) * sb, bi = (xv.x * u.y + xv.y * u.x) * sb;
        const __half rh = __float2half_rn(br), ih = __float2half_rn(bi);
        const __half rl = __float2half_rn(br - __half2float(rh)), il = __float2half_rn(bi - __half2float(ih));
        const int64_t o = (int64_t(k) * nt + int64_t(i3) * p + c) * kpad + k0 + r;
        planes[o] = rh;
        planes[plane + o] = ih;
        planes[2 * plane + o] = rl;
        planes[3 * plane + o] = il;
    }
}

// Sum the column-range parts of a split final wave (fwd_tc_kernel with
// g.split > 1) into y, in part order (deterministic).  One thread per
// (tile, CTA rank, i3 of the span, row).
__global__ void fwd_split_reduce_kernel(TcGeom g, int64_t tiles, float2* __restrict__ y, int64_t ldy) {
    const int span = g.nmma * g.nh3;
    const int nr = 1 + g.pair;
    const int64_t total = tiles * nr * span * TC_ROWS;
    const int64_t nv3 = int64_t(g.n1) * g.n2 * g.n3;
    const int64_t pl = int64_t(g.n1) * g.n2;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int row = int(e % TC_ROWS);
        int64_t rest = e / TC_ROWS;
        const int i3l = int(rest % span);
        rest /= span;
        const int rank = int(rest % nr);
        const int64_t tt = rest / nr;
        const TcTile tl = tc_tile(g, tt * g.split, uint32_t(rank));
        const int i1 = tl.i1_0 + row / 32, i2 = tl.i2_0 + row % 32, n = tl.i3_0 + i3l;
        if (i1 >= g.n1 || i2 >= g.n2 || n >= g.nt) continue;
        const int i3 = n / g.p, c = n - (n / g.p) * g.p;
        float2 acc = make_float2(0.f, 0.f);
        for (int p = 0; p < g.split; ++p) {
            const float2 v = g.ypart[(((tt * g.split + p) * nr + rank) * span + i3l) * TC_ROWS + row];
            acc.x += v.x;
            acc.y += v.y;
        }
        y[ldy * c + int64_t(tl.k) * nv3 + i1 + int64_t(g.n1) * i2 + pl * i3] = acc;
    }
}

// The same for the adjoint GEMM's split final wave (fwd_tc_kernel<.., ADJ>,
// parts = K-stage ranges of the rows): the parts of each (slot tile, n) are
// summed in part order into G[k][n][slot].
__global__ void adjg_split_reduce_kernel(TcGeom g, int64_t tiles, float2* __restrict__ G) {
    const int span = g.nmma * g.nh3;
    const int nr = 1 + g.pair;
    const int64_t total = tiles * nr * span * TC_ROWS;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int row = int(e % TC_ROWS);
        int64_t rest = e / TC_ROWS;
        const int i3l = int(rest % span);
        rest /= span;
        const int rank = int(rest % nr);
        const int64_t tt = rest / nr;
        const TcTile tl = tc_tile(g, tt * g.split, uint32_t(rank));
        const int n = tl.i3_0 + i3l;
        if (n >= g.nt) continue;
        float2 acc = make_float2(0.f, 0.f);
        for (int p = 0; p < g.split; ++p) {
            const float2 v = g.ypart[(((tt * g.split + p) * nr + rank) * span + i3l) * TC_ROWS + row];
            acc.x += v.x;
            acc.y += v.y;
        }
        G[(int64_t(tl.k) * g.nt + n) * g.gslots + int64_t(tl.i1_0 / TC_TI1) * TC_ROWS + row] = acc;
    }
}

// ------------------------------------------------- store-side V arena (K6'')
// V_t[i1][b][c] = sum_a U1t[i1][a] G[a + r1 (b + r2 c)] for every tensor t
// (the reference's mode-1 product, src/tensor.cpp:106-108, done once per
// store instead of once per tile), accumulated in fp64 from the c64 factors
// and stored [i1/4][c + r3 b][i1 % 4] as float2; rows i1 >= n1 of the last
// group of four are zero.
__global__ void build_v_kernel(const TDesc* __restrict__ td, const float2* __restrict__ arena,
                               const TcDesc* __restrict__ tcd, int n1, float2* __restrict__ varena) {
    const int64_t t = blockIdx.x;
    const TDesc d = td[t];
    const int r23 = d.r2 * d.r3;
    const int n1p = (n1 + 3) & ~3;
    float2* out = varena + tcd[t].off_v;
    const int ev = fexp_e2(tcd[t].fexp) + fexp_e3(tcd[t].fexp);  // V carries the factors' normalisation
    for (int e = threadIdx.x; e < n1p * r23; e += blockDim.x) {
        const int i1 = e / r23, bc = e - i1 * r23;
        double vr = 0.0, vi = 0.0;
        if (i1 < n1) {
            const float2* u = arena + d.off_u1 + int64_t(i1) * d.r1;
            const float2* gp = arena + d.off_core + int64_t(bc) * d.r1;
            for (int a = 0; a < d.r1; ++a) {
                const float2 ua = u[a], ga = gp[a];
                vr += double(ua.x) * ga.x - double(ua.y) * ga.y;
                vi += double(ua.x) * ga.y + double(ua.y) * ga.x;
            }
        }
        const float fr = float(ldexp(vr, ev)), fi = float(ldexp(vi, ev));
        const int b = bc % d.r2, c = bc / d.r2;  // bc = b + r2 c (core order)
        out[int64_t(i1 >> 2) * 4 * r23 + int64_t(c + d.r3 * b) * 4 + (i1 & 3)] = make_float2(fr, fi);
    }
}


// Per tensor: max over (i1, c) of the 2-norm over b of V[i1, b, c] — a
// bound on |W[row, c]| / |x_j| because every row of the normalised U2 has
// norm <= 1 (factor_scale_kernel).
__global__ void vbound_kernel(const TDesc* __restrict__ td, const TcDesc* __restrict__ tcd,
                              const float2* __restrict__ varena, int n1, float* __restrict__ vbound) {
    const int64_t t = blockIdx.x;
    const int r2 = tcd[t].r2, r3 = tcd[t].r3;
    const float2* v = varena + tcd[t].off_v;
    float m = 0.f;
    for (int e = threadIdx.x; e < n1 * r3; e += blockDim.x) {
        const int i1 = e / r3, c = e - i1 * r3;
        float s2 = 0.f;
        for (int b = 0; b < r2; ++b) {
            const float2 x = v[int64_t(i1 >> 2) * 4 * r2 * r3 + int64_t(c + r3 * b) * 4 + (i1 & 3)];
            s2 += x.x * x.x + x.y * x.y;
        }
        m = fmaxf(m, sqrtf(s2));
    }
    __shared__ float red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float r = 0.f;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
        vbound[t] = r * 1.0001f;  // margin for the fp32 norm's rounding
    }
    (void)td;
}


// ------------------------------------------------ store-side U2 arena (K6 U2)
// U2 of every tensor with an odd row stride r2 | 1 and n2 rounded up to TI2
// rows (the padding rows and columns are zero).
__global__ void build_u2_kernel(const TDesc* __restrict__ td, const float2* __restrict__ arena,
                                const TcDesc* __restrict__ tcd, int n2, float2* __restrict__ u2arena) {
    const int64_t t = blockIdx.x;
    const TDesc d = td[t];
    const int ld2 = d.r2 | 1;
    const int n2p = (n2 + TC_TI2 - 1) / TC_TI2 * TC_TI2;
    float2* out = u2arena + tcd[t].off_u2;
    const int e2 = fexp_e2(tcd[t].fexp);
    for (int e = threadIdx.x; e < n2p * ld2; e += blockDim.x) {
        const int i2 = e / ld2, b = e - i2 * ld2;
        const float2 u = (i2 < n2 && b < d.r2) ? arena[d.off_u2 + int64_t(i2) * d.r2 + b] : make_float2(0.f, 0.f);
        out[e] = make_float2(ldexpf(u.x, -e2), ldexpf(u.y, -e2));  // normalised U2 (row norms <= 1), exact
    }
}

// ------------------------------------------ store-side W arena (WA forward)
// W = V x_2 U2 of every tensor, scaled by the forward's A scale wsc and split
// into the A operand's 4 fp16 planes, for stores whose W fits the memory
// budget (build_warena, tm_capi.cu): [plane][k][row][kpad] fp16 with rows
// tile-major ([i1 / 4][i2 / 32][i1 % 4][i2 % 32], TC_ROWS per tile) and K the
// component's packed column stream.  The arithmetic is the producer warps'
// (tc_produce_column: FFMA2 complex multiply-adds over b in order, the wsc
// multiply, f16_split2), so the A tiles are the same bits.  One block per
// (tensor, row tile), one thread per row.  wt (optional): the same planes
// transposed, [plane][k][slot < kpadt][row] (the adjoint GEMM's K-major A:
// M = the packed (j, r3) slots, K = rows).
__global__ void build_warena_kernel(const TcDesc* __restrict__ tcd, const float2* __restrict__ varena,
                                    const float2* __restrict__ u2arena, const int* __restrict__ kofs, int64_t ncols,
                                    int q, int n1, int n2, int nt2, int64_t rows_pad, int64_t kpad, float wsc,
                                    __half* __restrict__ wa, __half* __restrict__ wt, int64_t kpadt) {
    using namespace sm100;
    const int64_t t = blockIdx.x;  // component-major tensor index k ncols + j
    const int k = int(t / ncols);
    const int tile = int(blockIdx.y), t1 = tile / nt2, t2 = tile - t1 * nt2;
    const int row = int(threadIdx.x);  // i2 + 32 i1 inside the tile
    const int i1 = t1 * TC_TI1 + row / TC_TI2, i2 = t2 * TC_TI2 + row % TC_TI2;
    if (i1 >= n1 || i2 >= n2) return;  // padding rows stay zero (the arena is cleared)
    const TcDesc d = tcd[t];
    const int r2 = d.r2, r3 = d.r3;
    const float2* V = varena + d.off_v + int64_t(i1 / TC_TI1) * TC_TI1 * r2 * r3 + (i1 % TC_TI1);
    const float2* U = u2arena + d.off_u2 + int64_t(i2) * (r2 | 1);
    const int64_t plane = int64_t(q) * rows_pad * kpad;
    unsigned short* o = reinterpret_cast<unsigned short*>(wa) + (int64_t(k) * rows_pad + int64_t(tile) * TC_ROWS + row) * kpad +
                        kofs[t];
    const uint64_t sc2 = f2_pack(wsc, wsc);
    for (int c = 0; c < r3; ++c) {
        uint64_t w = 0;
        for (int b = 0; b < r2; ++b) cfma2v(w, V[(c + r3 * b) * TC_TI1], U[b]);
        asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(w) : "l"(sc2));
        uint32_t hi, lo;
        f16_split2(w, hi, lo);
        o[c] = static_cast<unsigned short>(hi);                  // Re hi
        o[plane + c] = static_cast<unsigned short>(lo);          // Re lo
        o[2 * plane + c] = static_cast<unsigned short>(hi >> 16);  // Im hi
        o[3 * plane + c] = static_cast<unsigned short>(lo >> 16);  // Im lo
        if (wt) {  // the adjoint GEMM's A operand: [plane][k][slot][row], rows contiguous
            const int64_t tp = int64_t(q) * kpadt * rows_pad;
            unsigned short* ot = reinterpret_cast<unsigned short*>(wt) +
                                 (int64_t(k) * kpadt + kofs[t] + c) * rows_pad + int64_t(tile) * TC_ROWS + row;
            ot[0] = static_cast<unsigned short>(hi);
            ot[tp] = static_cast<unsigned short>(lo);
            ot[2 * tp] = static_cast<unsigned short>(hi >> 16);
            ot[3 * tp] = static_cast<unsigned short>(lo >> 16);
        }
    }
}

// ---------------------------------------- factor normalisation (per tensor)
// The tensor-core operands rely on two bounds that hold for the reference's
// orthonormal factors: |U3| <= 1 (fp16 scale of the B planes) and U2 row
// norms <= 1 (the |W| bound behind the A scale).  A valid store need not be
// orthonormal (proj/src/io.cpp:131-139 checks ranks only): T = G x1 U1 x2 U2
// x3 U3 is unchanged by U3 -> U3 2^-e3, U2 -> U2 2^-e2, V = U1 x1 G -> V
// 2^(e2+e3), and powers of two are exact.  Per tensor: e3 = the binary
// exponent of max |U3| and e2 that of the largest U2 row norm (frexp: the
// normalised maxima fall in [1/2, 1)), packed into TcDesc::fexp.
__global__ void factor_scale_kernel(const TDesc* __restrict__ td, const float2* __restrict__ arena, int n2, int n3,
                                    TcDesc* __restrict__ tcd) {
    const int64_t t = blockIdx.x;
    const TDesc d = td[t];
    float m3 = 0.f, m2 = 0.f;
    for (int e = threadIdx.x; e < n3 * d.r3; e += blockDim.x) {
        const float2 u = arena[d.off_u3 + e];
        m3 = fmaxf(m3, sqrtf(u.x * u.x + u.y * u.y));
    }
    for (int i2 = threadIdx.x; i2 < n2; i2 += blockDim.x) {
        float s2 = 0.f;
        for (int b = 0; b < d.r2; ++b) {
            const float2 u = arena[d.off_u2 + int64_t(i2) * d.r2 + b];
            s2 += u.x * u.x + u.y * u.y;
        }
        m2 = fmaxf(m2, sqrtf(s2) * 1.0001f);  // margin for the fp32 norm's rounding
    }
    __shared__ float r3[32], r2[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m3 = fmaxf(m3, __shfl_xor_sync(0xffffffffu, m3, o));
        m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    }
    if ((threadIdx.x & 31) == 0) {
        r3[threadIdx.x >> 5] = m3;
        r2[threadIdx.x >> 5] = m2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            m3 = fmaxf(m3, r3[w]);
            m2 = fmaxf(m2, r2[w]);
        }
        int e3 = 0, e2 = 0;
        if (m3 > 0.f) frexpf(m3, &e3);
        if (m2 > 0.f) frexpf(m2, &e2);
        e3 = max(-100, min(100, e3));
        e2 = max(-100, min(100, e2));
        tcd[t].fexp = (e2 & 0xff) | ((e3 & 0xff) << 8);
    }
}

}  // namespace tmb
