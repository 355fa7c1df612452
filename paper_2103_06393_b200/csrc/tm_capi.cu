// C ABI of the B200 Tucker-compressed coupling matvec (include/tuckmat_b200.h).
//
// Host orchestration only: validation with the reference's error messages,
// the device store (K6 pack), work buffers, and the launch plan of the
// forward / adjoint / ACA kernels.  No CPU fallback: every product runs on
// the device or fails with TM_CUDA_ERROR.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tuckmat_b200.h"
#include "tm_aux_kernels.cuh"
#include "tm_common.cuh"
#include "tm_kernels_cc.cuh"
#include "tm_kernels_tc.cuh"
#include "tm_adj_tc.cuh"
#include "tm_adj2_tc.cuh"
#include "tm_k3w_tc.cuh"
#include "tm_tmap.h"
#include "tm_io_internal.hpp"

using namespace tmb;

namespace {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

struct TmError : std::runtime_error {
    int code;
    TmError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void contract(const std::string& m) { throw TmError(TM_CONTRACT_VIOLATION, m); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation)
            throw TmError(TM_CAPACITY_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
        throw TmError(TM_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CK(x) ck((x), #x)

void launched(cudaError_t e, const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    ck(e == cudaSuccess ? cudaGetLastError() : e, what);
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    void release() {  // on the device that owns the buffer
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            bytes = 0;
            CK(cudaMalloc(&p, std::max<size_t>(need, 256)));
            bytes = std::max<size_t>(need, 256);
        }
        return p;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return TM_OK;
    } catch (const TmError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const tmb_io::ParseFail& e) {  // streaming ingest (tm_io.cpp)
        g_last_error = e.what();
        return TM_PARSE_ERROR;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return TM_CAPACITY_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TM_ERROR;
    }
}

int64_t align2(int64_t v) { return (v + 1) & ~int64_t(1); }

constexpr size_t kSmemBudget = 100 * 1024;  // 2 CTAs / SM
constexpr size_t kSmemMax = 227 * 1024;

}  // namespace

struct tm_store {
    int device = 0;
    int dtype = TM_C64;
    int q = 0;
    int64_t ncols = 0;
    int64_t dims[3] = {0, 0, 0};
    int64_t m2 = 0;
    int rmax[3] = {1, 1, 1};
    std::vector<int32_t> ranks;  // [col][comp][mode]
    std::vector<TDesc> host_desc;  // build-time only
    int64_t dec_madds = 0;
    TDesc* d_desc = nullptr;
    void* d_arena = nullptr;
    int64_t arena_elems = 0;
    void* d_v = nullptr;
    // dense-U ACA store (tm_store_create_dense_aca): U is m1 x r (dims = {m1, 1, 1}, q = 1)
    bool dense = false;
    void* d_u = nullptr;
    int64_t device_bytes = 0;
    // tensor-core (tcgen05 fp16-split) forward data: V / U2 operand copies, K offsets
    bool tc_ok = false;
    int* d_kofs = nullptr;   // [q*ncols] component-major K offset of each tensor
    int* d_kc = nullptr;     // [q] K extent of each component
    float vmax = 0.f;            // max per-tensor |W| bound (W = V x_2 U2): the fp16 scale of A
    float* d_vbound = nullptr;  // [q*ncols] per-tensor bound of |W| / |x_j|
    TcDesc* d_tcd = nullptr;  // [q*ncols] tensor-core descriptors
    float2* d_varena = nullptr;  // mode-1 products V = U1 x_1 G
    float2* d_u2arena = nullptr;  // U2 with odd row strides
    // W arena (W = V x_2 U2 as the forward's fp16-split A operand, built when it
    // fits the memory budget: the forward then runs without producer warps)
    __half* d_warena = nullptr;
    // the adjoint GEMM (run_adjoint_gemm): the arena transposed, [plane][k][slot][row]
    __half* d_wt = nullptr;
    int64_t wt_kpadt = 0;  // slots per component, a multiple of 256 (CTA-pair slot tiles)
    int* d_kcr = nullptr;  // [q] the GEMM's K extent (rows) per component
    CUtensorMap wt_map{};
    DevBuf gbuf, phit;     // per call: G and the row-contiguous Phi planes
    DevBuf gkmax;          // per call: the components' Phi scales (phimax_k_kernel)
    int64_t warena_rows = 0;
    CUtensorMap warena_map{};
    // K3W (tm_k3w_tc.cuh, many right-hand sides on a W-arena store): per-slot
    // U3S / descriptor tables and the unswizzled W-plane map, built on first use
    __half* d_k3pa = nullptr;      // the W arena's fp16 planes on K3W's padded slot stream
    __half* d_k3b1 = nullptr;      // GEMM1's B operand per (component, stage, i3 block)
    uint32_t* d_k3flag = nullptr;  // [q][kpad8 / 16] column-end bits per stage
    int* d_k3kc = nullptr;         // [q] padded slots per component
    int* d_k3gend = nullptr;       // [q][nks] W stages needed through each GEMM2 stage
    int64_t k3_kpad8 = 0;

    // tensor-core adjoint: chunk-aligned, i3-contiguous U3 planes
    bool tca_ok = false;
    __half* d_aplanes = nullptr;
    int* d_nch = nullptr;     // [q] chunks per component
    int* d_cstart = nullptr;  // [q][maxch + 1] first column of each chunk
    int maxch = 0;
    int64_t nslots = 0;       // slots per component (maxch * 128)
    CUtensorMap adj_bmap{};
    // right-hand-side groups (adj_tc2_kernel<NR>): the adjoint U3 planes packed
    // in 128 / NR-slot chunks, built on the first adjoint with p >= 2 (ensure_adj_pack)
    struct AdjPack {
        bool ok = false;
        __half* d_aplanes = nullptr;
        int* d_nch = nullptr;
        int* d_cstart = nullptr;
        int maxch = 0;
        int64_t nslots = 0;
        CUtensorMap bmap{};
    } adjp[2];  // [0]: 64-slot chunks (pairs), [1]: 32-slot chunks (quads)
    int64_t kpad = 0;
    DevBuf xbplanes;        // the forward's per-call B operand (build_xb_kernel)
    size_t xb_zeroed = 0;   // bytes of xbplanes zeroed since allocation
    std::mutex mu;
    // completion event of the latest product: products share the work
    // buffers below, so each one's stream waits for it first (order_after_prev)
    cudaEvent_t done = nullptr;
    DevBuf part, xin, yout, wbuf, phiplanes, rsum, scal;
    DevBuf ypart;  // partial tiles of a split final wave of the tensor-core forward
    DevBuf ccpart;  // partial y blocks of a column-split CUDA-core forward (small stores)

    int64_t nv() const { return dims[0] * dims[1] * dims[2]; }
    int64_t rows() const { return q * nv(); }
    size_t csize() const { return dtype == TM_C64 ? sizeof(float2) : sizeof(double2); }
    ~tm_store() {
        if (done) {
            cudaEventSynchronize(done);
            cudaEventDestroy(done);
        }
        if (d_kofs) cudaFree(d_kofs);
        if (d_kc) cudaFree(d_kc);

        if (d_vbound) cudaFree(d_vbound);
        if (d_tcd) cudaFree(d_tcd);
        if (d_varena) cudaFree(d_varena);
        if (d_u2arena) cudaFree(d_u2arena);
        if (d_warena) cudaFree(d_warena);
        if (d_wt) cudaFree(d_wt);
        if (d_k3pa) cudaFree(d_k3pa);
        if (d_k3b1) cudaFree(d_k3b1);
        if (d_k3flag) cudaFree(d_k3flag);
        if (d_k3kc) cudaFree(d_k3kc);
        if (d_k3gend) cudaFree(d_k3gend);
        if (d_kcr) cudaFree(d_kcr);
        if (d_aplanes) cudaFree(d_aplanes);
        for (auto& a : adjp) {
            if (a.d_aplanes) cudaFree(a.d_aplanes);
            if (a.d_nch) cudaFree(a.d_nch);
            if (a.d_cstart) cudaFree(a.d_cstart);
        }
        if (d_nch) cudaFree(d_nch);
        if (d_cstart) cudaFree(d_cstart);
        if (d_desc) cudaFree(d_desc);
        if (d_arena) cudaFree(d_arena);
        if (d_v) cudaFree(d_v);
        if (d_u) cudaFree(d_u);
    }
};

namespace {

// Device-side ordering of the products on one store.  They share the store's
// work buffers (B planes, Phi planes, partials, scales), and the host mutex
// only serialises the enqueue: a TM_DEVICE call returns with its kernels
// still running.  So every product's stream(s) first wait for the previous
// product's completion event, and the product records its own at the end —
// TM_DEVICE calls on different streams and TM_HOST calls on their private
// streams are serialised on the device too.
void order_after_prev(tm_store* s, cudaStream_t st) { CK(cudaStreamWaitEvent(st, s->done, 0)); }
void mark_done(tm_store* s, cudaStream_t st) { CK(cudaEventRecord(s->done, st)); }

// ------------------------------------------------------------ store build --
// c64 stores run the forward on the tcgen05 fp16-split kernel (chained TMEM
// accumulation, tm_kernels_tc.cuh) whenever the store qualifies;
// TMB_DISABLE_TC=1 forces the CUDA-core kernel (used by the tests to check
// one against the other).
bool tc_disabled() {
    const char* d = std::getenv("TMB_DISABLE_TC");
    return d && d[0] == '1';
}

int tc_chain() {
    const char* e = std::getenv("TMB_TC_CHAIN");
    const int v = e ? std::atoi(e) : 0;
    // 32 stages x 6 truncating MMAs per accumulator: 3.7e-6 at config 4 (the
    // physics-rank store; 24: 2.8e-6, 48: 5.4e-6 — tools/validate_full.py
    // --chains, profiles/r02i_tune.jsonl); each fold moves the 256 KB
    // accumulator through red.global.add, so longer chains cost less (24 -> 32:
    // -3.5 % forward time per SM clock, same box)
    return v > 0 ? v : 32;
}

bool warena_disabled() {
    const char* e = std::getenv("TMB_WARENA");
    return e && *e == '0';
}

// TMB_ADJ_GEMM=0: no adjoint GEMM on the W arena (the consumer-warp adjoint instead)
bool adjg_disabled() {
    const char* e = std::getenv("TMB_ADJ_GEMM");
    return e && *e == '0';
}

// The W arena: W = V x_2 U2 of every tensor as the forward's fp16-split A
// operand, precomputed once (build_warena_kernel) when it fits
// $TMB_WARENA_GB (default 24 GB) and half of the free device memory — small
// and medium grids (configs 2, 3, 5: 0.7 / 1.1 / 2.6 GB), not config 4
// (~220 GB).  The forward then streams A by TMA like B, with no producer
// warps; the adjoint keeps the V arena.  TMB_WARENA=0 disables it.
void build_warena(tm_store* s) {
    if (warena_disabled() || s->ncols == 0) return;
    const int nt1 = int((s->dims[0] + TC_TI1 - 1) / TC_TI1), nt2 = int((s->dims[1] + TC_TI2 - 1) / TC_TI2);
    const int64_t rows_pad = int64_t(nt1) * nt2 * TC_ROWS;
    const size_t bytes = size_t(4) * s->q * size_t(rows_pad) * size_t(s->kpad) * sizeof(__half);
    // the adjoint GEMM's transposed arena (slots padded to CTA-pair tiles of 256)
    const int64_t kpadt = (s->kpad + 255) / 256 * 256;
    const size_t tbytes = adjg_disabled() ? 0 : size_t(4) * s->q * size_t(kpadt) * size_t(rows_pad) * sizeof(__half);
    double cap_gb = 24.0;
    if (const char* e = std::getenv("TMB_WARENA_GB")) cap_gb = std::atof(e);
    size_t freeb = 0, total = 0;
    CK(cudaMemGetInfo(&freeb, &total));
    if (double(bytes + tbytes) > cap_gb * 1e9 || bytes + tbytes > freeb / 2 || nt1 * nt2 > 65535 ||
        rows_pad >= (int64_t(1) << 31))
        return;
    CK(cudaMalloc(&s->d_warena, bytes));
    CK(cudaMemset(s->d_warena, 0, bytes));
    if (tbytes) {
        CK(cudaMalloc(&s->d_wt, tbytes));
        CK(cudaMemset(s->d_wt, 0, tbytes));
        std::vector<int> kcr(static_cast<size_t>(s->q), int(rows_pad));
        CK(cudaMalloc(&s->d_kcr, kcr.size() * sizeof(int)));
        CK(cudaMemcpy(s->d_kcr, kcr.data(), kcr.size() * sizeof(int), cudaMemcpyHostToDevice));
        s->wt_kpadt = kpadt;
        s->wt_map = make_tmap_3d_f16(s->d_wt, uint64_t(rows_pad), uint64_t(kpadt), uint64_t(4 * s->q),
                                     uint64_t(rows_pad) * 2, uint64_t(kpadt) * rows_pad * 2, 16, TC_ROWS,
                                     CU_TENSOR_MAP_SWIZZLE_32B);
    }
    const int64_t ntens = s->ncols * s->q;
    build_warena_kernel<<<dim3(unsigned(ntens), unsigned(nt1 * nt2)), TC_ROWS>>>(
        s->d_tcd, s->d_varena, s->d_u2arena, s->d_kofs, s->ncols, s->q, int(s->dims[0]), int(s->dims[1]), nt2,
        rows_pad, s->kpad, fp16_scale(s->vmax * 1.0001f), s->d_warena, s->d_wt, kpadt);
    launched(cudaSuccess, "build_warena_kernel");
    CK(cudaDeviceSynchronize());
    s->warena_rows = rows_pad;
    s->warena_map = make_tmap_3d_f16(s->d_warena, uint64_t(s->kpad), uint64_t(rows_pad), uint64_t(4 * s->q),
                                     uint64_t(s->kpad) * 2, uint64_t(rows_pad) * s->kpad * 2, 16, TC_ROWS,
                                     CU_TENSOR_MAP_SWIZZLE_32B);
    s->device_bytes += int64_t(bytes + tbytes);
}

// B planes of the tensor-core forward (see tm_kernels_tc.cuh), built once.
void build_tc(tm_store* s, const std::vector<TDesc>& desc) {
    int dev = 0, major = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (s->dtype != TM_C64 || s->ncols == 0 || major != 10) return;
    if (s->rmax[0] > TC_RMAX || s->rmax[1] > TC_RMAX || s->rmax[2] > TC_RMAX) return;
    if (s->dims[2] < 16) return;
    {  // the forward's worst-case plan (single CTA, two 128-voxel i3 halves) must fit
        const int u2_off = TC_SLOT_V + int(round16(uint32_t(TC_TI1 * s->rmax[1] * s->rmax[2] * 8)));
        const size_t slot = size_t((u2_off + TC_TI2 * (s->rmax[1] | 1) * 8 + 127) / 128 * 128);
        const int nst_min = s->rmax[2] > 16 ? 3 : 2;
        const size_t need = 1024 + size_t(nst_min) * (TC_A_STAGE + 2 * TC_FPLANES * TC_NMAX * 32) + TC_JR * slot +
                            (2 * TC_NST_MAX + 2 * TC_JR + 2) * 8 + 16;
        if (need > kSmemMax) return;  // ranks too large for the factor ring: CUDA-core kernels
    }
    const int64_t ntens = s->ncols * s->q;
    std::vector<int> kofs(static_cast<size_t>(ntens)), kc(static_cast<size_t>(s->q), 0);
    for (int k = 0; k < s->q; ++k) {
        int64_t acc = 0;
        for (int64_t j = 0; j < s->ncols; ++j) {
            kofs[static_cast<size_t>(k * s->ncols + j)] = int(acc);
            acc += desc[static_cast<size_t>(k * s->ncols + j)].r3;
        }
        if (acc >= (int64_t(1) << 30)) return;
        kc[static_cast<size_t>(k)] = int(acc);
        s->kpad = std::max<int64_t>(s->kpad, (acc + 15) / 16 * 16);
    }
    const int64_t n3 = s->dims[2];
    // V arena: per tensor ceil(n1/4)*4 x r2 x r3 float2, [i1/4][c + r3 b][i1%4]
    const int64_t n1p = (s->dims[0] + 3) / 4 * 4;
    std::vector<TcDesc> tcd(static_cast<size_t>(ntens));
    int64_t voff = 0, u2off = 0;
    const int64_t n2p = (s->dims[1] + TC_TI2 - 1) / TC_TI2 * TC_TI2;
    for (int64_t t = 0; t < ntens; ++t) {
        const TDesc& d = desc[static_cast<size_t>(t)];
        TcDesc& c = tcd[static_cast<size_t>(t)];
        c.off_v = voff;
        c.off_u2 = u2off;
        c.off_u3 = d.off_u3;
        u2off += n2p * (d.r2 | 1);
        c.r2 = d.r2;
        c.r3 = d.r3;
        c.pad0 = c.pad1 = c.pad2 = c.fexp = 0;
        voff += n1p * d.r2 * d.r3;
    }
    // adjoint chunks: whole columns, at most AJ_CH (j, c) slots each
    std::vector<int> aslot(static_cast<size_t>(ntens), 0), nch(static_cast<size_t>(s->q), 0);
    std::vector<std::vector<int>> cst(static_cast<size_t>(s->q));
    for (int k = 0; k < s->q; ++k) {
        int fill = AJ_CH, chunk = -1;
        for (int64_t j = 0; j < s->ncols; ++j) {
            const size_t t = static_cast<size_t>(k * s->ncols + j);
            const int r3 = desc[t].r3;
            if (fill + r3 > AJ_CH || int64_t(cst[k].size()) == 0 ||
                (j - cst[static_cast<size_t>(k)].back()) >= AJ_MAXCOLS) {
                ++chunk;
                fill = 0;
                cst[static_cast<size_t>(k)].push_back(int(j));
            }
            aslot[t] = chunk * AJ_CH + fill;
            tcd[t].pad0 = fill;
            fill += r3;
        }
        nch[static_cast<size_t>(k)] = chunk + 1;
        s->maxch = std::max(s->maxch, chunk + 1);
    }
    s->nslots = int64_t(s->maxch) * AJ_CH;
    std::vector<int> cstart(static_cast<size_t>(s->q) * (s->maxch + 1), int(s->ncols));
    for (int k = 0; k < s->q; ++k)
        for (size_t n = 0; n < cst[static_cast<size_t>(k)].size(); ++n)
            cstart[static_cast<size_t>(k) * (s->maxch + 1) + n] = cst[static_cast<size_t>(k)][n];
    const int64_t n3p = (n3 + 7) / 8 * 8;
    const size_t abytes = size_t(TC_BPLANES) * s->q * s->nslots * n3p * sizeof(__half);
    const size_t vbytes = size_t(voff) * sizeof(float2);
    const size_t u2bytes = size_t(u2off) * sizeof(float2);
    CK(cudaMalloc(&s->d_kofs, kofs.size() * sizeof(int)));
    CK(cudaMalloc(&s->d_kc, kc.size() * sizeof(int)));
    CK(cudaMalloc(&s->d_tcd, tcd.size() * sizeof(TcDesc)));
    CK(cudaMalloc(&s->d_varena, std::max<size_t>(vbytes, 16)));
    CK(cudaMalloc(&s->d_u2arena, std::max<size_t>(u2bytes, 16)));
    CK(cudaMalloc(&s->d_aplanes, abytes));
    CK(cudaMalloc(&s->d_nch, nch.size() * sizeof(int)));
    CK(cudaMalloc(&s->d_cstart, cstart.size() * sizeof(int)));
    CK(cudaMemcpy(s->d_nch, nch.data(), nch.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s->d_cstart, cstart.data(), cstart.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemset(s->d_aplanes, 0, abytes));
    CK(cudaMemcpy(s->d_tcd, tcd.data(), tcd.size() * sizeof(TcDesc), cudaMemcpyHostToDevice));
    // per-tensor power-of-two factor normalisation of the tensor-core operand
    // copies (non-orthonormal factors stay inside fp16's range)
    factor_scale_kernel<<<unsigned(ntens), 256>>>(s->d_desc, static_cast<const float2*>(s->d_arena),
                                                  int(s->dims[1]), int(n3), s->d_tcd);
    launched(cudaSuccess, "factor_scale_kernel");
    {
        DevBuf as;
        int* d_as = static_cast<int*>(as.get(aslot.size() * sizeof(int)));
        CK(cudaMemcpy(d_as, aslot.data(), aslot.size() * sizeof(int), cudaMemcpyHostToDevice));
        build_adj_bplanes_kernel<<<unsigned(ntens), 256>>>(s->d_desc, static_cast<const float2*>(s->d_arena), d_as,
                                                           s->ncols, s->q, int(n3), int(n3p), s->nslots, s->d_tcd,
                                                           s->d_aplanes);
        launched(cudaSuccess, "build_adj_bplanes_kernel");
        CK(cudaDeviceSynchronize());
    }
    s->adj_bmap = make_tmap_3d_f16(s->d_aplanes, uint64_t(n3), uint64_t(s->nslots), uint64_t(TC_BPLANES * s->q),
                                   uint64_t(n3p) * 2, uint64_t(s->nslots) * n3p * 2, 16, AJ_CH,
                                   CU_TENSOR_MAP_SWIZZLE_32B);
    s->tca_ok = true;
    CK(cudaMemcpy(s->d_kofs, kofs.data(), kofs.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s->d_kc, kc.data(), kc.size() * sizeof(int), cudaMemcpyHostToDevice));
    build_v_kernel<<<unsigned(ntens), 256>>>(s->d_desc, static_cast<const float2*>(s->d_arena), s->d_tcd,
                                             int(s->dims[0]), s->d_varena);
    launched(cudaSuccess, "build_v_kernel");
    build_u2_kernel<<<unsigned(ntens), 256>>>(s->d_desc, static_cast<const float2*>(s->d_arena), s->d_tcd,
                                              int(s->dims[1]), s->d_u2arena);
    launched(cudaSuccess, "build_u2_kernel");
    CK(cudaMalloc(&s->d_vbound, size_t(ntens) * sizeof(float)));
    vbound_kernel<<<unsigned(ntens), 256>>>(s->d_desc, s->d_tcd, s->d_varena, int(s->dims[0]), s->d_vbound);
    launched(cudaSuccess, "vbound_kernel");
    CK(cudaDeviceSynchronize());
    {  // the A operand's fp16 scale: max over tensors of the |W| bound
        std::vector<float> vb(static_cast<size_t>(ntens));
        CK(cudaMemcpy(vb.data(), s->d_vbound, vb.size() * sizeof(float), cudaMemcpyDeviceToHost));
        for (float v : vb) s->vmax = std::max(s->vmax, v);
    }
    s->device_bytes += int64_t(vbytes + u2bytes + abytes + tcd.size() * sizeof(TcDesc) + (kofs.size() + kc.size()) * sizeof(int));
    s->tc_ok = true;
    build_warena(s);
}

void build_store(tm_store* s, const tm_store_desc& d, const tmb_io::PayloadFill* fill = nullptr) {
    const int64_t n1 = d.dims[0], n2 = d.dims[1], n3 = d.dims[2];
    const int64_t ntens = s->ncols * s->q;
    // host-side tensor table: source offsets ([col][comp] order) and
    // destination descriptors (component-major order)
    std::vector<int64_t> src_off(static_cast<size_t>(ntens) + 1, 0);
    std::vector<TDesc> desc(static_cast<size_t>(std::max<int64_t>(ntens, 1)));
    int64_t doff = 0;
    for (int g = 0; g < 3; ++g) s->rmax[g] = 1;
    for (int64_t i = 0; i < ntens; ++i) {
        const int32_t* r = d.ranks + 3 * i;
        for (int g = 0; g < 3; ++g) {
            if (r[g] < 1 || r[g] > d.dims[g])
                contract("store: tucker rank " + std::to_string(r[g]) + " out of range for mode " +
                         std::to_string(g + 1));
            s->rmax[g] = std::max(s->rmax[g], int(r[g]));
        }
        const int64_t sz = int64_t(r[0]) * r[1] * r[2] + n1 * r[0] + n2 * r[1] + n3 * r[2];
        src_off[i + 1] = src_off[i] + sz;
        const int64_t j = i / s->q, k = i % s->q;
        TDesc& t = desc[static_cast<size_t>(k * s->ncols + j)];
        t.r1 = r[0];
        t.r2 = r[1];
        t.r3 = r[2];
        t.pad = 0;
        t.off_core = doff;
        doff += align2(int64_t(r[0]) * r[1] * r[2]);
        t.off_u1 = doff;
        doff += align2(n1 * r[0]);
        t.off_u2 = doff;
        doff += align2(n2 * r[1]);
        t.off_u3 = doff;
        doff += align2(n3 * r[2]);
        s->dec_madds += n1 * r[0] * r[1] * r[2] + n1 * n2 * r[1] * r[2] + n1 * n2 * n3 * r[2];
    }
    s->ranks.assign(d.ranks, d.ranks + 3 * ntens);
    s->host_desc = desc;
    // slack: the tensor-core path bulk-copies whole tile rows of U1/U2 and
    // may read past the last tensor's segments
    s->arena_elems = doff + 16 * 64 + 4096;
    const size_t cs = s->csize();
    CK(cudaMalloc(&s->d_arena, size_t(s->arena_elems) * cs));
    CK(cudaMalloc(reinterpret_cast<void**>(&s->d_desc), desc.size() * sizeof(TDesc)));
    CK(cudaMemcpy(s->d_desc, desc.data(), desc.size() * sizeof(TDesc), cudaMemcpyHostToDevice));
    s->device_bytes = int64_t(s->arena_elems * cs + desc.size() * sizeof(TDesc));

    // pack in bounded chunks of whole tensors
    const int64_t total = src_off[static_cast<size_t>(ntens)];
    (void)total;
    const int64_t chunk_cap = int64_t(16) << 20;  // 16 M complex128 = 256 MiB of staging
    auto chunk_end = [&](int64_t t0) {
        int64_t t1 = t0 + 1;
        while (t1 < ntens && src_off[t1 + 1] - src_off[t0] <= chunk_cap) ++t1;
        return t1;
    };
    auto make_jobs = [&](int64_t t0, int64_t t1, PackJob* jobs) {
        for (int64_t i = t0; i < t1; ++i) {
            const int64_t j = i / s->q, k = i % s->q;
            jobs[i - t0] = {src_off[i] - src_off[t0], k * s->ncols + j};
        }
    };
    auto pack = [&](const double2* src, const PackJob* jb, int64_t njobs, cudaStream_t st) {
        if (s->dtype == TM_C64)
            pack_kernel<float2><<<unsigned(njobs), 256, 0, st>>>(src, jb, s->d_desc, int(n1), int(n2), int(n3),
                                                                 static_cast<float2*>(s->d_arena));
        else
            pack_kernel<double2><<<unsigned(njobs), 256, 0, st>>>(src, jb, s->d_desc, int(n1), int(n2), int(n3),
                                                                  static_cast<double2*>(s->d_arena));
        launched(cudaSuccess, "pack_kernel");
    };
    if (fill) {
        // Streaming ingest: the host reads chunk c into pinned buffer c % 2
        // while the copy + pack of chunk c - 1 run on the stream; no host copy
        // of the whole payload ever exists.
        struct Pipe {
            void* h[2] = {nullptr, nullptr};
            PackJob* hj[2] = {nullptr, nullptr};
            cudaEvent_t done[2] = {nullptr, nullptr};
            cudaStream_t st = nullptr;
            ~Pipe() {
                if (st) cudaStreamSynchronize(st);
                for (int b = 0; b < 2; ++b) {
                    if (h[b]) cudaFreeHost(h[b]);
                    if (hj[b]) cudaFreeHost(hj[b]);
                    if (done[b]) cudaEventDestroy(done[b]);
                }
                if (st) cudaStreamDestroy(st);
            }
        } pp;
        int64_t maxjobs = 1, maxel = 1;
        for (int64_t t0 = 0; t0 < ntens;) {
            const int64_t t1 = chunk_end(t0);
            maxjobs = std::max(maxjobs, t1 - t0);
            maxel = std::max(maxel, src_off[t1] - src_off[t0]);
            t0 = t1;
        }
        DevBuf dstage[2], djobs[2];
        CK(cudaStreamCreateWithFlags(&pp.st, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CK(cudaHostAlloc(&pp.h[b], size_t(maxel) * sizeof(double2), cudaHostAllocDefault));
            CK(cudaHostAlloc(reinterpret_cast<void**>(&pp.hj[b]), size_t(maxjobs) * sizeof(PackJob),
                             cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&pp.done[b], cudaEventDisableTiming));
            dstage[b].get(size_t(maxel) * sizeof(double2));
            djobs[b].get(size_t(maxjobs) * sizeof(PackJob));
        }
        int c = 0;
        for (int64_t t0 = 0; t0 < ntens; ++c) {
            const int64_t t1 = chunk_end(t0);
            const int b = c & 1;
            if (c >= 2) CK(cudaEventSynchronize(pp.done[b]));  // buffer b's previous chunk is packed
            const int64_t elems = src_off[t1] - src_off[t0];
            (*fill)(t0, t1, static_cast<double*>(pp.h[b]));
            make_jobs(t0, t1, pp.hj[b]);
            CK(cudaMemcpyAsync(dstage[b].p, pp.h[b], size_t(elems) * sizeof(double2), cudaMemcpyHostToDevice, pp.st));
            CK(cudaMemcpyAsync(djobs[b].p, pp.hj[b], size_t(t1 - t0) * sizeof(PackJob), cudaMemcpyHostToDevice,
                               pp.st));
            pack(static_cast<const double2*>(dstage[b].p), static_cast<const PackJob*>(djobs[b].p), t1 - t0, pp.st);
            CK(cudaEventRecord(pp.done[b], pp.st));
            t0 = t1;
        }
        CK(cudaStreamSynchronize(pp.st));
    } else {
        DevBuf stage, jobbuf;
        int64_t t0 = 0;
        while (t0 < ntens) {
            const int64_t t1 = chunk_end(t0);
            const int64_t elems = src_off[t1] - src_off[t0];
            const double2* src;
            if (d.payload_on_device) {
                src = reinterpret_cast<const double2*>(d.payload) + src_off[t0];
            } else {
                void* st = stage.get(size_t(elems) * sizeof(double2));
                CK(cudaMemcpy(st, d.payload + 2 * src_off[t0], size_t(elems) * sizeof(double2),
                              cudaMemcpyHostToDevice));
                src = static_cast<const double2*>(st);
            }
            std::vector<PackJob> jobs(static_cast<size_t>(t1 - t0));
            make_jobs(t0, t1, jobs.data());
            void* jb = jobbuf.get(jobs.size() * sizeof(PackJob));
            CK(cudaMemcpy(jb, jobs.data(), jobs.size() * sizeof(PackJob), cudaMemcpyHostToDevice));
            pack(src, static_cast<const PackJob*>(jb), t1 - t0, nullptr);
            CK(cudaDeviceSynchronize());
            t0 = t1;
        }
    }

    build_tc(s, s->host_desc);
    s->host_desc.clear();
    s->host_desc.shrink_to_fit();

    if (d.v) {
        if (d.m2 < 1) contract("store: ACA V needs m2 >= 1");
        s->m2 = d.m2;
        const int64_t n = d.m2 * s->ncols;
        CK(cudaMalloc(&s->d_v, size_t(std::max<int64_t>(n, 1)) * cs));
        s->device_bytes += n * int64_t(cs);
        if (n > 0) {
            DevBuf vst;
            const double2* src;
            if (d.v_on_device) {
                src = reinterpret_cast<const double2*>(d.v);
            } else {
                void* st = vst.get(size_t(n) * sizeof(double2));
                CK(cudaMemcpy(st, d.v, size_t(n) * sizeof(double2), cudaMemcpyHostToDevice));
                src = static_cast<const double2*>(st);
            }
            const unsigned grid = unsigned(std::min<int64_t>((n + 255) / 256, 4096));
            if (s->dtype == TM_C64)
                convert_kernel<float2><<<grid, 256>>>(src, n, static_cast<float2*>(s->d_v));
            else
                convert_kernel<double2><<<grid, 256>>>(src, n, static_cast<double2*>(s->d_v));
            launched(cudaSuccess, "convert_kernel");
            CK(cudaDeviceSynchronize());
        }
    }
}

tm_store* create_store(const tm_store_desc& d, int device, int dtype, const tmb_io::PayloadFill* fill = nullptr) {
    if (dtype != TM_C64 && dtype != TM_C128) contract("store: dtype must be TM_C64 or TM_C128");
    if (d.q < 1 || d.ncols < 0 || d.dims[0] < 1 || d.dims[1] < 1 || d.dims[2] < 1)
        contract("store: non-positive dimensions");
    if (d.dims[0] > (1 << 30) || d.dims[1] > (1 << 30) || d.dims[2] > (1 << 30))
        contract("store: grid dimension too large");
    if (d.ncols > 0 && (!d.ranks || (!d.payload && !fill))) contract("store: ranks and payload are required");
    if (d.v && d.m2 < 1) contract("store: ACA V needs m2 >= 1");
    // validate every rank before touching the device (reference: read_tucker,
    // src/io.cpp:133-139, and the TuckerTensor invariant 1 <= r_g <= n_g)
    for (int64_t i = 0; i < d.ncols * d.q; ++i)
        for (int g = 0; g < 3; ++g) {
            const int32_t r = d.ranks[3 * i + g];
            if (r < 1 || r > d.dims[g])
                contract("store: tucker rank " + std::to_string(r) + " out of range for mode " + std::to_string(g + 1));
        }
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw TmError(TM_CUDA_ERROR, "store: no CUDA device " + std::to_string(device));
    DeviceGuard guard(device);
    auto* s = new tm_store;
    if (cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming) != cudaSuccess) {
        s->done = nullptr;
        delete s;
        throw TmError(TM_CUDA_ERROR, "store: cannot create the completion event");
    }
    s->device = device;
    s->dtype = dtype;
    s->q = d.q;
    s->ncols = d.ncols;
    for (int g = 0; g < 3; ++g) s->dims[g] = d.dims[g];
    try {
        build_store(s, d, fill);
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

// ------------------------------------------------------------ kernel plan --

// Parts per tile for a launch of `tiles` (< one wave of `wave` CTAs) tiles:
// the split s in [1, smax] that minimises the launch's rounds per part,
// ceil(tiles s / wave) / s (a 96-tile launch on 148 CTAs: s = 3, two rounds
// of thirds = 2/3 of a tile; s = 1 leaves 52 CTAs idle for a whole tile).
int best_split(int64_t tiles, int64_t wave, int smax) {
    if (tiles <= 0 || tiles >= wave) return 1;
    int best = 1;
    double bt = 1.0;
    for (int sp = 2; sp <= smax; ++sp) {
        const double t = double((tiles * sp + wave - 1) / wave) / sp;
        if (t < bt - 1e-9) {
            bt = t;
            best = sp;
        }
    }
    return best;
}

int num_sms(int dev);

template <typename C, int RM, int CN, int NW, int TI1>
struct CcPlan {
    static constexpr int ROWS = RM * NW, TI2 = ROWS / TI1, TI3 = 32 * CN;
    CcGeom g{};
    size_t smem = 0;
    dim3 grid;
    CcPlan(const tm_store* s, bool adjoint) {
        g.ncols = s->ncols;
        g.n1 = int(s->dims[0]);
        g.n2 = int(s->dims[1]);
        g.n3 = int(s->dims[2]);
        g.q = s->q;
        g.nt1 = int((g.n1 + TI1 - 1) / TI1);
        g.nt2 = int((g.n2 + TI2 - 1) / TI2);
        g.rmax1 = s->rmax[0];
        g.rmax2 = s->rmax[1];
        g.rmax3 = s->rmax[2];
        const int nt3 = (g.n3 + TI3 - 1) / TI3;
        const size_t slot = size_t(cc_slot_elems<TI1, TI2, TI3>(g.rmax1, g.rmax2, g.rmax3)) * sizeof(C);
        const size_t red = adjoint ? size_t(8 * NW) * sizeof(C) : 0;
        int jb = 8;
        while (jb > 1 && slot * jb + red > kSmemBudget) --jb;
        if (slot * jb + red > kSmemMax)
            throw TmError(TM_CAPACITY_ERROR,
                          "tucker ranks (" + std::to_string(g.rmax1) + "," + std::to_string(g.rmax2) + "," +
                              std::to_string(g.rmax3) + ") exceed the shared-memory plan of the CUDA-core kernel");
        g.jb = jb;
        smem = slot * jb + red;
        g.ntiles = int(int64_t(g.nt1) * g.nt2 * nt3);
        g.nsplit = 1;
        g.part_stride = 0;
        grid = dim3(unsigned(g.ntiles), unsigned(s->q), 1);
    }
    // Small stores (tiles x q x p below two CTAs per SM): split each tile's
    // column loop into parts so the launch fills the GPU (config 1: 54 CTAs).
    void split_for(int64_t p, int nsm) {
        const int64_t ctas = int64_t(g.ntiles) * g.q * std::min<int64_t>(p, 65535);
        if (ctas >= 2 * int64_t(nsm) || g.ncols < 2) return;
        g.nsplit = int(std::min<int64_t>({int64_t(16), g.ncols, (2 * int64_t(nsm) + ctas - 1) / ctas}));
        grid.x = unsigned(int64_t(g.ntiles) * g.nsplit);
    }
};

template <typename C, int RM, int CN, int NW, int TI1>
void run_forward_cc(tm_store* s, const C* x, int64_t ldx, int64_t p, C* y, int64_t ldy, cudaStream_t st, int kb,
                    int ke) {
    CcPlan<C, RM, CN, NW, TI1> plan(s, false);
    plan.g.k0 = kb;
    plan.grid.y = unsigned(ke - kb);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    plan.split_for(p, num_sms(dev));
    auto kern = fwd_cc_kernel<C, RM, CN, NW, TI1>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.smem)));
    const int64_t rows = s->q * s->nv();
    for (int64_t c0 = 0; c0 < p; c0 += 65535) {
        dim3 grid = plan.grid;
        const int64_t pc = std::min<int64_t>(65535, p - c0);
        grid.z = unsigned(pc);
        if (plan.g.nsplit > 1) {  // partial y per part, then a fixed-order sum
            CcGeom g = plan.g;
            g.part_stride = rows * pc;
            C* yp = static_cast<C*>(s->ccpart.get(size_t(g.nsplit) * size_t(rows * pc) * sizeof(C)));
            kern<<<grid, NW * 32, plan.smem, st>>>(s->d_desc, static_cast<const C*>(s->d_arena), g, x + ldx * c0,
                                                   ldx, yp, rows);
            launched(cudaSuccess, "fwd_cc_kernel");
            const unsigned rb = unsigned(std::min<int64_t>((rows * pc + 255) / 256, 4096));
            cc_split_reduce_kernel<C><<<rb, 256, 0, st>>>(yp, g.nsplit, g.part_stride, rows, pc, y + ldy * c0, ldy,
                                                          int64_t(kb) * s->nv(), int64_t(ke - kb) * s->nv());
            launched(cudaSuccess, "cc_split_reduce_kernel");
        } else {
            kern<<<grid, NW * 32, plan.smem, st>>>(s->d_desc, static_cast<const C*>(s->d_arena), plan.g, x + ldx * c0,
                                                   ldx, y + ldy * c0, ldy);
            launched(cudaSuccess, "fwd_cc_kernel");
        }
    }
}

template <typename C, int RM, int CN, int NW, int TI1>
void run_adjoint_cc(tm_store* s, const C* phi, int64_t ldphi, int64_t p, C* z, int64_t ldz, cudaStream_t st) {
    CcPlan<C, RM, CN, NW, TI1> plan(s, true);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    plan.split_for(p, num_sms(dev));
    const int64_t ntiles = plan.g.ntiles;
    const int64_t nred = ntiles * s->q;
    C* part = static_cast<C*>(s->part.get(size_t(s->ncols * p * nred) * sizeof(C)));
    auto kern = adj_cc_kernel<C, RM, CN, NW, TI1>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.smem)));
    for (int64_t c0 = 0; c0 < p; c0 += 65535) {
        dim3 grid = plan.grid;
        grid.z = unsigned(std::min<int64_t>(65535, p - c0));
        kern<<<grid, NW * 32, plan.smem, st>>>(s->d_desc, static_cast<const C*>(s->d_arena), plan.g,
                                               phi + ldphi * c0, ldphi, part + s->ncols * nred * c0);
        launched(cudaSuccess, "adj_cc_kernel");
    }
    const int64_t warps = s->ncols * p;
    const unsigned blocks = unsigned((warps * 32 + 255) / 256);
    adj_reduce_kernel<C><<<blocks, 256, 0, st>>>(part, s->ncols, p, nred, z, ldz);
    launched(cudaSuccess, "adj_reduce_kernel");
}

// n3-dependent choice of lanes-per-i3 (CN): smallest padded n3, weighted by
// the smem-traffic cost of narrow micro-tiles.
int pick_cn(int64_t n3) {
    double best = 1e300;
    int cn = 4;
    const int cands[3] = {4, 2, 1};
    const double cost[3] = {1.0, 1.2, 1.6};
    for (int i = 0; i < 3; ++i) {
        const int64_t ti3 = 32 * cands[i];
        const double c = double((n3 + ti3 - 1) / ti3 * ti3) * cost[i];
        if (c < best - 1e-9) {
            best = c;
            cn = cands[i];
        }
    }
    return cn;
}

int num_sms(int dev) {
    int n = 0;
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

// Host I/O overlapped with the tensor-core kernels, per (rhs, component)
// block of q*n_v rows: the forward copies each finished block of y to the
// host while later waves compute; the adjoint copies Phi in block by block
// ahead of the waves that need it (tm_forward / tm_adjoint with TM_HOST).
struct HostPipe {
    cudaStream_t copy = nullptr;  // nullptr: no host copies (only the block hook)
    void* host = nullptr;  // forward: y (out); adjoint: phi (in)
    int64_t ldhost = 0;
    // forward: called (on the host, while enqueueing) once components [k0, k1)
    // of right-hand sides [c0, c0 + pb) are complete on `st` — the sharded
    // store's per-component reduce hangs off it (tm_shard.cuh)
    std::function<void(int64_t k0, int64_t k1, int64_t c0, int64_t pb, cudaStream_t st)> block_done;
};

// One pass of the tensor-core forward over pb right-hand sides: the B
// operand x (x) U3 of the pass is built per call (build_xb_kernel) and the
// tiles span the N space n = i3 * pb + c, so W is produced once for all
// right-hand sides of the pass.
void run_forward_pass(const tm_store* s, const float2* x, int64_t ldx, int64_t p, float2* y, int64_t ldy,
                      cudaStream_t st, const HostPipe* hp, int64_t hc0, int kb, int ke) {
    TcGeom g{};
    g.ncols = s->ncols;
    g.n1 = int(s->dims[0]);
    g.n2 = int(s->dims[1]);
    g.n3 = int(s->dims[2]);
    g.q = s->q;
    g.p = int(p);
    g.nt = int(int64_t(g.n3) * p);
    g.nt1 = (g.n1 + TC_TI1 - 1) / TC_TI1;
    g.nt2 = (g.n2 + TC_TI2 - 1) / TC_TI2;
    g.nmma = std::min(TC_NMAX, (g.nt + 15) / 16 * 16);
    g.nh3 = g.nt > TC_NMAX ? 2 : 1;
    g.nt3 = (g.nt + g.nmma * g.nh3 - 1) / (g.nmma * g.nh3);
    g.wsc = fp16_scale(s->vmax * 1.0001f);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const int nsm = num_sms(dev);
    // CTA-pair kernel (cta_group::2, M = 256 over two i1 blocks, each CTA
    // holding half of the 256-voxel i3 span of B): halves the B-operand
    // shared-memory reads per MMA and the B stage.  Needs full 256-voxel i3
    // tiles and an even number of i1 blocks.
    {
        const char* e = std::getenv("TMB_DISABLE_PAIR");
        g.pair = (!(e && *e && *e != '0') && g.nmma == TC_NMAX && g.nh3 == 2 && g.nt1 % 2 == 0 && nsm >= 2) ? 1 : 0;
    }
    if (g.pair) g.nt1 /= 2;
    g.ntiles = int64_t(g.q) * g.nt3 * g.nt2 * g.nt1;
    g.rmax2 = s->rmax[1];
    g.rmax3 = s->rmax[2];
    g.u2_off = TC_SLOT_V + int(round16(uint32_t(TC_TI1 * g.rmax2 * g.rmax3 * 8)));
    g.slot_bytes = (g.u2_off + TC_TI2 * (g.rmax2 | 1) * 8 + 127) / 128 * 128;
    g.b_stage = (g.pair ? 1 : g.nh3) * TC_FPLANES * g.nmma * 32;
    g.chain = tc_chain();
    {
        const char* dbg = std::getenv("TMB_TC_DEBUG");
        g.debug = dbg ? std::atoi(dbg) : 0;
    }
    // W arena (build_warena): A by TMA, no producers and no factor slots
    const bool wa = s->d_warena && !warena_disabled();
    auto smem_for = [&](int nst) {
        return 1024 + size_t(nst) * (TC_A_STAGE + g.b_stage) + (wa ? 0 : size_t(TC_JR) * g.slot_bytes) +
               (2 * TC_NST_MAX + 2 * TC_JR + 2) * 8 + 16;
    };
    // a column opens up to ceil((15 + r3) / 16) A stages at once: 2 for r3 <= 16, 3 up to TC_RMAX
    const int nst_min = (s->rmax[2] > 16 && !wa) ? 3 : 2;
    g.nst = TC_NST_MAX;
    if (const char* e = std::getenv("TMB_TC_NST")) if (std::atoi(e) >= 2) g.nst = std::min(TC_NST_MAX, std::atoi(e));
    g.nst = std::max(g.nst, nst_min);
    while (g.nst > nst_min && smem_for(g.nst) > kSmemMax) --g.nst;
    const size_t smem = smem_for(g.nst);
    if (smem > kSmemMax) throw TmError(TM_CAPACITY_ERROR, "tensor-core forward: shared-memory plan too large");
    const bool big = s->rmax[2] > 16;  // the r3 <= 32 instantiations
    auto kfpair = wa ? fwd_tc_kernel<true, false, true> : (big ? fwd_tc_kernel<true, true> : fwd_tc_kernel<true>);
    auto kfsingle = wa ? fwd_tc_kernel<false, false, true> : (big ? fwd_tc_kernel<false, true> : fwd_tc_kernel<false>);
    CK(cudaFuncSetAttribute(kfsingle, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CK(cudaFuncSetAttribute(kfpair, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // grid: CTAs; a wave covers `wave` tiles (pair tiles in pair mode)
    // (up to 8 parts per tile when there are fewer tiles than SMs: best_split)
    const unsigned grid = g.pair ? unsigned(std::min<int64_t>(2 * 8 * g.ntiles, nsm & ~1))
                                 : unsigned(std::min<int64_t>(8 * g.ntiles, nsm));
    const int64_t wave = g.pair ? grid / 2 : grid;
    g.prof = nullptr;
    if (g.debug & 8) {
        CK(cudaMalloc(&g.prof, 32 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(g.prof, 0, 32 * sizeof(unsigned long long), st));
    }
    tm_store* ms = const_cast<tm_store*>(s);
    float2* rsum = static_cast<float2*>(ms->rsum.get(size_t(grid) * g.nmma * g.nh3 * TC_ROWS * sizeof(float2)));
    // B = sb x (x) U3 for the pass (sb from max |x|), 4 fp16 planes [pl][q][nt][kpad]
    float* wmax = static_cast<float*>(ms->scal.get(2 * sizeof(float))) + 1;  // max |x| of the pass
    CK(cudaMemsetAsync(wmax, 0, sizeof(float), st));
    xmax_kernel<<<unsigned(std::min<int64_t>((s->ncols * p + 255) / 256, 1184)), 256, 0, st>>>(x, ldx, s->ncols, p,
                                                                                              wmax);
    launched(cudaSuccess, "xmax_kernel");
    const size_t xbbytes = size_t(TC_FPLANES) * s->q * size_t(g.nt) * s->kpad * sizeof(__half);
    void* prev = ms->xbplanes.p;
    __half* xb = static_cast<__half*>(ms->xbplanes.get(xbbytes));
    if (xb != prev || ms->xb_zeroed < xbbytes) {  // padding rows / K slots must hold finite values
        CK(cudaMemsetAsync(xb, 0, ms->xbplanes.bytes, st));
        ms->xb_zeroed = ms->xbplanes.bytes;
    }
    build_xb_kernel<<<unsigned(s->ncols * (ke - kb)), 256, 0, st>>>(
        s->d_desc, static_cast<const float2*>(s->d_arena), s->d_kofs, x, ldx, int(p), s->ncols, s->q, g.n3,
        int64_t(g.nt), s->kpad, wmax, s->d_tcd, xb, int64_t(kb) * s->ncols);
    launched(cudaSuccess, "build_xb_kernel");
    const CUtensorMap bmap = make_tmap_3d_f16(xb, uint64_t(s->kpad), uint64_t(g.nt), uint64_t(TC_FPLANES * s->q),
                                              uint64_t(s->kpad) * 2, uint64_t(g.nt) * s->kpad * 2, 16,
                                              uint32_t(g.nmma), CU_TENSOR_MAP_SWIZZLE_32B);
    // One launch per wave of `grid` tiles: every CTA starts its tile at the
    // same time, so the CTAs of one component stream its B planes (184 MB
    // per component at config 4, more than L2) in K-lockstep and share them
    // in L2.  A persistent schedule over all tiles drifts apart by the
    // per-component cost differences and re-reads B from HBM (725 GB per
    // config-4 forward, measured).
    const int64_t tpb = g.ntiles / g.q;  // tiles per component (all right-hand sides of the pass)
    const int64_t nv = s->nv();
    int64_t bdone = kb;
    const int span = g.nmma * g.nh3;
    const int64_t tend = int64_t(ke) * tpb;  // components [kb, ke): tiles [kb tpb, ke tpb)
    for (int64_t t0 = int64_t(kb) * tpb; t0 < tend; t0 += wave) {
        const int64_t tiles = std::min<int64_t>(tend - t0, wave);
        // A final partial wave splits each tile's columns into parts (partial tiles
        // to ypart, summed by fwd_split_reduce_kernel) so the launch fills the GPU.
        g.split = best_split(tiles, wave, int(std::min<int64_t>(8, std::max<int64_t>(1, s->ncols))));
        if (const char* e = std::getenv("TMB_FWD_NOSPLIT")) if (*e && *e != '0') g.split = 1;
        g.tile0 = t0;
        g.t_begin = 0;
        g.t_end = tiles * g.split;
        g.ypart = nullptr;
        if (g.split > 1)
            g.ypart = static_cast<float2*>(ms->ypart.get(size_t(tiles) * g.split * (1 + g.pair) * span * TC_ROWS *
                                                         sizeof(float2)));
        if (g.pair) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(TC_THREADS);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            launched(cudaLaunchKernelEx(&cfg, kfpair, bmap, wa ? s->warena_map : bmap,
                                        static_cast<const TcDesc*>(s->d_tcd),
                                        static_cast<const float2*>(s->d_varena),
                                        static_cast<const float2*>(s->d_u2arena), static_cast<const int*>(s->d_kc),
                                        static_cast<const int*>(s->d_kofs), g, x, ldx, y, ldy, rsum,
                                        static_cast<const float*>(wmax)),
                     "fwd_tc_kernel<pair>");
        } else {
            kfsingle<<<grid, TC_THREADS, smem, st>>>(bmap, wa ? s->warena_map : bmap, s->d_tcd, s->d_varena,
                                                     s->d_u2arena,
                                                                  s->d_kc, s->d_kofs, g, x, ldx, y, ldy, rsum, wmax);
            launched(cudaSuccess, "fwd_tc_kernel");
        }
        if (g.split > 1) {
            const int64_t n = tiles * (1 + g.pair) * span * TC_ROWS;
            fwd_split_reduce_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(g, tiles, y,
                                                                                                     ldy);
            launched(cudaSuccess, "fwd_split_reduce_kernel");
        }
        const int64_t bnow = (t0 + tiles) / tpb;
        if (hp && hp->block_done && bnow > bdone) hp->block_done(bdone, bnow, hc0, p, st);
        if (hp && hp->copy && bnow > bdone) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, st));
            CK(cudaStreamWaitEvent(hp->copy, ev, 0));
            CK(cudaEventDestroy(ev));
            for (int64_t k = bdone; k < bnow; ++k)  // component k of every right-hand side of the pass
                for (int64_t c = 0; c < p; ++c)
                    CK(cudaMemcpyAsync(static_cast<float2*>(hp->host) + hp->ldhost * (hc0 + c) + k * nv,
                                       y + ldy * c + k * nv, size_t(nv) * sizeof(float2), cudaMemcpyDeviceToHost,
                                       hp->copy));
        }
        if (hp) bdone = std::max(bdone, bnow);
    }
    if (g.prof) {  // wait profile: mean cycles per recording thread, per role
        unsigned long long h[32];
        CK(cudaMemcpyAsync(h, g.prof, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaFree(g.prof));
        static const char* names[5] = {"tma", "mma", "loader", "producers", "fold"};
        static const char* w1[5] = {"empty", "cfree", "fempty", "ffull", "cfull"};
        static const char* w2[5] = {"-", "full", "-", "empty", "-"};
        for (int r = 0; r < 5; ++r)
            std::fprintf(stderr, "[tc-prof] %-9s total %14llu  wait %-6s %14llu  wait %-5s %14llu\n", names[r], h[3 * r],
                         w1[r], h[3 * r + 1], w2[r], h[3 * r + 2]);
    }
}

// The tensor-core forward: passes of up to pbmax right-hand sides (the B
// operand of a pass is 4 q n3 kpad fp16 per right-hand side).
void run_forward_tc(const tm_store* s, const float2* x, int64_t ldx, int64_t p, float2* y, int64_t ldy,
                    cudaStream_t st, const HostPipe* hp = nullptr, int kb = 0, int ke = -1) {
    if (ke < 0) ke = s->q;
    const size_t per_rhs = size_t(TC_FPLANES) * s->q * size_t(s->dims[2]) * s->kpad * sizeof(__half);
    size_t cap = size_t(4) << 30;  // B-operand budget per pass (TMB_XB_CAP_MB overrides, e.g. for tests)
    if (const char* e = std::getenv("TMB_XB_CAP_MB")) if (std::atoll(e) > 0) cap = size_t(std::atoll(e)) << 20;
    const int64_t pbmax = std::max<int64_t>(1, std::min<int64_t>(p, int64_t(cap / per_rhs)));
    for (int64_t c0 = 0; c0 < p; c0 += pbmax) {
        const int64_t pb = std::min<int64_t>(pbmax, p - c0);
        run_forward_pass(s, x + ldx * c0, ldx, pb, y + ldy * c0, ldy, st, hp, c0, kb, ke);
    }
}

// K3W (tm_k3w_tc.cuh): the batched forward of a W-arena store at the
// algorithmic cost (T decompressed once per tile from the arena on CUDA
// cores, Y += T X on tcgen05), for p >= TMB_K3_PMIN (default 16) right-hand
// sides and r3 <= 16; TMB_K3=0 disables it (the x-in-B arena forward).
bool k3w_ok(const tm_store* s, int64_t p) {
    if (!s->d_warena || warena_disabled() || tc_disabled() || s->rmax[2] > 16 || s->ncols >= (int64_t(1) << 25))
        return false;
    if (const char* e = std::getenv("TMB_K3")) if (*e == '0') return false;
    int64_t pmin = 16;
    if (const char* e = std::getenv("TMB_K3_PMIN")) if (std::atoll(e) > 0) pmin = std::atoll(e);
    return p >= pmin;
}

void ensure_k3w(tm_store* s, cudaStream_t st) {
    if (s->d_k3pa) return;
    const int64_t n3 = s->dims[2], m = s->ncols;
    const int nt3 = int((n3 + K3_NI3 - 1) / K3_NI3);
    // K3W's slot stream (tm_k3w_tc.cuh): columns back to back, at most two
    // overlapping a 16-slot stage; flags per stage: bit 0 half 1 present,
    // bit 1 it ends in the stage, bit 2 half 0 continues the previous stage
    std::vector<int> poff(size_t(s->q * m)), kc8(size_t(s->q));
    std::vector<std::vector<uint32_t>> flags(size_t(s->q));
    std::vector<std::vector<int2>> sdesc(size_t(s->q));
    std::vector<std::vector<int>> cends(size_t(s->q), std::vector<int>(size_t(m)));  // stage where column j ends
    int64_t kpad8 = 16;
    for (int k = 0; k < s->q; ++k) {
        int64_t pos = 0;
        auto& fk = flags[size_t(k)];
        auto& dk = sdesc[size_t(k)];
        auto& cend = cends[size_t(k)];
        std::vector<int> over;  // columns overlapping each stage so far
        auto stage_at = [&](size_t stg) {
            if (stg >= fk.size()) {
                fk.resize(stg + 1, 0u);
                dk.resize(stg + 1, make_int2(-1, -1));
                over.resize(stg + 1, 0);
            }
        };
        for (int64_t j = 0; j < m; ++j) {
            const int r3 = s->ranks[size_t((j * s->q + k) * 3 + 2)];
            size_t s0 = size_t(pos / 16);
            stage_at(s0);
            if (over[s0] == 2) {  // a third column would overlap the stage: start the next one
                pos = int64_t(s0 + 1) * 16;
                s0 = size_t(pos / 16);
                stage_at(s0);
            }
            const int64_t end = pos + r3 - 1;
            const size_t s1 = size_t(end / 16);
            const int t = int(k * m + j);
            if (over[s0] == 0) {
                dk[s0].x = t;  // half 0: ends in this stage (it starts at slot 0)
            } else {
                dk[s0].y = t;  // half 1
                fk[s0] |= 1u;
                if (s1 == s0) fk[s0] |= 2u;
            }
            ++over[s0];
            if (s1 > s0) {  // continues as half 0 of the next stage
                stage_at(s1);
                dk[s1].x = t;
                fk[s1] |= 4u;
                over[s1] = 1;
            }
            cend[size_t(j)] = int(s1);
            poff[size_t(t)] = int(pos);
            pos = end + 1;
        }
        kc8[size_t(k)] = int(pos);
        kpad8 = std::max<int64_t>(kpad8, (pos + 15) / 16 * 16);
    }
    if (kpad8 >= (int64_t(1) << 30)) throw TmError(TM_CAPACITY_ERROR, "K3W: slot stream too long");
    const int64_t nstg = kpad8 / 16;
    // gend[k][kk]: the W stages through the one where column 16 (kk + 1) - 1 ends
    const int64_t nks = (m + 15) / 16;
    std::vector<int> gend(size_t(s->q * nks), 0);
    for (int k = 0; k < s->q; ++k)
        for (int64_t kk = 0; kk < nks; ++kk)
            gend[size_t(k * nks + kk)] = cends[size_t(k)][size_t(std::min<int64_t>(16 * (kk + 1), m) - 1)] + 1;
    std::vector<uint32_t> fl(size_t(s->q * nstg), 0u);
    std::vector<int2> sd(size_t(s->q * nstg), make_int2(-1, -1));
    for (int k = 0; k < s->q; ++k) {
        std::copy(flags[size_t(k)].begin(), flags[size_t(k)].end(), fl.begin() + k * nstg);
        std::copy(sdesc[size_t(k)].begin(), sdesc[size_t(k)].end(), sd.begin() + k * nstg);
    }
    const uint64_t rows_pad = uint64_t(s->warena_rows), kp = uint64_t(kpad8);
    const size_t pab = size_t(4) * s->q * rows_pad * kp * sizeof(__half);
    const size_t b1b = size_t(s->q) * size_t(nstg) * size_t(nt3) * K3_B1_BYTES;
    int* d_poff = nullptr;
    int2* d_sd = nullptr;
    CK(cudaMalloc(&s->d_k3pa, pab));
    CK(cudaMalloc(&s->d_k3b1, b1b));
    CK(cudaMalloc(&s->d_k3flag, fl.size() * sizeof(uint32_t)));
    CK(cudaMalloc(&s->d_k3kc, kc8.size() * sizeof(int)));
    CK(cudaMalloc(&s->d_k3gend, gend.size() * sizeof(int)));
    CK(cudaMemcpy(s->d_k3gend, gend.data(), gend.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&d_poff, poff.size() * sizeof(int)));
    CK(cudaMalloc(&d_sd, sd.size() * sizeof(int2)));
    s->device_bytes += int64_t(pab + b1b + fl.size() * 4 + kc8.size() * 4);
    s->k3_kpad8 = kpad8;
    CK(cudaMemcpy(s->d_k3flag, fl.data(), fl.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s->d_k3kc, kc8.data(), kc8.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_poff, poff.data(), poff.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sd, sd.data(), sd.size() * sizeof(int2), cudaMemcpyHostToDevice));
    CK(cudaMemsetAsync(s->d_k3pa, 0, pab, st));
    build_k3w_pa_kernel<<<unsigned(s->q * m), 256, 0, st>>>(s->d_desc, s->d_kofs, d_poff, m, s->q, s->d_warena,
                                                           int64_t(rows_pad), s->kpad, nstg,
                                                           reinterpret_cast<unsigned char*>(s->d_k3pa));
    launched(cudaSuccess, "build_k3w_pa_kernel");
    build_k3w_b1_kernel<<<unsigned(s->q * nstg * nt3), 256, 0, st>>>(
        s->d_desc, s->d_tcd, static_cast<const float2*>(s->d_arena), d_sd, d_poff, int(n3), nt3, nstg, s->d_k3b1);
    launched(cudaSuccess, "build_k3w_b1_kernel");
    CK(cudaStreamSynchronize(st));
    CK(cudaFree(d_poff));
    CK(cudaFree(d_sd));
}

void run_forward_k3w(tm_store* s, const float2* x, int64_t ldx, int64_t p, float2* y, int64_t ldy, cudaStream_t st,
                     const HostPipe* hp = nullptr) {
    ensure_k3w(s, st);
    K3Geom g{};
    g.ncols = s->ncols;
    g.n1 = int(s->dims[0]);
    g.n2 = int(s->dims[1]);
    g.n3 = int(s->dims[2]);
    g.q = s->q;
    g.nt1 = (g.n1 + TC_TI1 - 1) / TC_TI1;
    g.nt2 = (g.n2 + TC_TI2 - 1) / TC_TI2;
    g.nt3 = (g.n3 + K3_NI3 - 1) / K3_NI3;
    g.ntiles = int64_t(g.q) * g.nt1 * g.nt2 * g.nt3;
    g.nks = int((s->ncols + 15) / 16);
    g.chain = tc_chain();
    // |T| <= r3 max |arena| < r3 2^14 (|U3 2^-e3| <= 1): T 2^-ceil(log2 r3) stays below 2^14
    int lr = 0;
    while ((1 << lr) < s->rmax[2]) ++lr;
    // D1 = 2^12 wsc T (B1 carries U3 2^12): tsc takes it below 2^14, the epilogue undoes wsc x tsc x sb
    g.tsc = ldexpf(1.f, -12 - lr);
    g.wsc = fp16_scale(s->vmax * 1.0001f) * TC_U3_SCALE;
    const size_t smem = 1024 + size_t(K3_NST) * (K3_A_STAGE + K3_B_STAGE) + size_t(K3_NWS) * K3_W_STAGE +
                        (2 * K3_NST + 2 * K3_NWS + 2 * K3_ND1 + 2) * 8 + 16;
    if (smem > kSmemMax) throw TmError(TM_CAPACITY_ERROR, "K3W forward: shared-memory plan too large");
    CK(cudaFuncSetAttribute(fwd_k3w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const unsigned grid = unsigned(std::min<int64_t>(g.ntiles, num_sms(dev)));
    float* rsum = static_cast<float*>(s->rsum.get(size_t(grid) * K3_YCOLS * TC_ROWS * sizeof(float)));
    const int64_t kpad = (s->ncols + 15) / 16 * 16;
    __half* planes = static_cast<__half*>(s->xbplanes.get(size_t(4) * 2 * K3_P * kpad * sizeof(__half)));
    float* xmax = static_cast<float*>(s->scal.get(2 * sizeof(float))) + 1;
    for (int64_t c0 = 0; c0 < p; c0 += K3_P) {
        const int pb = int(std::min<int64_t>(K3_P, p - c0));
        CK(cudaMemsetAsync(xmax, 0, sizeof(float), st));
        xmax_kernel<<<unsigned(std::min<int64_t>((s->ncols * pb + 255) / 256, 1184)), 256, 0, st>>>(
            x + ldx * c0, ldx, s->ncols, pb, xmax);
        launched(cudaSuccess, "xmax_kernel");
        k3_xplanes_kernel<<<unsigned(std::min<int64_t>((K3_P * kpad + 255) / 256, 4096)), 256, 0, st>>>(
            x + ldx * c0, ldx, s->ncols, pb, kpad, xmax, planes);
        launched(cudaSuccess, "k3_xplanes_kernel");
        const CUtensorMap xmap = make_tmap_3d_f16(planes, uint64_t(kpad), uint64_t(2 * K3_P), 4, uint64_t(kpad) * 2,
                                                  uint64_t(2 * K3_P) * kpad * 2, 16, 2 * K3_P,
                                                  CU_TENSOR_MAP_SWIZZLE_32B);
        g.p = pb;
        // TM_HOST (hp->copy): one launch per component, each component's y block copied
        // out on the copy stream while the next one computes (tiles are component-major)
        const bool pipe = hp && hp->copy;
        const int nl = pipe ? g.q : 1;
        const int64_t tpl = g.ntiles / nl;
        for (int l = 0; l < nl; ++l) {
            K3Geom gl = g;
            gl.tile0 = int64_t(l) * tpl;
            gl.ntiles = tpl;
            fwd_k3w_kernel<<<unsigned(std::min<int64_t>(tpl, grid)), K3_THREADS, smem, st>>>(
                xmap, reinterpret_cast<const unsigned char*>(s->d_k3pa), s->d_k3b1, s->d_k3kc, s->d_k3flag,
                s->k3_kpad8 / 16, s->d_k3gend, gl, y + ldy * c0, ldy, rsum, xmax);
            launched(cudaSuccess, "fwd_k3w_kernel");
            if (pipe) {
                const int64_t nv = s->nv();
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, st));
                CK(cudaStreamWaitEvent(hp->copy, ev, 0));
                CK(cudaEventDestroy(ev));
                CK(cudaMemcpy2DAsync(static_cast<float2*>(hp->host) + hp->ldhost * c0 + int64_t(l) * nv,
                                     size_t(hp->ldhost) * sizeof(float2), y + ldy * c0 + int64_t(l) * nv,
                                     size_t(ldy) * sizeof(float2), size_t(nv) * sizeof(float2), size_t(pb),
                                     cudaMemcpyDeviceToHost, hp->copy));
            }
        }
    }
}

void forward_dev(tm_store* s, const void* x, int64_t ldx, int64_t p, void* y, int64_t ldy, cudaStream_t st,
                 const HostPipe* hook = nullptr, int kb = 0, int ke = -1) {
    if (ke < 0) ke = s->q;
    if (!hook && kb == 0 && ke == s->q && k3w_ok(s, p)) {
        run_forward_k3w(s, static_cast<const float2*>(x), ldx, p, static_cast<float2*>(y), ldy, st);
        return;
    }
    if (s->tc_ok && !tc_disabled()) {
        run_forward_tc(s, static_cast<const float2*>(x), ldx, p, static_cast<float2*>(y), ldy, st, hook, kb, ke);
        return;
    }
    struct AtEnd {  // the CUDA-core kernels finish every component at once
        const HostPipe* h;
        const tm_store* s;
        int64_t p;
        cudaStream_t st;
        ~AtEnd() noexcept(false) {
            if (h && h->block_done && std::uncaught_exceptions() == 0) h->block_done(kb, ke, 0, p, st);
        }
        int kb, ke;
    } at_end{hook, s, p, st, kb, ke};
    const int cn = pick_cn(s->dims[2]);
    if (s->dtype == TM_C64) {
        auto X = static_cast<const float2*>(x);
        auto Y = static_cast<float2*>(y);
        if (cn == 4) run_forward_cc<float2, 8, 4, 8, 8>(s, X, ldx, p, Y, ldy, st, kb, ke);
        else if (cn == 2) run_forward_cc<float2, 8, 2, 8, 8>(s, X, ldx, p, Y, ldy, st, kb, ke);
        else run_forward_cc<float2, 8, 1, 8, 8>(s, X, ldx, p, Y, ldy, st, kb, ke);
    } else {
        auto X = static_cast<const double2*>(x);
        auto Y = static_cast<double2*>(y);
        if (cn == 4) run_forward_cc<double2, 4, 4, 8, 8>(s, X, ldx, p, Y, ldy, st, kb, ke);
        else if (cn == 2) run_forward_cc<double2, 4, 2, 8, 8>(s, X, ldx, p, Y, ldy, st, kb, ke);
        else run_forward_cc<double2, 4, 1, 8, 8>(s, X, ldx, p, Y, ldy, st, kb, ke);
    }
}

// Shared-memory plan of adj_tc_kernel with `nst` A/B stages (the default
// ring, or 2 stages for stores with large rank-(r2, r3) factor slots).
size_t adj_tc_smem(const tm_store* s, int nst = AJ_NST) {
    const int u2_off = TC_SLOT_V + int(round16(uint32_t(TC_TI1 * s->rmax[1] * s->rmax[2] * 8)));
    const int slot = (u2_off + TC_TI2 * (s->rmax[1] | 1) * 8 + 127) / 128 * 128;
    return 1024 + size_t(nst) * (AJ_A_STAGE + AJ_B_STAGE) + size_t(TC_JR) * slot +
           size_t(2) * AJ_MAXCOLS * AJ_NPW * sizeof(float2) + (2 * nst + 2 * TC_JR + 4) * 8 + 16;
}

// The smallest tensor-core adjoint plan fits (2-stage ring)
bool adj_tc_fits(const tm_store* s) { return adj_tc_smem(s, 2) <= kSmemMax; }

// Chunk packing of the adjoint U3 planes for adj_tc2_kernel<NR> (ch = 128 / NR
// slots per chunk, whole columns per chunk; TcDesc.pad1 (ch 64) / pad2 (ch 32)
// = the column's slot inside its chunk), built once per chunk size.  Returns
// false when some column's r3 exceeds the chunk.
bool ensure_adj_pack(tm_store* s, int which) {
    const int ch = which == 0 ? 64 : 32;
    auto& ap = s->adjp[which];
    if (ap.ok) return true;
    if (s->rmax[2] > ch) return false;
    const int64_t ntens = s->ncols * s->q;
    // products still in flight read the descriptor table rewritten below
    CK(cudaEventSynchronize(s->done));
    std::vector<TcDesc> tcd(static_cast<size_t>(ntens));
    CK(cudaMemcpy(tcd.data(), s->d_tcd, tcd.size() * sizeof(TcDesc), cudaMemcpyDeviceToHost));
    std::vector<int> aslot(static_cast<size_t>(ntens), 0), nch(static_cast<size_t>(s->q), 0);
    std::vector<std::vector<int>> cst(static_cast<size_t>(s->q));
    int maxch = 0;
    for (int k = 0; k < s->q; ++k) {
        int fill = ch, chunk = -1;
        for (int64_t j = 0; j < s->ncols; ++j) {
            const size_t t = static_cast<size_t>(k * s->ncols + j);
            const int r3 = tcd[t].r3;
            if (fill + r3 > ch || cst[static_cast<size_t>(k)].empty()) {
                ++chunk;
                fill = 0;
                cst[static_cast<size_t>(k)].push_back(int(j));
            }
            aslot[t] = chunk * ch + fill;
            (which == 0 ? tcd[t].pad1 : tcd[t].pad2) = fill;
            fill += r3;
        }
        nch[static_cast<size_t>(k)] = chunk + 1;
        maxch = std::max(maxch, chunk + 1);
    }
    std::vector<int> cstart(static_cast<size_t>(s->q) * (maxch + 1), int(s->ncols));
    for (int k = 0; k < s->q; ++k)
        for (size_t n = 0; n < cst[static_cast<size_t>(k)].size(); ++n)
            cstart[static_cast<size_t>(k) * (maxch + 1) + n] = cst[static_cast<size_t>(k)][n];
    const int64_t n3 = s->dims[2], n3p = (n3 + 7) / 8 * 8;
    const int64_t nslots = int64_t(maxch) * ch;
    const size_t abytes = size_t(TC_BPLANES) * s->q * nslots * n3p * sizeof(__half);
    CK(cudaMalloc(&ap.d_aplanes, abytes));
    CK(cudaMalloc(&ap.d_nch, nch.size() * sizeof(int)));
    CK(cudaMalloc(&ap.d_cstart, cstart.size() * sizeof(int)));
    CK(cudaMemcpy(ap.d_nch, nch.data(), nch.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ap.d_cstart, cstart.data(), cstart.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s->d_tcd, tcd.data(), tcd.size() * sizeof(TcDesc), cudaMemcpyHostToDevice));
    CK(cudaMemset(ap.d_aplanes, 0, abytes));
    DevBuf as;
    int* d_as = static_cast<int*>(as.get(aslot.size() * sizeof(int)));
    CK(cudaMemcpy(d_as, aslot.data(), aslot.size() * sizeof(int), cudaMemcpyHostToDevice));
    build_adj_bplanes_kernel<<<unsigned(ntens), 256>>>(s->d_desc, static_cast<const float2*>(s->d_arena), d_as,
                                                       s->ncols, s->q, int(n3), int(n3p), nslots, s->d_tcd,
                                                       ap.d_aplanes);
    launched(cudaSuccess, "build_adj_bplanes_kernel");
    CK(cudaDeviceSynchronize());
    ap.bmap = make_tmap_3d_f16(ap.d_aplanes, uint64_t(n3), uint64_t(nslots), uint64_t(TC_BPLANES * s->q),
                               uint64_t(n3p) * 2, uint64_t(nslots) * n3p * 2, 16, uint32_t(ch),
                               CU_TENSOR_MAP_SWIZZLE_32B);
    ap.maxch = maxch;
    ap.nslots = nslots;
    s->device_bytes += int64_t(abytes + (nch.size() + cstart.size()) * sizeof(int));
    ap.ok = true;
    return true;
}

// Shared-memory plan of adj_tc2_kernel<NR, PAIR> (PAIR stages 4 of the 6 U3 planes' halves).
template <int NR>
size_t adj_group_smem(int slot_bytes, bool pair = false) {
    using P = A2<NR>;
    const size_t bstage = pair ? size_t(4) * P::B_PLANE : size_t(P::B_STAGE);
    return 1024 + size_t(P::NST) * (P::A_STAGE + bstage) + size_t(TC_JR) * slot_bytes +
           size_t(P::RED) * sizeof(float2) + (2 * P::NST + 2 * TC_JR + 4) * 8 + 16;
}

// One pass of adj_tc2_kernel<NR> over right-hand-side groups [grp0, grp0 + ngrp).
template <int NR>
void launch_adj_groups(tm_store* s, const AjGeom& g, const CUtensorMap& amap, int64_t grp0, int64_t ngrp,
                       const float* phimax, float2* part, int nsm, cudaStream_t st) {
    const auto& ap = s->adjp[NR == 2 ? 0 : 1];
    AjGeom g2 = g;  // g.pair: CTA pairs over two row tiles (nrt even), as the single-RHS kernel
    g2.maxch = ap.maxch;
    const int64_t tpg = int64_t(g.q) * (g.nrt >> g2.pair);  // (pair) tiles per group
    g2.ntiles = (grp0 + ngrp) * tpg;
    const size_t smem2 = adj_group_smem<NR>(g.slot_bytes, g2.pair != 0);
    if (smem2 > kSmemMax) throw TmError(TM_CAPACITY_ERROR, "tensor-core adjoint: shared-memory plan too large");
    const bool big = s->rmax[2] > 16;  // the r3 <= 32 instantiations
    auto k2pair = big ? adj_tc2_kernel<NR, true, true> : adj_tc2_kernel<NR, true>;
    auto k2single = big ? adj_tc2_kernel<NR, false, true> : adj_tc2_kernel<NR, false>;
    CK(cudaFuncSetAttribute(k2single, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
    CK(cudaFuncSetAttribute(k2pair, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
    const unsigned grid2 = g2.pair ? unsigned(std::min<int64_t>(2 * 8 * ngrp * tpg, nsm & ~1))
                                   : unsigned(std::min<int64_t>(8 * ngrp * tpg, nsm));
    const int64_t wave = g2.pair ? grid2 / 2 : grid2;
    for (int64_t t0 = grp0 * tpg; t0 < g2.ntiles; t0 += wave) {
        const int64_t tiles = std::min<int64_t>(g2.ntiles - t0, wave);
        g2.split = best_split(tiles, wave, 8);
        g2.tile0 = t0;
        g2.t_begin = 0;
        g2.t_end = tiles * g2.split;
        if (g2.pair) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid2);
            cfg.blockDim = dim3(AJ_THREADS);
            cfg.dynamicSmemBytes = smem2;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            launched(cudaLaunchKernelEx(&cfg, k2pair, amap, ap.bmap,
                                        static_cast<const TcDesc*>(s->d_tcd), static_cast<const float2*>(s->d_varena),
                                        static_cast<const float2*>(s->d_u2arena), static_cast<const int*>(ap.d_nch),
                                        static_cast<const int*>(ap.d_cstart), g2, static_cast<const float*>(phimax),
                                        part),
                     "adj_tc2_kernel<pair>");
        } else {
            k2single<<<grid2, AJ_THREADS, smem2, st>>>(amap, ap.bmap, s->d_tcd, s->d_varena,
                                                                        s->d_u2arena, ap.d_nch, ap.d_cstart, g2,
                                                                        phimax, part);
            launched(cudaSuccess, "adj_tc2_kernel");
        }
    }
}

bool adj_pack_fits(const tm_store* s, int nr, int slot_bytes) {
    return s->rmax[2] <= 128 / nr &&
           (nr == 4 ? adj_group_smem<4>(slot_bytes) : adj_group_smem<2>(slot_bytes)) <= kSmemMax;
}

void run_adjoint_tc(tm_store* s, const float2* phi, int64_t ldphi, int64_t p, float2* z, int64_t ldz,
                    cudaStream_t st, const HostPipe* hp = nullptr) {
    AjGeom g{};
    g.ncols = s->ncols;
    g.n1 = int(s->dims[0]);
    g.n2 = int(s->dims[1]);
    g.n3 = int(s->dims[2]);
    g.q = s->q;
    g.nt1 = (g.n1 + TC_TI1 - 1) / TC_TI1;
    g.nt2 = (g.n2 + TC_TI2 - 1) / TC_TI2;
    g.p = int(p);
    g.nrt = int64_t(g.nt1) * g.nt2;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const int nsm = num_sms(dev);
    {  // CTA-pair kernel (cta_group::2 over two row tiles): half the B reads per MMA
        const char* e = std::getenv("TMB_DISABLE_PAIR");
        g.pair = (!(e && *e && *e != '0') && g.nrt % 2 == 0 && nsm >= 2) ? 1 : 0;
    }
    g.ntiles = int64_t(p) * g.q * (g.nrt >> g.pair);
    g.rmax2 = s->rmax[1];
    g.rmax3 = s->rmax[2];
    g.u2_off = TC_SLOT_V + int(round16(uint32_t(TC_TI1 * g.rmax2 * g.rmax3 * 8)));
    g.slot_bytes = (g.u2_off + TC_TI2 * (g.rmax2 | 1) * 8 + 127) / 128 * 128;
    g.maxch = s->maxch;
    {
        const char* dbg = std::getenv("TMB_TC_DEBUG");
        g.debug = dbg ? std::atoi(dbg) : 0;
    }
    const size_t bstage = g.pair ? size_t(4) * AJ_B_PLANE : size_t(AJ_B_STAGE);
    auto smem_for = [&](int nst) {
        return 1024 + size_t(nst) * (AJ_A_STAGE + bstage) + size_t(TC_JR) * g.slot_bytes +
               size_t(2) * AJ_MAXCOLS * AJ_NPW * sizeof(float2) + (2 * nst + 2 * TC_JR + 4) * 8 + 16;
    };
    // the default ring, or a 2-stage ring when large factor slots leave no room for it
    const bool small_ring = smem_for(g.pair ? AJ_NST2 : AJ_NST) > kSmemMax;
    const size_t smem = smem_for(small_ring ? 2 : (g.pair ? AJ_NST2 : AJ_NST));
    if (smem > kSmemMax) throw TmError(TM_CAPACITY_ERROR, "tensor-core adjoint: shared-memory plan too large");
    // Phi -> scaled 2-term fp16 planes (per call)
    g.nks = (g.n3 + 15) / 16;
    const int64_t n3p = (g.n3 + 7) / 8 * 8;
    const int64_t R = g.nrt * TC_ROWS;
    if (int64_t(p) * g.q > 65535) throw TmError(TM_CAPACITY_ERROR, "tensor-core adjoint: too many right-hand sides");
    __half* planes = static_cast<__half*>(s->phiplanes.get(size_t(AJ_APLANES) * p * g.q * R * n3p * sizeof(__half)));
    const int64_t nblk = int64_t(p) * g.q;  // (rhs, component) blocks
    const int64_t nv = s->nv();
    float* scal = static_cast<float*>(s->scal.get(size_t(nblk + 2) * sizeof(float)));
    float* phimax = scal + 2;  // [p][q]
    CK(cudaMemsetAsync(phimax, 0, size_t(nblk) * sizeof(float), st));
    // prepare (absmax, split) blocks [b0, b1) of Phi on the compute stream
    auto prepare = [&](int64_t b0, int64_t b1) {
        if (b1 <= b0) return;
        absmax_kernel<<<dim3(148, unsigned(b1 - b0)), 256, 0, st>>>(phi, ldphi, nv, g.q, b0, phimax);
        launched(cudaSuccess, "absmax_kernel");
        dim3 sgrid(unsigned(g.nrt), unsigned((n3p + 31) / 32), unsigned(b1 - b0));
        adj_split_phi_kernel<<<sgrid, 256, 0, st>>>(phi, ldphi, g.n1, g.n2, g.n3, int(n3p), g.q, int(p), g.nt2,
                                                    g.nrt, b0, phimax, planes);
        launched(cudaSuccess, "adj_split_phi_kernel");
    };
    std::vector<cudaEvent_t> arrived;
    if (hp) {  // host Phi: copy every block in ahead of the waves, on the copy stream
        arrived.resize(size_t(nblk));
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t c = b / g.q, k = b - c * g.q;
            CK(cudaMemcpyAsync(const_cast<float2*>(phi) + ldphi * c + k * nv,
                               static_cast<const float2*>(hp->host) + hp->ldhost * c + k * nv,
                               size_t(nv) * sizeof(float2), cudaMemcpyHostToDevice, hp->copy));
            CK(cudaEventCreateWithFlags(&arrived[size_t(b)], cudaEventDisableTiming));
            CK(cudaEventRecord(arrived[size_t(b)], hp->copy));
        }
    } else {
        prepare(0, nblk);
    }
    const CUtensorMap amap = make_tmap_3d_f16(planes, uint64_t(g.n3), uint64_t(R), uint64_t(AJ_APLANES * p * g.q),
                                              uint64_t(n3p) * 2, uint64_t(R) * n3p * 2, 16, TC_ROWS,
                                              CU_TENSOR_MAP_SWIZZLE_32B);
    const int64_t nred = g.nrt * g.q;
    float2* part = static_cast<float2*>(s->part.get(size_t(s->ncols * p * nred) * sizeof(float2)));
    const bool big = s->rmax[2] > 16;  // the r3 <= 32 instantiations
    auto kpair = big ? (small_ring ? adj_tc_kernel<true, 2, true> : adj_tc_kernel<true, 0, true>)
                     : (small_ring ? adj_tc_kernel<true, 2> : adj_tc_kernel<true>);
    auto ksingle = big ? (small_ring ? adj_tc_kernel<false, 2, true> : adj_tc_kernel<false, 0, true>)
                       : (small_ring ? adj_tc_kernel<false, 2> : adj_tc_kernel<false>);
    CK(cudaFuncSetAttribute(ksingle, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CK(cudaFuncSetAttribute(kpair, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // (up to 8 parts per tile when there are fewer tiles than SMs: best_split)
    const unsigned grid = g.pair ? unsigned(std::min<int64_t>(2 * 8 * g.ntiles, nsm & ~1))
                                 : unsigned(std::min<int64_t>(8 * g.ntiles, nsm));
    const int64_t wave = g.pair ? grid / 2 : grid;
    const int64_t tpb = g.nrt >> g.pair;  // tiles per (rhs, component) block
    int64_t bready = hp ? 0 : nblk;
    // Right-hand-side groups (adj_tc2_kernel<NR>: W once for NR right-hand
    // sides): quads first, then a pair; an odd last right-hand side goes
    // through the single-RHS kernel below.  TMB_ADJ_NR = 1 / 2 / 4 caps NR.
    int64_t tfirst = 0;
    {
        int nrmax = 4;
        if (const char* e = std::getenv("TMB_ADJ_NR")) nrmax = std::atoi(e);
        if (const char* e = std::getenv("TMB_ADJ_NR1")) if (*e && *e != '0') nrmax = 1;
        const bool q4 = nrmax >= 4 && p >= 4 && adj_pack_fits(s, 4, g.slot_bytes) && ensure_adj_pack(s, 1);
        const int64_t quads = q4 ? p / 4 : 0;
        const bool q2 = nrmax >= 2 && p - 4 * quads >= 2 && adj_pack_fits(s, 2, g.slot_bytes) &&
                        ensure_adj_pack(s, 0);
        const int64_t pairs = q2 ? (p - 4 * quads) / 2 : 0;
        if (quads + pairs > 0) {
            for (; bready < nblk; ++bready) {  // every block of the pass is read by some wave
                CK(cudaStreamWaitEvent(st, arrived[size_t(bready)], 0));
                prepare(bready, bready + 1);
            }
            if (quads > 0) launch_adj_groups<4>(s, g, amap, 0, quads, phimax, part, nsm, st);
            // pairs start at right-hand side 4 quads = pair index 2 quads
            if (pairs > 0) launch_adj_groups<2>(s, g, amap, 2 * quads, pairs, phimax, part, nsm, st);
            tfirst = (4 * quads + 2 * pairs) * g.q * tpb;  // the remaining (odd) right-hand side's tiles
        }
    }
    for (int64_t t0 = tfirst; t0 < g.ntiles; t0 += wave) {  // one launch per wave (see run_forward_tc)
        const int64_t tiles = std::min<int64_t>(g.ntiles - t0, wave);
        // a final partial wave splits each tile's chunk range into parts so the
        // launch still fills the GPU (partials are per column: no extra reduction)
        g.split = best_split(tiles, wave, 8);
        if (const char* e = std::getenv("TMB_ADJ_NOSPLIT")) if (*e && *e != '0') g.split = 1;
        g.tile0 = t0;
        g.t_begin = 0;
        g.t_end = tiles * g.split;
        const int64_t bneed = (t0 + tiles - 1) / tpb + 1;  // blocks this wave reads
        for (; bready < bneed; ++bready) {
            CK(cudaStreamWaitEvent(st, arrived[size_t(bready)], 0));
            prepare(bready, bready + 1);
        }
        if (g.pair) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(AJ_THREADS);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            launched(cudaLaunchKernelEx(&cfg, kpair, amap, s->adj_bmap,
                                        static_cast<const TcDesc*>(s->d_tcd), static_cast<const float2*>(s->d_varena),
                                        static_cast<const float2*>(s->d_u2arena), static_cast<const int*>(s->d_nch),
                                        static_cast<const int*>(s->d_cstart), g, static_cast<const float*>(phimax),
                                        part),
                     "adj_tc_kernel<pair>");
        } else {
            ksingle<<<grid, AJ_THREADS, smem, st>>>(amap, s->adj_bmap, s->d_tcd, s->d_varena,
                                                                  s->d_u2arena, s->d_nch, s->d_cstart, g, phimax,
                                                                  part);
            launched(cudaSuccess, "adj_tc_kernel");
        }
    }
    for (cudaEvent_t e : arrived) CK(cudaEventDestroy(e));
    const int64_t warps = s->ncols * p;
    const unsigned blocks = unsigned((warps * 32 + 255) / 256);
    adj_reduce_kernel<float2><<<blocks, 256, 0, st>>>(part, s->ncols, p, nred, z, ldz);
    launched(cudaSuccess, "adj_reduce_kernel");
}

// The adjoint of a W-arena store as one GEMM per pass of right-hand sides:
// G = conj(W)^T Phi on fwd_tc_kernel<PAIR, false, true, true> (A = the
// transposed arena, B = Phi as row-contiguous fp16 planes from
// adjg_split_phi_kernel; M = slot tiles, N = (i3, c), K = rows), then
// adjg_contract_kernel applies U3 and the scales.  The MACs are the forward
// arena kernel's (rows x n3 p x slots), with no consumer warps.
void run_adjoint_gemm(tm_store* s, const float2* phi, int64_t ldphi, int64_t p, float2* z, int64_t ldz,
                      cudaStream_t st, const HostPipe* hp = nullptr) {
    const int n1 = int(s->dims[0]), n2 = int(s->dims[1]), n3 = int(s->dims[2]);
    const int nt1r = (n1 + TC_TI1 - 1) / TC_TI1, nt2r = (n2 + TC_TI2 - 1) / TC_TI2;
    const int64_t R = int64_t(nt1r) * nt2r * TC_ROWS, nv = s->nv(), kt = s->wt_kpadt;
    // passes of pb right-hand sides: G (q n3 pb kt float2) and the Phi planes (4 q n3 pb R fp16) within budget
    const size_t per_rhs = std::max(size_t(s->q) * n3 * kt * sizeof(float2), size_t(4) * s->q * n3 * R * 2);
    const int64_t pbmax = std::max<int64_t>(1, std::min<int64_t>({p, int64_t((size_t(2) << 30) / per_rhs),
                                                                   int64_t(65535 / n3)}));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const int nsm = num_sms(dev);
    float* phimax = static_cast<float*>(s->scal.get(size_t(pbmax * s->q + 2) * sizeof(float))) + 2;
    for (int64_t c0 = 0; c0 < p; c0 += pbmax) {
        const int64_t pb = std::min<int64_t>(pbmax, p - c0);
        const float2* ph = phi + ldphi * c0;
        const int64_t nt = int64_t(n3) * pb;
        CK(cudaMemsetAsync(phimax, 0, size_t(pb * s->q) * sizeof(float), st));
        __half* planes = static_cast<__half*>(s->phit.get(size_t(4) * s->q * nt * R * sizeof(__half)));
        // TM_HOST (hp->copy): Phi arrives component by component on the copy stream and
        // each component's absmax and split run once it is in, ahead of the GEMM waves
        // that read it (split_upto); otherwise all components at once
        const bool pipe = hp && hp->copy;
        std::vector<cudaEvent_t> arrived;
        int ksplit = 0;
        auto split_upto = [&](int kend) {
            for (; ksplit < kend; ++ksplit) {
                CK(cudaStreamWaitEvent(st, arrived[size_t(ksplit)], 0));
                absmax_comp_kernel<<<dim3(148, unsigned(pb)), 256, 0, st>>>(ph, ldphi, nv, s->q, ksplit, phimax);
                launched(cudaSuccess, "absmax_comp_kernel");
                adjg_split_phi_kernel<<<dim3(unsigned(nt1r * nt2r), unsigned(nt), 1u), TC_ROWS, 0, st>>>(
                    ph, ldphi, n1, n2, n3, int(pb), s->q, nt2r, R, nt, phimax, planes, ksplit);
                launched(cudaSuccess, "adjg_split_phi_kernel");
            }
        };
        if (pipe) {
            arrived.resize(size_t(s->q));
            for (int k = 0; k < s->q; ++k) {
                CK(cudaMemcpy2DAsync(const_cast<float2*>(ph) + int64_t(k) * nv, size_t(ldphi) * sizeof(float2),
                                     static_cast<const float2*>(hp->host) + hp->ldhost * c0 + int64_t(k) * nv,
                                     size_t(hp->ldhost) * sizeof(float2), size_t(nv) * sizeof(float2), size_t(pb),
                                     cudaMemcpyHostToDevice, hp->copy));
                CK(cudaEventCreateWithFlags(&arrived[size_t(k)], cudaEventDisableTiming));
                CK(cudaEventRecord(arrived[size_t(k)], hp->copy));
            }
        } else {
            absmax_kernel<<<dim3(148, unsigned(pb * s->q)), 256, 0, st>>>(ph, ldphi, nv, s->q, 0, phimax);
            launched(cudaSuccess, "absmax_kernel");
            adjg_split_phi_kernel<<<dim3(unsigned(nt1r * nt2r), unsigned(nt), unsigned(s->q)), TC_ROWS, 0, st>>>(
                ph, ldphi, n1, n2, n3, int(pb), s->q, nt2r, R, nt, phimax, planes, 0);
            launched(cudaSuccess, "adjg_split_phi_kernel");
        }
        TcGeom g{};
        g.ncols = s->ncols;
        g.n1 = n1;
        g.n2 = n2;
        g.n3 = n3;
        g.q = s->q;
        g.p = int(pb);
        g.nt = int(nt);
        g.nmma = std::min(TC_NMAX, (g.nt + 15) / 16 * 16);
        g.nh3 = g.nt > TC_NMAX ? 2 : 1;
        g.nt3 = (g.nt + g.nmma * g.nh3 - 1) / (g.nmma * g.nh3);
        g.nt1 = int(kt / TC_ROWS);  // slot tiles play the forward's i1 blocks (nt2 = 1)
        g.nt2 = 1;
        g.pair = (g.nmma == TC_NMAX && g.nh3 == 2 && g.nt1 % 2 == 0 && nsm >= 2) ? 1 : 0;
        if (g.pair) g.nt1 /= 2;
        g.ntiles = int64_t(g.q) * g.nt3 * g.nt2 * g.nt1;
        g.b_stage = (g.pair ? 1 : g.nh3) * TC_FPLANES * g.nmma * 32;
        g.chain = tc_chain();
        g.gslots = kt;
        g.split = 1;
        auto smem_for = [&](int nst) {
            return 1024 + size_t(nst) * (TC_A_STAGE + g.b_stage) + (2 * TC_NST_MAX + 2 * TC_JR + 2) * 8 + 16;
        };
        g.nst = TC_NST_MAX;
        while (g.nst > 2 && smem_for(g.nst) > kSmemMax) --g.nst;
        const size_t smem = smem_for(g.nst);
        auto kpair = fwd_tc_kernel<true, false, true, true>;
        auto ksingle = fwd_tc_kernel<false, false, true, true>;
        CK(cudaFuncSetAttribute(ksingle, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaFuncSetAttribute(kpair, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const unsigned grid = g.pair ? unsigned(std::min<int64_t>(2 * g.ntiles, nsm & ~1))
                                     : unsigned(std::min<int64_t>(g.ntiles, nsm));
        const int64_t wave = g.pair ? grid / 2 : grid;
        float2* rsum =
            static_cast<float2*>(s->rsum.get(size_t(grid) * g.nmma * g.nh3 * TC_ROWS * sizeof(float2)));
        float2* G = static_cast<float2*>(s->gbuf.get(size_t(s->q) * nt * kt * sizeof(float2)));
        const CUtensorMap bmap = make_tmap_3d_f16(planes, uint64_t(R), uint64_t(nt), uint64_t(TC_FPLANES * s->q),
                                                  uint64_t(R) * 2, uint64_t(nt) * R * 2, 16, uint32_t(g.nmma),
                                                  CU_TENSOR_MAP_SWIZZLE_32B);
        for (int64_t t0 = 0; t0 < g.ntiles; t0 += wave) {  // one launch per wave (see run_forward_pass)
            const int64_t tiles = std::min<int64_t>(g.ntiles - t0, wave);
            // a final partial wave splits each tile's K (row) stages into parts:
            // partial G tiles to ypart, summed in part order by adjg_split_reduce_kernel
            g.split = best_split(tiles, wave, 8);
            if (const char* e = std::getenv("TMB_ADJ_NOSPLIT")) if (*e && *e != '0') g.split = 1;
            g.tile0 = t0;
            g.t_begin = 0;
            g.t_end = tiles * g.split;
            g.ypart = nullptr;
            if (g.split > 1)
                g.ypart = static_cast<float2*>(s->ypart.get(size_t(tiles) * g.split * (1 + g.pair) * g.nmma * g.nh3 *
                                                            TC_ROWS * sizeof(float2)));
            if (pipe) split_upto(int((t0 + tiles - 1) / (g.ntiles / g.q)) + 1);  // the components this wave reads
            if (g.pair) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(TC_THREADS);
                cfg.dynamicSmemBytes = smem;
                cfg.stream = st;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = 2;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                launched(cudaLaunchKernelEx(&cfg, kpair, bmap, s->wt_map, static_cast<const TcDesc*>(s->d_tcd),
                                            static_cast<const float2*>(s->d_varena),
                                            static_cast<const float2*>(s->d_u2arena), static_cast<const int*>(s->d_kcr),
                                            static_cast<const int*>(s->d_kofs), g, static_cast<const float2*>(nullptr),
                                            int64_t(0), G, int64_t(0), rsum, static_cast<const float*>(phimax)),
                         "fwd_tc_kernel<pair, adjoint GEMM>");
            } else {
                ksingle<<<grid, TC_THREADS, smem, st>>>(bmap, s->wt_map, s->d_tcd, s->d_varena, s->d_u2arena,
                                                        s->d_kcr, s->d_kofs, g, nullptr, 0, G, 0, rsum, phimax);
                launched(cudaSuccess, "fwd_tc_kernel<adjoint GEMM>");
            }
            if (g.split > 1) {
                const int64_t n = tiles * (1 + g.pair) * g.nmma * g.nh3 * TC_ROWS;
                adjg_split_reduce_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(g, tiles,
                                                                                                           G);
                launched(cudaSuccess, "adjg_split_reduce_kernel");
            }
        }
        if (pipe) split_upto(s->q);
        float* kmax = static_cast<float*>(s->gkmax.get(size_t(s->q) * sizeof(float)));
        phimax_k_kernel<<<1, 256, 0, st>>>(phimax, int(pb), s->q, kmax);
        launched(cudaSuccess, "phimax_k_kernel");
        adjg_contract_kernel<<<unsigned(s->ncols), 256, 0, st>>>(
            G, kt, nt, int(pb), s->q, s->ncols, n3, s->d_tcd, static_cast<const float2*>(s->d_arena), s->d_kofs,
            kmax, fp16_scale(s->vmax * 1.0001f), z + ldz * c0, ldz);
        launched(cudaSuccess, "adjg_contract_kernel");
        for (auto ev : arrived) CK(cudaEventDestroy(ev));
    }
}

void adjoint_dev(tm_store* s, const void* phi, int64_t ldphi, int64_t p, void* z, int64_t ldz, cudaStream_t st) {
    if (s->ncols == 0 || p == 0) return;
    if (s->d_wt && !warena_disabled() && !adjg_disabled() && !tc_disabled()) {
        run_adjoint_gemm(s, static_cast<const float2*>(phi), ldphi, p, static_cast<float2*>(z), ldz, st);
        return;
    }
    if (s->tca_ok && !tc_disabled() && adj_tc_fits(s) && int64_t(p) * s->q <= 65535) {
        run_adjoint_tc(s, static_cast<const float2*>(phi), ldphi, p, static_cast<float2*>(z), ldz, st);
        return;
    }
    const int cn = pick_cn(s->dims[2]);
    if (s->dtype == TM_C64) {
        auto P = static_cast<const float2*>(phi);
        auto Z = static_cast<float2*>(z);
        if (cn == 4) run_adjoint_cc<float2, 8, 4, 8, 8>(s, P, ldphi, p, Z, ldz, st);
        else if (cn == 2) run_adjoint_cc<float2, 8, 2, 8, 8>(s, P, ldphi, p, Z, ldz, st);
        else run_adjoint_cc<float2, 8, 1, 8, 8>(s, P, ldphi, p, Z, ldz, st);
    } else {
        auto P = static_cast<const double2*>(phi);
        auto Z = static_cast<double2*>(z);
        if (cn == 4) run_adjoint_cc<double2, 4, 4, 8, 8>(s, P, ldphi, p, Z, ldz, st);
        else if (cn == 2) run_adjoint_cc<double2, 4, 2, 8, 8>(s, P, ldphi, p, Z, ldz, st);
        else run_adjoint_cc<double2, 4, 1, 8, 8>(s, P, ldphi, p, Z, ldz, st);
    }
}

void aca_vhx_dev(const tm_store* s, const void* x, int64_t ldx, int64_t p, void* w, cudaStream_t st) {
    const int64_t warps = s->ncols * p;
    if (warps == 0) return;
    const unsigned blocks = unsigned((warps * 32 + 255) / 256);
    if (s->dtype == TM_C64)
        aca_vhx_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<const float2*>(s->d_v), s->m2, s->ncols,
                                                       static_cast<const float2*>(x), ldx, p, static_cast<float2*>(w));
    else
        aca_vhx_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<const double2*>(s->d_v), s->m2, s->ncols,
                                                        static_cast<const double2*>(x), ldx, p,
                                                        static_cast<double2*>(w));
    launched(cudaSuccess, "aca_vhx_kernel");
}

void aca_vt_dev(const tm_store* s, const void* t, int64_t p, void* z, int64_t ldz, cudaStream_t st) {
    const int64_t n = s->m2 * p;
    if (n == 0) return;
    const unsigned blocks = unsigned((n + 255) / 256);
    if (s->dtype == TM_C64)
        aca_vt_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<const float2*>(s->d_v), s->m2, s->ncols,
                                                      static_cast<const float2*>(t), p, static_cast<float2*>(z), ldz);
    else
        aca_vt_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<const double2*>(s->d_v), s->m2, s->ncols,
                                                       static_cast<const double2*>(t), p, static_cast<double2*>(z),
                                                       ldz);
    launched(cudaSuccess, "aca_vt_kernel");
}

// Dense-U ACA products (aca_forward's `fac.dense_u * w` and aca_adjoint's
// `fac.dense_u.adjoint() * phi`, src/matvec.cpp:158,173) on the device: the
// same two reduction kernels as the V side, with U (m1 x r) in V's place.
void dense_u_times(const tm_store* s, const void* t, int64_t p, void* y, int64_t ldy, cudaStream_t st) {
    const int64_t m1 = s->dims[0], n = m1 * p;
    if (n == 0) return;
    const unsigned blocks = unsigned((n + 255) / 256);
    if (s->dtype == TM_C64)
        aca_vt_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<const float2*>(s->d_u), m1, s->ncols,
                                                      static_cast<const float2*>(t), p, static_cast<float2*>(y), ldy);
    else
        aca_vt_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<const double2*>(s->d_u), m1, s->ncols,
                                                       static_cast<const double2*>(t), p, static_cast<double2*>(y),
                                                       ldy);
    launched(cudaSuccess, "aca_vt_kernel<dense U>");
}

void dense_uh_times(const tm_store* s, const void* phi, int64_t ldphi, int64_t p, void* t, cudaStream_t st) {
    const int64_t warps = s->ncols * p;
    if (warps == 0) return;
    const unsigned blocks = unsigned((warps * 32 + 255) / 256);
    if (s->dtype == TM_C64)
        aca_vhx_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<const float2*>(s->d_u), s->dims[0], s->ncols,
                                                       static_cast<const float2*>(phi), ldphi, p,
                                                       static_cast<float2*>(t));
    else
        aca_vhx_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<const double2*>(s->d_u), s->dims[0], s->ncols,
                                                        static_cast<const double2*>(phi), ldphi, p,
                                                        static_cast<double2*>(t));
    launched(cudaSuccess, "aca_vhx_kernel<dense U>");
}

// complex128 host or device block -> the store's dtype, into fresh device memory
void* upload_converted(const tm_store* s, const double* src, int64_t n, bool on_device) {
    void* dst = nullptr;
    CK(cudaMalloc(&dst, size_t(std::max<int64_t>(n, 1)) * s->csize()));
    if (n == 0) return dst;
    DevBuf st;
    const double2* d = reinterpret_cast<const double2*>(src);
    if (!on_device) {
        void* p = st.get(size_t(n) * sizeof(double2));
        CK(cudaMemcpy(p, src, size_t(n) * sizeof(double2), cudaMemcpyHostToDevice));
        d = static_cast<const double2*>(p);
    }
    const unsigned grid = unsigned(std::min<int64_t>((n + 255) / 256, 4096));
    if (s->dtype == TM_C64)
        convert_kernel<float2><<<grid, 256>>>(d, n, static_cast<float2*>(dst));
    else
        convert_kernel<double2><<<grid, 256>>>(d, n, static_cast<double2*>(dst));
    launched(cudaSuccess, "convert_kernel");
    CK(cudaDeviceSynchronize());
    return dst;
}

void reject_dense(const tm_store* s, const char* what) {
    if (s->dense)
        contract(std::string(what) + ": the store holds a dense ACA U (no Tucker columns); use the aca products");
}

void zero_dev(const tm_store* s, void* y, int64_t rows, int64_t p, int64_t ldy, cudaStream_t st) {
    if (rows * p == 0) return;
    const unsigned blocks = unsigned(std::min<int64_t>((rows * p + 255) / 256, 8192));
    if (s->dtype == TM_C64)
        zero_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<float2*>(y), rows, p, ldy);
    else
        zero_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<double2*>(y), rows, p, ldy);
    launched(cudaSuccess, "zero_kernel");
}

// ------------------------------------------------------------ host staging --
// Runs `body(dev_in, ld_in, dev_out, ld_out)` with host-side in/out blocks
// staged through the store's work buffers on a private stream.
template <typename Body>
void with_host_io(tm_store* s, const void* in, int64_t ldin, int64_t inrows, int64_t p, void* out, int64_t ldout,
                  int64_t outrows, Body body) {
    const size_t cs = s->csize();
    void* din = s->xin.get(size_t(std::max<int64_t>(inrows * p, 1)) * cs);
    void* dout = s->yout.get(size_t(std::max<int64_t>(outrows * p, 1)) * cs);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
        order_after_prev(s, st);
        if (inrows * p > 0)
            CK(cudaMemcpy2DAsync(din, size_t(inrows) * cs, in, size_t(ldin) * cs, size_t(inrows) * cs, size_t(p),
                                 cudaMemcpyHostToDevice, st));
        body(din, inrows, dout, outrows, st);
        if (outrows * p > 0)
            CK(cudaMemcpy2DAsync(out, size_t(ldout) * cs, dout, size_t(outrows) * cs, size_t(outrows) * cs, size_t(p),
                                 cudaMemcpyDeviceToHost, st));
        mark_done(s, st);
        CK(cudaStreamSynchronize(st));
    } catch (...) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        throw;
    }
    CK(cudaStreamDestroy(st));
}

// TM_HOST products on the tensor-core path: host I/O overlapped with the
// kernels block by block (HostPipe).  Returns false when the product does
// not take the tensor-core path (the caller then uses with_host_io).
// `xrows` / `prep`: the ACA forward copies its x (m2 rows) in and forms w = V^H x
// on the device first (prep returns the device input of the column products).
bool forward_host_pipelined(tm_store* s, const void* x, int64_t ldx, int64_t p, void* y, int64_t ldy,
                            int64_t xrows = -1,
                            const std::function<const void*(const void*, cudaStream_t)>& prep = nullptr) {
    if (!(s->tc_ok && !tc_disabled())) return false;
    if (xrows < 0) xrows = s->ncols;
    const size_t cs = s->csize();
    void* din = s->xin.get(size_t(std::max<int64_t>(xrows * p, 1)) * cs);
    void* dout = s->yout.get(size_t(std::max<int64_t>(s->rows() * p, 1)) * cs);
    cudaStream_t st, cp;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
    auto done = [&]() {
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(cp);
        cudaStreamDestroy(st);
        cudaStreamDestroy(cp);
    };
    try {
        order_after_prev(s, st);
        order_after_prev(s, cp);
        CK(cudaMemcpy2DAsync(din, size_t(xrows) * cs, x, size_t(ldx) * cs, size_t(xrows) * cs, size_t(p),
                             cudaMemcpyHostToDevice, st));
        const float2* xin = static_cast<const float2*>(prep ? prep(din, st) : din);
        HostPipe hp;
        hp.copy = cp;
        hp.host = y;
        hp.ldhost = ldy;
        if (k3w_ok(s, p))
            run_forward_k3w(s, xin, s->ncols, p, static_cast<float2*>(dout), s->rows(), st, &hp);
        else
            run_forward_tc(s, xin, s->ncols, p, static_cast<float2*>(dout), s->rows(), st, &hp);
        mark_done(s, st);
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamSynchronize(cp));
    } catch (...) {
        done();
        throw;
    }
    done();
    return true;
}

// `zrows` / `post`: the ACA adjoint maps the column products t to z = V t (m2
// rows) on the device before the copy out (post returns the device z).
bool adjoint_host_pipelined(tm_store* s, const void* phi, int64_t ldphi, int64_t p, void* z, int64_t ldz,
                            int64_t zrows = -1,
                            const std::function<void*(void*, cudaStream_t)>& post = nullptr) {
    const bool gemm = s->d_wt && !warena_disabled() && !adjg_disabled() && !tc_disabled();  // adjoint_dev's choice
    if (!gemm && !(s->tca_ok && !tc_disabled() && adj_tc_fits(s) && int64_t(p) * s->q <= 65535)) return false;
    if (zrows < 0) zrows = s->ncols;
    const size_t cs = s->csize();
    void* din = s->xin.get(size_t(std::max<int64_t>(s->rows() * p, 1)) * cs);
    void* dout = s->yout.get(size_t(std::max<int64_t>(s->ncols * p, 1)) * cs);
    cudaStream_t st, cp;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
    auto done = [&]() {
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(cp);
        cudaStreamDestroy(st);
        cudaStreamDestroy(cp);
    };
    try {
        order_after_prev(s, st);
        order_after_prev(s, cp);
        HostPipe hp;
        hp.copy = cp;
        hp.host = const_cast<void*>(phi);
        hp.ldhost = ldphi;
        if (gemm)
            run_adjoint_gemm(s, static_cast<const float2*>(din), s->rows(), p, static_cast<float2*>(dout), s->ncols, st,
                             &hp);
        else
            run_adjoint_tc(s, static_cast<const float2*>(din), s->rows(), p, static_cast<float2*>(dout), s->ncols, st,
                           &hp);
        void* zdev = post ? post(dout, st) : dout;
        CK(cudaMemcpy2DAsync(z, size_t(ldz) * cs, zdev, size_t(zrows) * cs, size_t(zrows) * cs, size_t(p),
                             cudaMemcpyDeviceToHost, st));
        mark_done(s, st);
        CK(cudaStreamSynchronize(st));
    } catch (...) {
        done();
        throw;
    }
    done();
    return true;
}

void check_common(const tm_store* s, int64_t p, int64_t ldin, int64_t inrows, int64_t ldout, int64_t outrows,
                  int where, const void* in, const void* out) {
    if (!s) contract("null store");
    if (p < 0) contract("negative right-hand-side count");
    if (ldin < std::max<int64_t>(inrows, 1) && p > 0) contract("leading dimension of the input is too small");
    if (ldout < std::max<int64_t>(outrows, 1) && p > 0) contract("leading dimension of the output is too small");
    if (where != TM_HOST && where != TM_DEVICE) contract("where must be TM_HOST or TM_DEVICE");
    if (p > 0 && ((inrows > 0 && !in) || (outrows > 0 && !out))) contract("null input or output pointer");
}

}  // namespace

// ================================================================== C ABI ==
extern "C" {

TM_API int tm_version(void) { return 1; }

TM_API const char* tm_last_error(void) { return g_last_error.c_str(); }

void tmb_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

TM_API int64_t tm_launch_count(void) { return g_launches.load(); }

TM_API int tm_store_create(const tm_store_desc* desc, int device, int dtype, tm_store** out) {
    return guarded([&] {
        if (!desc || !out) contract("tm_store_create: null argument");
        *out = create_store(*desc, device, dtype);
    });
}

TM_API int tm_store_create_dense_aca(const double* u, int64_t m1, const double* v, int64_t m2, int64_t r,
                                     int on_device, int device, int dtype, tm_store** out) {
    return guarded([&] {
        if (!out) contract("tm_store_create_dense_aca: null argument");
        if (dtype != TM_C64 && dtype != TM_C128) contract("store: dtype must be TM_C64 or TM_C128");
        if (m1 < 1 || m2 < 1 || r < 0) contract("store: dense ACA needs m1, m2 >= 1 and r >= 0");
        if (r > 0 && (!u || !v)) contract("store: dense ACA needs U and V");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev)
            throw TmError(TM_CUDA_ERROR, "store: no CUDA device " + std::to_string(device));
        DeviceGuard guard(device);
        auto* s = new tm_store;
        try {
            CK(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
            s->device = device;
            s->dtype = dtype;
            s->dense = true;
            s->q = 1;
            s->ncols = r;
            s->dims[0] = m1;
            s->dims[1] = s->dims[2] = 1;
            s->m2 = m2;
            s->d_u = upload_converted(s, u, m1 * r, on_device != 0);
            s->d_v = upload_converted(s, v, m2 * r, on_device != 0);
            s->device_bytes = (m1 + m2) * r * int64_t(s->csize());
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

TM_API int tm_store_destroy(tm_store* s) {
    return guarded([&] {
        if (!s) return;
        DeviceGuard guard(s->device);
        delete s;
    });
}

TM_API int tm_store_info(const tm_store* s, int32_t* q, int64_t* ncols, int64_t* dims3, int32_t* dtype, int64_t* m2,
                         int64_t* device_bytes) {
    return guarded([&] {
        if (!s) contract("null store");
        if (q) *q = s->q;
        if (ncols) *ncols = s->ncols;
        if (dims3)
            for (int g = 0; g < 3; ++g) dims3[g] = s->dims[g];
        if (dtype) *dtype = s->dtype;
        if (m2) *m2 = s->m2;
        if (device_bytes) *device_bytes = s->device_bytes;
    });
}

TM_API int tm_store_kernels(const tm_store* s, int32_t* forward_tc, int32_t* adjoint_tc) {
    return guarded([&] {
        if (!s) contract("null store");
        const bool off = tc_disabled();
        if (forward_tc) *forward_tc = (s->tc_ok && !off) ? (s->d_warena && !warena_disabled() ? 2 : 1) : 0;
        if (adjoint_tc)
            *adjoint_tc = (s->d_wt && !warena_disabled() && !adjg_disabled() && !off) ? 3
                          : (s->tca_ok && !off && adj_tc_fits(s)) ? 1
                                                                  : 0;
    });
}

// assemble_column (src/scene.cpp:127-150) for a batch of source columns, on
// the device, complex128 (the GPU compressor's field evaluation, §8f-1).
// src: device pointer to m x 7 doubles {midpoint xyz, unit direction xyz,
// weight}; cols: host array of nb column indices; out: device pointer to nb
// x q x n_v complex128.  Enqueued on `stream` (NULL = legacy default) and
// synchronised only for the singularity check.
TM_API int tm_assemble_columns(const double* origin3, double spacing, const int64_t* dims3, int q, int op, double k0,
                               const double* src, int64_t m, const int64_t* cols, int64_t nb, void* out,
                               void* stream) {
    return guarded([&] {
        if (!origin3 || !dims3 || (nb > 0 && (!src || !cols || !out))) contract("tm_assemble_columns: null argument");
        if (q != 3 && q != 12) contract("tm_assemble_columns: q must be 3 (PWC) or 12 (PWL)");
        if (op != 0 && op != 1) contract("tm_assemble_columns: op must be 0 (E) or 1 (H)");
        if (!(spacing > 0)) contract("tm_assemble_columns: spacing must be positive");
        for (int g = 0; g < 3; ++g)
            if (dims3[g] < 1 || dims3[g] > (int64_t(1) << 30)) contract("tm_assemble_columns: bad grid dimension");
        for (int64_t b = 0; b < nb; ++b)
            if (cols[b] < 0 || cols[b] >= m) contract("tm_assemble_columns: column index out of range");
        if (nb == 0) return;
        if (nb > 65535) contract("tm_assemble_columns: at most 65535 columns per call");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        AsmScene sc{origin3[0], origin3[1], origin3[2], spacing, k0, int(dims3[0]), int(dims3[1]), int(dims3[2]), q, op};
        // per-thread scratch reused across calls (a cudaMalloc / cudaFree pair per
        // call costs more than the kernel for the ACA's one-voxel row batches)
        int dev = 0;
        CK(cudaGetDevice(&dev));
        static thread_local std::map<int, std::pair<DevBuf, DevBuf>> scratch;
        DevBuf& cb = scratch[dev].first;
        DevBuf& bb = scratch[dev].second;
        int64_t* d_cols = static_cast<int64_t*>(cb.get(size_t(nb) * sizeof(int64_t)));
        int* d_bad = static_cast<int*>(bb.get(sizeof(int)));
        CK(cudaMemcpyAsync(d_cols, cols, size_t(nb) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
        const int64_t nv = dims3[0] * dims3[1] * dims3[2];
        const unsigned gx = unsigned(std::min<int64_t>((nv + 255) / 256, 4096));
        assemble_kernel<<<dim3(gx, unsigned(nb)), 256, 0, st>>>(sc, src, d_cols, nb, static_cast<double2*>(out), d_bad);
        launched(cudaSuccess, "assemble_kernel");
        int hbad = 0;
        CK(cudaMemcpyAsync(&hbad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hbad) throw TmError(TM_SINGULARITY_ERROR, "field kernel: observation point hits the source");
    });
}

TM_API int tm_rows(tm_store* s, const int64_t* rows, int64_t nrows, void* out, int64_t ldout, int where,
                   void* stream) {
    return guarded([&] {
        if (!s) contract("null store");
        reject_dense(s, "tm_rows");
        if (nrows < 0) contract("negative row count");
        if (where != TM_HOST && where != TM_DEVICE) contract("where must be TM_HOST or TM_DEVICE");
        if (nrows > 0 && (!rows || !out)) contract("null rows or output pointer");
        if (nrows > 0 && ldout < nrows) contract("leading dimension of the output is too small");
        for (int64_t r = 0; r < nrows; ++r)
            if (rows[r] < 0 || rows[r] >= s->rows()) contract("element: index out of range");
        if (nrows == 0 || s->ncols == 0) return;
        if (nrows > 65535) contract("tm_rows: at most 65535 rows per call");
        std::lock_guard<std::mutex> lock(s->mu);
        DeviceGuard guard(s->device);
        const size_t cs = s->csize();
        cudaStream_t st = where == TM_DEVICE ? static_cast<cudaStream_t>(stream) : nullptr;
        bool own = false;
        if (where == TM_HOST) {
            CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            own = true;
        }
        try {
            order_after_prev(s, st);
            int64_t* d_rows = static_cast<int64_t*>(s->wbuf.get(size_t(nrows) * sizeof(int64_t)));
            CK(cudaMemcpyAsync(d_rows, rows, size_t(nrows) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            void* dout = where == TM_DEVICE ? out : s->yout.get(size_t(nrows * s->ncols) * cs);
            const int64_t ld = where == TM_DEVICE ? ldout : nrows;
            const dim3 grid(unsigned((s->ncols + 127) / 128), unsigned(nrows));
            if (s->dtype == TM_C64)
                rows_kernel<float2><<<grid, 128, 0, st>>>(s->d_desc, static_cast<const float2*>(s->d_arena), s->ncols,
                                                          s->dims[0], s->dims[1], s->nv(), d_rows,
                                                          static_cast<float2*>(dout), ld);
            else
                rows_kernel<double2><<<grid, 128, 0, st>>>(s->d_desc, static_cast<const double2*>(s->d_arena),
                                                           s->ncols, s->dims[0], s->dims[1], s->nv(), d_rows,
                                                           static_cast<double2*>(dout), ld);
            launched(cudaSuccess, "rows_kernel");
            if (where == TM_HOST)
                CK(cudaMemcpy2DAsync(out, size_t(ldout) * cs, dout, size_t(nrows) * cs, size_t(nrows) * cs,
                                     size_t(s->ncols), cudaMemcpyDeviceToHost, st));
            mark_done(s, st);
            CK(cudaStreamSynchronize(st));
        } catch (...) {
            if (own) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
            }
            throw;
        }
        if (own) CK(cudaStreamDestroy(st));
    });
}

TM_API int tm_opcounts(const tm_store* s, int64_t p, int64_t* dec, int64_t* acc) {
    return guarded([&] {
        if (!s) contract("null store");
        if (dec) *dec = s->dec_madds;
        if (acc) *acc = s->ncols * s->q * s->nv() * p;
    });
}

TM_API int tm_forward(tm_store* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y, int64_t ldy,
                      int where, void* stream, int64_t* ops) {
    return guarded([&] {
        if (!s) contract("null store");
        reject_dense(s, "forward");
        if (xrows != s->ncols)
            contract("forward: x has " + std::to_string(xrows) + " rows, expected m = " + std::to_string(s->ncols));
        check_common(s, p, ldx, xrows, ldy, s->rows(), where, x, y);
        std::lock_guard<std::mutex> lock(s->mu);
        DeviceGuard guard(s->device);
        if (p > 0) {
            if (where == TM_DEVICE) {
                order_after_prev(s, static_cast<cudaStream_t>(stream));
                forward_dev(s, x, ldx, p, y, ldy, static_cast<cudaStream_t>(stream));
                mark_done(s, static_cast<cudaStream_t>(stream));
            } else if (!forward_host_pipelined(s, x, ldx, p, y, ldy))
                with_host_io(s, x, ldx, xrows, p, y, ldy, s->rows(),
                             [&](void* din, int64_t ldi, void* dout, int64_t ldo, cudaStream_t st) {
                                 forward_dev(s, din, ldi, p, dout, ldo, st);
                             });
        }
        if (ops) {
            ops[0] += s->dec_madds;
            ops[1] += s->ncols * s->q * s->nv() * p;
        }
    });
}

TM_API int tm_forward_components(tm_store* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y,
                                 int64_t ldy, int32_t k0, int32_t k1, void* stream) {
    return guarded([&] {
        if (!s) contract("null store");
        reject_dense(s, "forward");
        if (xrows != s->ncols)
            contract("forward: x has " + std::to_string(xrows) + " rows, expected m = " + std::to_string(s->ncols));
        if (k0 < 0 || k1 > s->q || k0 > k1) contract("tm_forward_components: component range out of range");
        check_common(s, p, ldx, xrows, ldy, s->rows(), TM_DEVICE, x, y);
        std::lock_guard<std::mutex> lock(s->mu);
        DeviceGuard guard(s->device);
        if (p > 0 && k1 > k0) {
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            order_after_prev(s, st);
            forward_dev(s, x, ldx, p, y, ldy, st, nullptr, k0, k1);
            mark_done(s, st);
        }
    });
}

TM_API int tm_adjoint(tm_store* s, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z, int64_t ldz,
                      int where, void* stream, int64_t* ops) {
    return guarded([&] {
        if (!s) contract("null store");
        reject_dense(s, "adjoint");
        if (phirows != s->rows())
            contract("adjoint: phi has " + std::to_string(phirows) + " rows, expected q*n_v = " +
                     std::to_string(s->rows()));
        check_common(s, p, ldphi, phirows, ldz, s->ncols, where, phi, z);
        std::lock_guard<std::mutex> lock(s->mu);
        DeviceGuard guard(s->device);
        if (p > 0 && s->ncols > 0) {
            if (where == TM_DEVICE) {
                order_after_prev(s, static_cast<cudaStream_t>(stream));
                adjoint_dev(s, phi, ldphi, p, z, ldz, static_cast<cudaStream_t>(stream));
                mark_done(s, static_cast<cudaStream_t>(stream));
            } else if (!adjoint_host_pipelined(s, phi, ldphi, p, z, ldz))
                with_host_io(s, phi, ldphi, phirows, p, z, ldz, s->ncols,
                             [&](void* din, int64_t ldi, void* dout, int64_t ldo, cudaStream_t st) {
                                 adjoint_dev(s, din, ldi, p, dout, ldo, st);
                             });
        }
        if (ops) {
            ops[0] += s->dec_madds;
            ops[1] += s->ncols * s->q * s->nv() * p;
        }
    });
}

TM_API int tm_aca_forward(tm_store* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y, int64_t ldy,
                          int where, void* stream) {
    return guarded([&] {
        if (!s) contract("null store");
        if (!s->d_v) contract("aca_forward: store carries no ACA V factor");
        if (xrows != s->m2)
            contract("aca_forward: x has " + std::to_string(xrows) + " rows, expected " + std::to_string(s->m2));
        check_common(s, p, ldx, xrows, ldy, s->rows(), where, x, y);
        std::lock_guard<std::mutex> lock(s->mu);
        DeviceGuard guard(s->device);
        if (p == 0) return;
        auto body = [&](const void* xin, int64_t ldi, void* yout, int64_t ldo, cudaStream_t st) {
            if (s->ncols == 0) {
                zero_dev(s, yout, s->rows(), p, ldo, st);
                return;
            }
            void* w = s->wbuf.get(size_t(s->ncols * p) * s->csize());
            aca_vhx_dev(s, xin, ldi, p, w, st);
            if (s->dense)
                dense_u_times(s, w, p, yout, ldo, st);
            else
                forward_dev(s, w, s->ncols, p, yout, ldo, st);
        };
        if (where == TM_DEVICE) {
            order_after_prev(s, static_cast<cudaStream_t>(stream));
            body(x, ldx, y, ldy, static_cast<cudaStream_t>(stream));
            mark_done(s, static_cast<cudaStream_t>(stream));
        } else if (s->dense || s->ncols == 0 ||
                   !forward_host_pipelined(s, x, ldx, p, y, ldy, s->m2, [&](const void* xin, cudaStream_t st) {
                       void* w = s->wbuf.get(size_t(s->ncols * p) * s->csize());
                       aca_vhx_dev(s, xin, s->m2, p, w, st);
                       return static_cast<const void*>(w);
                   })) {
            with_host_io(s, x, ldx, xrows, p, y, ldy, s->rows(),
                         [&](void* din, int64_t ldi, void* dout, int64_t ldo, cudaStream_t st) {
                             body(din, ldi, dout, ldo, st);
                         });
        }
    });
}

TM_API int tm_aca_adjoint(tm_store* s, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z,
                          int64_t ldz, int where, void* stream) {
    return guarded([&] {
        if (!s) contract("null store");
        if (!s->d_v) contract("aca_adjoint: store carries no ACA V factor");
        if (phirows != s->rows())
            contract("aca_adjoint: phi has " + std::to_string(phirows) + " rows, expected " +
                     std::to_string(s->rows()));
        check_common(s, p, ldphi, phirows, ldz, s->m2, where, phi, z);
        std::lock_guard<std::mutex> lock(s->mu);
        DeviceGuard guard(s->device);
        if (p == 0) return;
        auto body = [&](const void* pin, int64_t ldi, void* zout, int64_t ldo, cudaStream_t st) {
            if (s->ncols == 0) {
                zero_dev(s, zout, s->m2, p, ldo, st);
                return;
            }
            void* t = s->wbuf.get(size_t(s->ncols * p) * s->csize());
            if (s->dense)
                dense_uh_times(s, pin, ldi, p, t, st);
            else
                adjoint_dev(s, pin, ldi, p, t, s->ncols, st);
            aca_vt_dev(s, t, p, zout, ldo, st);
        };
        if (where == TM_DEVICE) {
            order_after_prev(s, static_cast<cudaStream_t>(stream));
            body(phi, ldphi, z, ldz, static_cast<cudaStream_t>(stream));
            mark_done(s, static_cast<cudaStream_t>(stream));
        } else if (s->dense || s->ncols == 0 ||
                   !adjoint_host_pipelined(s, phi, ldphi, p, z, ldz, s->m2, [&](void* t, cudaStream_t st) {
                       void* zd = s->ypart.get(size_t(s->m2 * p) * s->csize());
                       aca_vt_dev(s, t, p, zd, s->m2, st);
                       return zd;
                   })) {
            with_host_io(s, phi, ldphi, phirows, p, z, ldz, s->m2,
                         [&](void* din, int64_t ldi, void* dout, int64_t ldo, cudaStream_t st) {
                             body(din, ldi, dout, ldo, st);
                         });
        }
    });
}

}  // extern "C"

#include "tm_shard.cuh"

// Streaming CTC1 / CTA1 ingest (tm_io.cpp): `d` carries the ranks (and V),
// the payload comes chunk by chunk from `fill`.
int tmb_io::create_store_streaming(const tm_store_desc* d, const PayloadFill& fill, int device, int dtype,
                                   tm_store** out) {
    return guarded([&] { *out = create_store(*d, device, dtype, &fill); });
}
