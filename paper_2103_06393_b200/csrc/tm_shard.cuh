// Multi-GPU column sharding at the C ABI: one host
// thread drives the GPUs of one box through a single-process NCCL
// communicator (ncclCommInitAll).
//
// The reference's stacked_forward sums private per-worker partials serially
// after all columns are done (src/matvec.cpp:30-38,58-59); here each GPU
// owns a contiguous, cost-balanced column range (a regular tm_store on its
// device) and the forward's partial y is reduced to the root GPU PER
// COMPONENT, on a communication stream, as soon as that component's waves
// have finished on every GPU — the reduce of component k overlaps the waves
// of components k + 1 ... (HostPipe::block_done).  The adjoint needs no
// reduction (rows of z are independent, src/matvec.cpp:78-96): Phi is
// broadcast, each GPU writes the z rows of its columns, and the rows are
// gathered to the root (ncclSend / ncclRecv) or copied straight to the
// host.  ACA stores shard U's columns with the matching columns of V: the
// forward reduces the partial y as above, the adjoint reduces the m2 x p
// partial V t.
//
// Row (voxel-slab) sharding, the alternative of SURVEY §8e (TM_SHARD_ROWS):
// the q * n1 (component, i1) slabs of the output are cut into one
// contiguous, cost-balanced range per GPU; a GPU holds each (component k,
// i1 rows [a, b)) piece of its range as a regular one-component store on the
// sub-grid (b - a) x n2 x n3 with all m columns (U1 rows sliced — the same
// operator restricted to those voxels).  The forward needs no reduction:
// each piece writes its rows of y (a strided copy from the piece's
// sub-grid layout, peer-to-peer for a device y on the root); the adjoint
// reads only its rows of Phi and reduces the m x p partial z (a few KB).
//
// A communicator whose device list repeats a device is EMULATED: the
// collectives become device-local copies and adds on the root's stream.
// That lets the sharded orchestration (column split, per-shard stores,
// per-component completion events, reduce / gather order) run and be
// tested on a single GPU; it is a functional check, never a measurement.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <memory>
#include <set>
#include <tuple>

#include "tm_aux_kernels.cuh"

struct tm_comm {
    std::vector<int> devices;
    bool emulated = false;
    std::vector<ncclComm_t> comms;
    ~tm_comm();
};

struct tm_sharded {
    tm_comm* comm = nullptr;  // products use its NCCL communicators
    std::vector<int> devices;  // own copy: destroying the store never touches the communicator
    int mode = TM_SHARD_COLUMNS;
    int dtype = TM_C64;
    int q = 0;
    int64_t ncols = 0, dims[3] = {0, 0, 0}, m2 = 0;
    std::vector<int64_t> c0, c1;  // columns: shard d's columns; rows: its (k n1 + i1) slab range
    std::vector<tm_store*> shards;  // columns mode: one store per device
    struct Piece {                   // rows mode: component k, i1 rows [a, b) on device index d
        size_t d = 0;
        int k = 0;
        int64_t a = 0, b = 0;
        tm_store* st = nullptr;
        DevBuf ybuf, pbuf, tbuf;  // piece output y, gathered Phi, partial adjoint
    };
    std::vector<Piece> pieces;
    std::vector<cudaStream_t> cst, mst;  // per shard: compute and communication streams
    std::vector<cudaEvent_t> done;       // per shard: end of the latest sharded product
    std::vector<DevBuf> xbuf, ybuf, zbuf;
    DevBuf zgather;
    std::mutex mu;
    int64_t nv() const { return dims[0] * dims[1] * dims[2]; }
    int64_t rows() const { return q * nv(); }
    size_t csize() const { return dtype == TM_C64 ? sizeof(float2) : sizeof(double2); }
    int dev(size_t d) const { return devices[d]; }
    size_t ndev() const { return devices.size(); }
    const tm_store* any_store() const { return mode == TM_SHARD_ROWS ? pieces.front().st : shards.front(); }
    ~tm_sharded() {
        for (size_t d = 0; d < done.size(); ++d)
            if (done[d]) {
                cudaSetDevice(dev(d));
                cudaEventSynchronize(done[d]);
            }
        for (Piece& pc : pieces) {
            cudaSetDevice(dev(pc.d));
            if (pc.st) delete pc.st;
            pc.ybuf.release();
            pc.pbuf.release();
            pc.tbuf.release();
        }
        for (size_t d = 0; d < ndev(); ++d) {
            cudaSetDevice(dev(d));
            if (d < done.size() && done[d]) cudaEventDestroy(done[d]);
            if (d < cst.size() && cst[d]) cudaStreamDestroy(cst[d]);
            if (d < mst.size() && mst[d]) cudaStreamDestroy(mst[d]);
            if (d < xbuf.size()) xbuf[d].release();
            if (d < ybuf.size()) ybuf[d].release();
            if (d < zbuf.size()) zbuf[d].release();
            if (d < shards.size() && shards[d]) delete shards[d];
        }
        cudaSetDevice(dev(0));
        zgather.release();
    }
};

namespace {

// NCCL is resolved at run time, on the first tm_comm_init: the library
// already loaded in the process if there is one (under Python, torch's
// bundled NCCL — linking the system libnccl.so.2 at build time would shadow
// it and break `import torch`), else $TMB_NCCL_LIB, else the system's
// libnccl.so.2.  Nothing in the single-GPU products touches NCCL.
struct Nccl {
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            if (const char* e = std::getenv("TMB_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            err = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
            return;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && err.empty()) err = std::string("NCCL symbol missing: ") + name;
        };
        sym(n.CommInitAll, "ncclCommInitAll");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.GetErrorString, "ncclGetErrorString");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.Reduce, "ncclReduce");
        sym(n.Broadcast, "ncclBroadcast");
        sym(n.Send, "ncclSend");
        sym(n.Recv, "ncclRecv");
    });
    if (!err.empty()) throw TmError(TM_CUDA_ERROR, err);
    return n;
}

}  // namespace

tm_comm::~tm_comm() {
    for (ncclComm_t c : comms)
        if (c) nccl().CommDestroy(c);
}

namespace {

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw TmError(TM_CUDA_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}
#define NCK(x) nck((x), #x)

// Contiguous column ranges of ~equal decompression cost (the reference's
// reconstruct_madds per column, src/matvec.cpp:10-15, plus the accumulate
// term): prefix-sum split, every shard at least one column when m >= ndev.
std::vector<int64_t> balanced_bounds(const tm_store_desc& d, int ndev) {
    const int64_t m = d.ncols, n1 = d.dims[0], n2 = d.dims[1], n3 = d.dims[2];
    std::vector<double> pre(static_cast<size_t>(m) + 1, 0.0);
    for (int64_t j = 0; j < m; ++j) {
        double c = 0;
        for (int k = 0; k < d.q; ++k) {
            const int32_t* r = d.ranks + 3 * (j * d.q + k);
            c += double(n1) * r[0] * r[1] * r[2] + double(n1) * n2 * r[1] * r[2] + double(n1) * n2 * n3 * r[2] +
                 double(n1) * n2 * n3;
        }
        pre[size_t(j) + 1] = pre[size_t(j)] + c;
    }
    std::vector<int64_t> b(static_cast<size_t>(ndev) + 1, m);
    b[0] = 0;
    for (int s = 1; s < ndev; ++s) {
        const double target = pre[size_t(m)] * s / ndev;
        int64_t j = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
        j = std::max<int64_t>(j, b[size_t(s) - 1] + (m - b[size_t(s) - 1] > ndev - s ? 1 : 0));
        b[size_t(s)] = std::min<int64_t>(j, m);
    }
    return b;
}

ncclDataType_t nccl_real(int dtype) { return dtype == TM_C64 ? ncclFloat : ncclDouble; }

// y[seg] += src[seg] on one device (the emulated reduce)
void add_into(const tm_sharded* S, void* y, const void* src, int64_t n, cudaStream_t st) {
    if (n == 0) return;
    const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 8192));
    if (S->dtype == TM_C64)
        add_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<float2*>(y), static_cast<const float2*>(src), n);
    else
        add_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<double2*>(y), static_cast<const double2*>(src), n);
    launched(cudaSuccess, "add_kernel");
}

// One unit of reduction: rows [r0, r0 + nrow) of right-hand sides [ca, cb)
// of the partial outputs, complete on shard d once ev[d] has fired.
struct RedUnit {
    int64_t r0, nrow, ca, cb;
    std::vector<cudaEvent_t> ev;
};

// Reduce the shards' partial outputs (out_d, leading dimension ld_d; shard 0
// = the root accumulates in place in out_0) unit by unit on the
// communication streams.
void reduce_units(tm_sharded* S, std::vector<RedUnit>& units, const std::vector<void*>& out,
                  const std::vector<int64_t>& ld) {
    const size_t nd = S->ndev();
    const size_t cs = S->csize();
    for (RedUnit& u : units) {
        if (S->comm->emulated || nd == 1) {
            DeviceGuard g(S->dev(0));
            for (size_t d = 0; d < nd; ++d) CK(cudaStreamWaitEvent(S->mst[0], u.ev[d], 0));
            for (size_t d = 1; d < nd; ++d)
                for (int64_t c = u.ca; c < u.cb; ++c)
                    add_into(S, static_cast<char*>(out[0]) + (c * ld[0] + u.r0) * cs,
                             static_cast<const char*>(out[d]) + (c * ld[d] + u.r0) * cs, u.nrow, S->mst[0]);
            continue;
        }
        for (size_t d = 0; d < nd; ++d) {
            DeviceGuard g(S->dev(d));
            CK(cudaStreamWaitEvent(S->mst[d], u.ev[d], 0));
        }
        NCK(nccl().GroupStart());
        for (size_t d = 0; d < nd; ++d)
            for (int64_t c = u.ca; c < u.cb; ++c) {
                char* p = static_cast<char*>(out[d]) + (c * ld[d] + u.r0) * cs;
                NCK(nccl().Reduce(p, d == 0 ? p : nullptr, size_t(u.nrow) * 2, nccl_real(S->dtype), ncclSum, 0,
                               S->comm->comms[d], S->mst[d]));
            }
        NCK(nccl().GroupEnd());
    }
}

// Forward-shaped sharded product: every shard computes a full-height partial
// output (rows_out x p) from its columns; the partials are summed into the
// root.  `in_rows_all`: true when every shard reads the whole input (ACA:
// x is m2 x p), false when shard d reads input rows [c0_d, c1_d).
template <typename Body>
void sharded_sum(tm_sharded* S, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y, int64_t ldy,
                 int64_t rows_out, bool host, cudaStream_t caller, bool in_rows_all, Body body) {
    const size_t nd = S->shards.size(), cs = S->csize();
    cudaEvent_t in_ready = nullptr;
    if (!host) {
        DeviceGuard g(S->dev(0));
        CK(cudaEventCreateWithFlags(&in_ready, cudaEventDisableTiming));
        CK(cudaEventRecord(in_ready, caller));
    }
    std::vector<void*> out(nd);
    std::vector<int64_t> ld(nd, rows_out);
    std::vector<std::vector<std::tuple<int64_t, int64_t, int64_t, int64_t, cudaEvent_t>>> blocks(nd);
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        tm_store* st = S->shards[d];
        const int64_t a = in_rows_all ? 0 : S->c0[d], n = in_rows_all ? xrows : S->c1[d] - S->c0[d];
        CK(cudaStreamWaitEvent(S->cst[d], S->done[d], 0));
        order_after_prev(st, S->cst[d]);
        if (!host) CK(cudaStreamWaitEvent(S->cst[d], in_ready, 0));
        void* xd = S->xbuf[d].get(size_t(std::max<int64_t>(n * p, 1)) * cs);
        if (n * p > 0)
            CK(cudaMemcpy2DAsync(xd, size_t(n) * cs, static_cast<const char*>(x) + size_t(a) * cs, size_t(ldx) * cs,
                                 size_t(n) * cs, size_t(p), host ? cudaMemcpyHostToDevice : cudaMemcpyDefault,
                                 S->cst[d]));
        out[d] = (d == 0 && !host) ? y : S->ybuf[d].get(size_t(std::max<int64_t>(rows_out * p, 1)) * cs);
        if (d == 0 && !host) ld[0] = ldy;
        HostPipe hp;
        hp.block_done = [&, d](int64_t k0, int64_t k1, int64_t ca, int64_t pb, cudaStream_t s2) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, s2));
            blocks[d].emplace_back(k0, k1, ca, ca + pb, ev);
        };
        body(st, xd, n, p, out[d], ld[d], S->cst[d], &hp);
        if (blocks[d].empty()) {  // no block reports (an empty shard): one event for everything
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, S->cst[d]));
            blocks[d].emplace_back(0, S->q, 0, p, ev);
        }
        mark_done(st, S->cst[d]);
    }
    // reduction units: per (component, pass) block when every shard reports
    // the same blocks (the tensor-core forward's waves), else one unit
    const int64_t nvr = rows_out / std::max<int64_t>(1, (rows_out == S->rows() ? S->q : 1));
    bool same = true;
    for (size_t d = 1; d < nd; ++d) {
        if (blocks[d].size() != blocks[0].size()) same = false;
        for (size_t b = 0; same && b < blocks[d].size(); ++b)
            same = std::get<0>(blocks[d][b]) == std::get<0>(blocks[0][b]) &&
                   std::get<1>(blocks[d][b]) == std::get<1>(blocks[0][b]) &&
                   std::get<2>(blocks[d][b]) == std::get<2>(blocks[0][b]) &&
                   std::get<3>(blocks[d][b]) == std::get<3>(blocks[0][b]);
    }
    std::vector<RedUnit> units;
    if (same && rows_out == S->rows()) {
        for (size_t b = 0; b < blocks[0].size(); ++b) {
            RedUnit u{std::get<0>(blocks[0][b]) * nvr, (std::get<1>(blocks[0][b]) - std::get<0>(blocks[0][b])) * nvr,
                      std::get<2>(blocks[0][b]), std::get<3>(blocks[0][b]), {}};
            for (size_t d = 0; d < nd; ++d) u.ev.push_back(std::get<4>(blocks[d][b]));
            units.push_back(std::move(u));
        }
    } else {
        RedUnit u{0, rows_out, 0, p, {}};
        for (size_t d = 0; d < nd; ++d) {
            DeviceGuard g(S->dev(d));
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, S->cst[d]));
            blocks[d].emplace_back(0, 0, 0, 0, ev);
            u.ev.push_back(ev);
        }
        units.push_back(std::move(u));
    }
    reduce_units(S, units, out, ld);
    {
        DeviceGuard g(S->dev(0));
        if (host && rows_out * p > 0)
            CK(cudaMemcpy2DAsync(y, size_t(ldy) * cs, out[0], size_t(rows_out) * cs, size_t(rows_out) * cs, size_t(p),
                                 cudaMemcpyDeviceToHost, S->mst[0]));
    }
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        CK(cudaEventRecord(S->done[d], S->comm->emulated || nd == 1 ? S->mst[0] : S->mst[d]));
        for (auto& b : blocks[d]) CK(cudaEventDestroy(std::get<4>(b)));
    }
    DeviceGuard g(S->dev(0));
    if (in_ready) CK(cudaEventDestroy(in_ready));
    if (host) {
        for (size_t d = 0; d < nd; ++d) CK(cudaEventSynchronize(S->done[d]));
    } else {
        for (size_t d = 0; d < nd; ++d) CK(cudaStreamWaitEvent(caller, S->done[d], 0));
    }
}

// Adjoint: every shard reads the whole of Phi and writes the z rows of its
// columns; host z receives each shard's rows directly, device z on the root
// gathers them (ncclSend / ncclRecv, or device copies when emulated).
void sharded_adjoint(tm_sharded* S, const void* phi, int64_t ldphi, int64_t p, void* z, int64_t ldz, bool host,
                     cudaStream_t caller) {
    const size_t nd = S->shards.size(), cs = S->csize();
    const int64_t rows = S->rows();
    cudaEvent_t in_ready = nullptr;
    if (!host) {
        DeviceGuard g(S->dev(0));
        CK(cudaEventCreateWithFlags(&in_ready, cudaEventDisableTiming));
        CK(cudaEventRecord(in_ready, caller));
    }
    // Phi on every device: host -> each device; device -> root copy (if strided) + broadcast
    std::vector<const void*> ph(nd, nullptr);
    std::vector<int64_t> ldp(nd, rows);
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        CK(cudaStreamWaitEvent(S->cst[d], S->done[d], 0));
        order_after_prev(S->shards[d], S->cst[d]);
        if (!host) CK(cudaStreamWaitEvent(S->cst[d], in_ready, 0));
    }
    if (host) {
        for (size_t d = 0; d < nd; ++d) {
            DeviceGuard g(S->dev(d));
            void* b = S->xbuf[d].get(size_t(std::max<int64_t>(rows * p, 1)) * cs);
            CK(cudaMemcpy2DAsync(b, size_t(rows) * cs, phi, size_t(ldphi) * cs, size_t(rows) * cs, size_t(p),
                                 cudaMemcpyHostToDevice, S->cst[d]));
            ph[d] = b;
        }
    } else if (S->comm->emulated || nd == 1) {
        for (size_t d = 0; d < nd; ++d) {
            ph[d] = phi;  // every shard lives on the root's device
            ldp[d] = ldphi;
        }
    } else {
        DeviceGuard g0(S->dev(0));
        const void* src = phi;
        if (ldphi != rows && p > 1) {  // NCCL moves contiguous blocks
            void* b = S->xbuf[0].get(size_t(rows * p) * cs);
            CK(cudaMemcpy2DAsync(b, size_t(rows) * cs, phi, size_t(ldphi) * cs, size_t(rows) * cs, size_t(p),
                                 cudaMemcpyDeviceToDevice, S->cst[0]));
            src = b;
        } else {
            ldp[0] = ldphi;
        }
        ph[0] = src;
        for (size_t d = 1; d < nd; ++d) {
            DeviceGuard g(S->dev(d));
            ph[d] = S->xbuf[d].get(size_t(std::max<int64_t>(rows * p, 1)) * cs);
        }
        NCK(nccl().GroupStart());
        for (size_t d = 0; d < nd; ++d)
            NCK(nccl().Broadcast(d == 0 ? src : ph[d], const_cast<void*>(ph[d]), size_t(rows * p) * 2,
                              nccl_real(S->dtype), 0, S->comm->comms[d], S->cst[d]));
        NCK(nccl().GroupEnd());
    }
    // per-shard adjoints into contiguous z blocks
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        const int64_t n = S->c1[d] - S->c0[d];
        void* zd = S->zbuf[d].get(size_t(std::max<int64_t>(n * p, 1)) * cs);
        if (n > 0) adjoint_dev(S->shards[d], ph[d], ldp[d], p, zd, n, S->cst[d]);
        mark_done(S->shards[d], S->cst[d]);
        if (host && n > 0)
            CK(cudaMemcpy2DAsync(static_cast<char*>(z) + size_t(S->c0[d]) * cs, size_t(ldz) * cs, zd, size_t(n) * cs,
                                 size_t(n) * cs, size_t(p), cudaMemcpyDeviceToHost, S->cst[d]));
    }
    if (!host) {
        // gather the rows on the root
        std::vector<cudaEvent_t> ev(nd);
        for (size_t d = 0; d < nd; ++d) {
            DeviceGuard g(S->dev(d));
            CK(cudaEventCreateWithFlags(&ev[d], cudaEventDisableTiming));
            CK(cudaEventRecord(ev[d], S->cst[d]));
        }
        DeviceGuard g0(S->dev(0));
        for (size_t d = 0; d < nd; ++d) CK(cudaStreamWaitEvent(S->mst[0], ev[d], 0));
        std::vector<void*> src(nd);
        if (S->comm->emulated || nd == 1) {
            for (size_t d = 0; d < nd; ++d) src[d] = S->zbuf[d].p;
        } else {
            int64_t tot = 0;
            for (size_t d = 1; d < nd; ++d) tot += (S->c1[d] - S->c0[d]) * p;
            char* gbuf = static_cast<char*>(S->zgather.get(size_t(std::max<int64_t>(tot, 1)) * cs));
            for (size_t d = 1; d < nd; ++d) {
                DeviceGuard g(S->dev(d));
                CK(cudaStreamWaitEvent(S->mst[d], ev[d], 0));
            }
            NCK(nccl().GroupStart());
            int64_t off = 0;
            src[0] = S->zbuf[0].p;
            for (size_t d = 1; d < nd; ++d) {
                const size_t cnt = size_t((S->c1[d] - S->c0[d]) * p) * 2;
                NCK(nccl().Recv(gbuf + off * cs, cnt, nccl_real(S->dtype), int(d), S->comm->comms[0], S->mst[0]));
                NCK(nccl().Send(S->zbuf[d].p, cnt, nccl_real(S->dtype), 0, S->comm->comms[d], S->mst[d]));
                src[d] = gbuf + off * cs;
                off += (S->c1[d] - S->c0[d]) * p;
            }
            NCK(nccl().GroupEnd());
        }
        for (size_t d = 0; d < nd; ++d) {
            const int64_t n = S->c1[d] - S->c0[d];
            if (n > 0)
                CK(cudaMemcpy2DAsync(static_cast<char*>(z) + size_t(S->c0[d]) * cs, size_t(ldz) * cs, src[d],
                                     size_t(n) * cs, size_t(n) * cs, size_t(p), cudaMemcpyDeviceToDevice, S->mst[0]));
        }
        for (cudaEvent_t e : ev) CK(cudaEventDestroy(e));
    }
    for (size_t d = 0; d < nd; ++d) {
        // the next product may rewrite this shard's z block once the gather has read it
        DeviceGuard g(S->dev(d));
        cudaStream_t last = host ? S->cst[d] : ((S->comm->emulated || nd == 1 || d == 0) ? S->mst[0] : S->mst[d]);
        CK(cudaEventRecord(S->done[d], last));
    }
    DeviceGuard g(S->dev(0));
    if (in_ready) CK(cudaEventDestroy(in_ready));
    if (host) {
        for (size_t d = 0; d < nd; ++d) CK(cudaEventSynchronize(S->done[d]));
    } else {
        CK(cudaStreamWaitEvent(caller, S->done[0], 0));
    }
}

// ------------------------------------------------------------ row sharding --

// Cut points (global slab index k n1 + i1) of the row partition: `nd`
// contiguous ranges of near-equal cost (a slab of component k costs
// cc[k] / n1); cuts inside a component on multiples of `align` rows leaving
// >= min_rows rows on both sides, else at the nearer component boundary.
// Bit-for-bit the same rule as sharded.py:row_pieces (tests compare them).
std::vector<int64_t> row_cuts(const std::vector<double>& cc, int64_t n1, int nd, int64_t align, int64_t min_rows) {
    const int q = int(cc.size());
    const int64_t step = std::max<int64_t>(align, 1), lo = std::max<int64_t>(min_rows, step);
    std::vector<double> pre(size_t(q) + 1, 0.0);
    for (int k = 0; k < q; ++k) pre[size_t(k) + 1] = pre[size_t(k)] + cc[size_t(k)];
    std::vector<int64_t> cuts{0};
    for (int s = 1; s < nd; ++s) {
        const double target = pre[size_t(q)] * s / nd;
        int k = int(std::upper_bound(pre.begin(), pre.end(), target) - pre.begin()) - 1;
        k = std::min(std::max(k, 0), q - 1);
        const double frac = cc[size_t(k)] > 0 ? (target - pre[size_t(k)]) / cc[size_t(k)] : 0.0;
        int64_t loc = int64_t(std::nearbyint(frac * double(n1) / double(step))) * step;  // round half to even
        if (loc < lo || n1 - loc < lo) loc = frac < 0.5 ? 0 : n1;
        cuts.push_back(std::max(cuts.back(), std::min<int64_t>(int64_t(k) * n1 + loc, int64_t(q) * n1)));
    }
    cuts.push_back(int64_t(q) * n1);
    return cuts;
}

// Per-component madds of one product (reconstruct_madds, src/matvec.cpp:10-15,
// plus the accumulate term at p = 1), exact in int64.
std::vector<double> component_costs(const tm_store_desc& d) {
    const int64_t n1 = d.dims[0], n2 = d.dims[1], n3 = d.dims[2];
    std::vector<double> cc(size_t(d.q), 0.0);
    for (int k = 0; k < d.q; ++k) {
        int64_t c = 0;
        for (int64_t j = 0; j < d.ncols; ++j) {
            const int32_t* r = d.ranks + 3 * (j * d.q + k);
            c += n1 * r[0] * r[1] * r[2] + n1 * n2 * r[1] * r[2] + n1 * n2 * n3 * r[2] + n1 * n2 * n3;
        }
        cc[size_t(k)] = double(c);
    }
    return cc;
}

// The piece (component k, i1 rows [a, b)) of a host store as a one-component
// store on the sub-grid (b - a) x n2 x n3: every column's tensor (j, k) with
// U1 restricted to rows [a, b) (col-major n1 x r1 -> (b - a) x r1).
tm_store* create_piece_store(const tm_store_desc& d, const std::vector<int64_t>& toff, int k, int64_t a, int64_t b,
                             int device, int dtype) {
    const int64_t n1 = d.dims[0], n2 = d.dims[1], n3 = d.dims[2], m = d.ncols, h = b - a;
    std::vector<int32_t> rk(size_t(3 * std::max<int64_t>(m, 1)));
    int64_t total = 0;
    for (int64_t j = 0; j < m; ++j) {
        const int32_t* r = d.ranks + 3 * (j * d.q + k);
        if (r[0] > h)
            contract("row sharding: a piece of " + std::to_string(h) + " i1 rows is below tucker rank r1 = " +
                     std::to_string(r[0]));
        for (int g = 0; g < 3; ++g) rk[size_t(3 * j + g)] = r[g];
        total += int64_t(r[0]) * r[1] * r[2] + h * r[0] + n2 * r[1] + n3 * r[2];
    }
    std::vector<double> pay(size_t(2 * std::max<int64_t>(total, 1)));
    double* o = pay.data();
    for (int64_t j = 0; j < m; ++j) {
        const int32_t* r = d.ranks + 3 * (j * d.q + k);
        const double* src = d.payload + 2 * toff[size_t(j * d.q + k)];
        const int64_t core = int64_t(r[0]) * r[1] * r[2];
        std::memcpy(o, src, size_t(2 * core) * sizeof(double));
        o += 2 * core;
        for (int c = 0; c < r[0]; ++c) {
            std::memcpy(o, src + 2 * (core + c * n1 + a), size_t(2 * h) * sizeof(double));
            o += 2 * h;
        }
        const int64_t rest = n2 * r[1] + n3 * r[2];
        std::memcpy(o, src + 2 * (core + n1 * r[0]), size_t(2 * rest) * sizeof(double));
        o += 2 * rest;
    }
    tm_store_desc sd = d;
    sd.q = 1;
    sd.dims[0] = h;
    sd.ranks = rk.data();
    sd.payload = pay.data();
    return create_store(sd, device, dtype);
}

void build_row_pieces(tm_sharded* S, const tm_store_desc& d, int dtype) {
    const int nd = int(S->ndev());
    const int64_t n1 = d.dims[0];
    int32_t r1max = 1;
    for (int64_t i = 0; i < d.ncols * d.q; ++i) r1max = std::max(r1max, d.ranks[3 * i]);
    const int64_t align = 2 * 4;  // the CTA-pair tile height of the tensor-core kernels (i1 rows)
    const std::vector<int64_t> cuts =
        row_cuts(component_costs(d), n1, nd, align, (int64_t(r1max) + align - 1) / align * align);
    std::vector<int64_t> toff(size_t(d.ncols * d.q) + 1, 0);
    for (int64_t i = 0; i < d.ncols * d.q; ++i) {
        const int32_t* r = d.ranks + 3 * i;
        toff[size_t(i) + 1] = toff[size_t(i)] + int64_t(r[0]) * r[1] * r[2] + d.dims[0] * r[0] +
                              d.dims[1] * r[1] + d.dims[2] * r[2];
    }
    S->pieces.reserve(size_t(d.q + nd));
    for (int s = 0; s < nd; ++s) {
        S->c0.push_back(cuts[size_t(s)]);
        S->c1.push_back(cuts[size_t(s) + 1]);
        for (int64_t r0 = cuts[size_t(s)]; r0 < cuts[size_t(s) + 1];) {
            const int k = int(r0 / n1);
            const int64_t e = std::min(cuts[size_t(s) + 1], int64_t(k + 1) * n1);
            S->pieces.emplace_back();
            tm_sharded::Piece& pc = S->pieces.back();
            pc.d = size_t(s);
            pc.k = k;
            pc.a = r0 - int64_t(k) * n1;
            pc.b = e - int64_t(k) * n1;
            pc.st = create_piece_store(d, toff, k, pc.a, pc.b, S->dev(size_t(s)), dtype);
            r0 = e;
        }
    }
}

// rows [a, b) of component k, right-hand side c: out (n1-pitched, full grid)
// <-> piece (h-pitched, sub-grid); n2 n3 rows of h elements.
void slab_copy(const tm_sharded* S, void* dst, size_t dpitch, const void* src, size_t spitch, int64_t h,
               cudaMemcpyKind kind, cudaStream_t st) {
    const size_t cs = S->csize();
    CK(cudaMemcpy2DAsync(dst, dpitch * cs, src, spitch * cs, size_t(h) * cs, size_t(S->dims[1] * S->dims[2]), kind,
                         st));
}

// Forward (aca: aca_forward) over the row pieces: every device reads the
// whole input, each piece computes its rows of y on the sub-grid and copies
// them into y (host, or device memory on the root — peer to peer).
void rows_forward(tm_sharded* S, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y, int64_t ldy,
                  bool host, cudaStream_t caller, bool aca) {
    const size_t nd = S->ndev(), cs = S->csize();
    cudaEvent_t in_ready = nullptr;
    if (!host) {
        DeviceGuard g(S->dev(0));
        CK(cudaEventCreateWithFlags(&in_ready, cudaEventDisableTiming));
        CK(cudaEventRecord(in_ready, caller));
    }
    std::vector<void*> xd(nd, nullptr);
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        CK(cudaStreamWaitEvent(S->cst[d], S->done[d], 0));
        if (!host) CK(cudaStreamWaitEvent(S->cst[d], in_ready, 0));
        xd[d] = S->xbuf[d].get(size_t(std::max<int64_t>(xrows * p, 1)) * cs);
        if (xrows * p > 0)
            CK(cudaMemcpy2DAsync(xd[d], size_t(xrows) * cs, x, size_t(ldx) * cs, size_t(xrows) * cs, size_t(p),
                                 host ? cudaMemcpyHostToDevice : cudaMemcpyDefault, S->cst[d]));
    }
    const int64_t nv = S->nv(), n1 = S->dims[0];
    for (tm_sharded::Piece& pc : S->pieces) {
        const size_t d = pc.d;
        DeviceGuard g(S->dev(d));
        tm_store* st = pc.st;
        const int64_t h = pc.b - pc.a, rp = st->rows();
        void* yt = pc.ybuf.get(size_t(std::max<int64_t>(rp * p, 1)) * cs);
        order_after_prev(st, S->cst[d]);
        if (st->ncols == 0) {
            zero_dev(st, yt, rp, p, rp, S->cst[d]);
        } else if (aca) {
            void* w = st->wbuf.get(size_t(st->ncols * p) * cs);
            aca_vhx_dev(st, xd[d], xrows, p, w, S->cst[d]);
            forward_dev(st, w, st->ncols, p, yt, rp, S->cst[d]);
        } else {
            forward_dev(st, xd[d], xrows, p, yt, rp, S->cst[d]);
        }
        mark_done(st, S->cst[d]);
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, S->cst[d]));
        CK(cudaStreamWaitEvent(S->mst[d], ev, 0));
        CK(cudaEventDestroy(ev));
        for (int64_t c = 0; c < p; ++c)
            slab_copy(S, static_cast<char*>(y) + size_t(c * ldy + pc.k * nv + pc.a) * cs, size_t(n1),
                      static_cast<const char*>(yt) + size_t(c * rp) * cs, size_t(h), h,
                      host ? cudaMemcpyDeviceToHost : cudaMemcpyDefault, S->mst[d]);
    }
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        // done[d]: this device's compute (cst) and copies (mst)
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, S->cst[d]));
        CK(cudaStreamWaitEvent(S->mst[d], ev, 0));
        CK(cudaEventDestroy(ev));
        CK(cudaEventRecord(S->done[d], S->mst[d]));
    }
    DeviceGuard g(S->dev(0));
    if (in_ready) CK(cudaEventDestroy(in_ready));
    if (host) {
        for (size_t d = 0; d < nd; ++d) CK(cudaEventSynchronize(S->done[d]));
    } else {
        for (size_t d = 0; d < nd; ++d) CK(cudaStreamWaitEvent(caller, S->done[d], 0));
    }
}

// Adjoint (aca: aca_adjoint) over the row pieces: each piece reads its rows
// of Phi, the pieces of a device sum their m x p (ACA: r_c x p, then V t,
// m2 x p) partials, and the devices' partials are reduced to the root.
void rows_adjoint(tm_sharded* S, const void* phi, int64_t ldphi, int64_t p, void* z, int64_t ldz, bool host,
                  cudaStream_t caller, bool aca) {
    const size_t nd = S->ndev(), cs = S->csize();
    const int64_t nv = S->nv(), n1 = S->dims[0], tr = S->ncols, outrows = aca ? S->m2 : S->ncols;
    cudaEvent_t in_ready = nullptr;
    if (!host) {
        DeviceGuard g(S->dev(0));
        CK(cudaEventCreateWithFlags(&in_ready, cudaEventDisableTiming));
        CK(cudaEventRecord(in_ready, caller));
    }
    std::vector<void*> out(nd, nullptr);
    std::vector<int64_t> ld(nd, outrows);
    std::vector<bool> first(nd, true);
    std::vector<tm_store*> any(nd, nullptr);
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        CK(cudaStreamWaitEvent(S->cst[d], S->done[d], 0));
        if (!host) CK(cudaStreamWaitEvent(S->cst[d], in_ready, 0));
    }
    for (tm_sharded::Piece& pc : S->pieces) {
        const size_t d = pc.d;
        DeviceGuard g(S->dev(d));
        tm_store* st = pc.st;
        const int64_t h = pc.b - pc.a, rp = st->rows();
        void* pt = pc.pbuf.get(size_t(std::max<int64_t>(rp * p, 1)) * cs);
        for (int64_t c = 0; c < p; ++c)
            slab_copy(S, static_cast<char*>(pt) + size_t(c * rp) * cs, size_t(h),
                      static_cast<const char*>(phi) + size_t(c * ldphi + pc.k * nv + pc.a) * cs, size_t(n1), h,
                      host ? cudaMemcpyHostToDevice : cudaMemcpyDefault, S->cst[d]);
        void* acc = S->zbuf[d].get(size_t(std::max<int64_t>(tr * p, 1)) * cs);
        void* t = first[d] ? acc : pc.tbuf.get(size_t(std::max<int64_t>(tr * p, 1)) * cs);
        order_after_prev(st, S->cst[d]);
        if (tr > 0) adjoint_dev(st, pt, rp, p, t, tr, S->cst[d]);
        mark_done(st, S->cst[d]);
        if (!first[d]) add_into(S, acc, t, tr * p, S->cst[d]);
        first[d] = false;
        any[d] = st;
    }
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        void* acc = S->zbuf[d].get(size_t(std::max<int64_t>(tr * p, 1)) * cs);
        if (first[d] && tr * p > 0) CK(cudaMemsetAsync(acc, 0, size_t(tr * p) * cs, S->cst[d]));  // no pieces here
        if (aca) {
            void* zp = S->ybuf[d].get(size_t(std::max<int64_t>(outrows * p, 1)) * cs);
            if (any[d])
                aca_vt_dev(any[d], acc, p, zp, outrows, S->cst[d]);
            else if (outrows * p > 0)
                CK(cudaMemsetAsync(zp, 0, size_t(outrows * p) * cs, S->cst[d]));
            out[d] = zp;
        } else {
            out[d] = acc;
        }
    }
    RedUnit u{0, outrows, 0, p, {}};
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, S->cst[d]));
        u.ev.push_back(ev);
    }
    std::vector<RedUnit> units{u};
    reduce_units(S, units, out, ld);
    {
        DeviceGuard g(S->dev(0));
        if (outrows * p > 0)
            CK(cudaMemcpy2DAsync(z, size_t(ldz) * cs, out[0], size_t(outrows) * cs, size_t(outrows) * cs, size_t(p),
                                 host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, S->mst[0]));
    }
    for (size_t d = 0; d < nd; ++d) {
        DeviceGuard g(S->dev(d));
        CK(cudaEventRecord(S->done[d], S->comm->emulated || nd == 1 ? S->mst[0] : S->mst[d]));
        CK(cudaEventDestroy(units[0].ev[d]));
    }
    DeviceGuard g(S->dev(0));
    if (in_ready) CK(cudaEventDestroy(in_ready));
    if (host) {
        for (size_t d = 0; d < nd; ++d) CK(cudaEventSynchronize(S->done[d]));
    } else {
        CK(cudaStreamWaitEvent(caller, S->done[0], 0));
    }
}

void add_ops(const tm_sharded* S, int64_t p, int64_t* ops) {
    auto one = [&](const tm_store* st) {
        ops[0] += st->dec_madds;
        ops[1] += st->ncols * st->q * st->nv() * p;
    };
    for (const tm_store* st : S->shards) one(st);
    for (const tm_sharded::Piece& pc : S->pieces) one(pc.st);
}

}  // namespace

extern "C" {

TM_API int tm_comm_init(int ndev, const int* devices, tm_comm** out) {
    return guarded([&] {
        if (!out || ndev < 1 || !devices) contract("tm_comm_init: need ndev >= 1 devices");
        int have = 0;
        CK(cudaGetDeviceCount(&have));
        for (int i = 0; i < ndev; ++i)
            if (devices[i] < 0 || devices[i] >= have)
                throw TmError(TM_CUDA_ERROR, "tm_comm_init: no CUDA device " + std::to_string(devices[i]));
        auto c = std::make_unique<tm_comm>();
        c->devices.assign(devices, devices + ndev);
        c->emulated = std::set<int>(c->devices.begin(), c->devices.end()).size() != size_t(ndev);
        if (!c->emulated) {
            c->comms.assign(size_t(ndev), nullptr);
            NCK(nccl().CommInitAll(c->comms.data(), ndev, devices));
            // peer access for the row-sharded products' direct slab copies (NVLink)
            for (int i = 0; i < ndev; ++i)
                for (int j = 0; j < ndev; ++j) {
                    int can = 0;
                    if (i == j || cudaDeviceCanAccessPeer(&can, devices[i], devices[j]) != cudaSuccess || !can)
                        continue;
                    DeviceGuard g(devices[i]);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
                    else CK(e);
                }
        }
        *out = c.release();
    });
}

TM_API int tm_comm_finalize(tm_comm* c) {
    return guarded([&] { delete c; });
}

TM_API int tm_comm_info(const tm_comm* c, int32_t* ndev, int32_t* emulated) {
    return guarded([&] {
        if (!c) contract("null communicator");
        if (ndev) *ndev = int32_t(c->devices.size());
        if (emulated) *emulated = c->emulated ? 1 : 0;
    });
}

TM_API int tm_sharded_create_mode(const tm_store_desc* desc, tm_comm* comm, int dtype, int mode, tm_sharded** out) {
    return guarded([&] {
        if (!desc || !comm || !out) contract("tm_sharded_create: null argument");
        if (mode != TM_SHARD_COLUMNS && mode != TM_SHARD_ROWS)
            contract("tm_sharded_create: mode must be TM_SHARD_COLUMNS or TM_SHARD_ROWS");
        if (desc->payload_on_device || desc->v_on_device)
            contract("tm_sharded_create: payload and V must be host arrays (each shard uploads its own columns)");
        const tm_store_desc& d = *desc;
        if (d.q < 1 || d.ncols < 0 || d.dims[0] < 1 || d.dims[1] < 1 || d.dims[2] < 1)
            contract("store: non-positive dimensions");
        if (d.ncols > 0 && (!d.ranks || !d.payload)) contract("store: ranks and payload are required");
        for (int64_t i = 0; i < d.ncols * d.q; ++i)
            for (int g = 0; g < 3; ++g)
                if (d.ranks[3 * i + g] < 1 || d.ranks[3 * i + g] > d.dims[g])
                    contract("store: tucker rank " + std::to_string(d.ranks[3 * i + g]) + " out of range for mode " +
                             std::to_string(g + 1));
        const int nd = int(comm->devices.size());
        auto S = std::make_unique<tm_sharded>();
        S->comm = comm;
        S->devices = comm->devices;
        S->mode = mode;
        S->dtype = dtype;
        S->q = d.q;
        S->ncols = d.ncols;
        S->m2 = d.v ? d.m2 : 0;
        for (int g = 0; g < 3; ++g) S->dims[g] = d.dims[g];
        S->cst.assign(size_t(nd), nullptr);
        S->mst.assign(size_t(nd), nullptr);
        S->done.assign(size_t(nd), nullptr);
        S->xbuf.resize(size_t(nd));
        S->ybuf.resize(size_t(nd));
        S->zbuf.resize(size_t(nd));
        for (int s = 0; s < nd; ++s) {
            DeviceGuard g(comm->devices[size_t(s)]);
            CK(cudaStreamCreateWithFlags(&S->cst[size_t(s)], cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&S->mst[size_t(s)], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&S->done[size_t(s)], cudaEventDisableTiming));
        }
        if (mode == TM_SHARD_ROWS) {
            build_row_pieces(S.get(), d, dtype);
            *out = S.release();
            return;
        }
        const std::vector<int64_t> b = balanced_bounds(d, nd);
        // payload offset (complex scalars) of each column
        std::vector<int64_t> col_off(size_t(d.ncols) + 1, 0);
        for (int64_t j = 0; j < d.ncols; ++j) {
            int64_t sz = 0;
            for (int k = 0; k < d.q; ++k) {
                const int32_t* r = d.ranks + 3 * (j * d.q + k);
                sz += int64_t(r[0]) * r[1] * r[2] + d.dims[0] * r[0] + d.dims[1] * r[1] + d.dims[2] * r[2];
            }
            col_off[size_t(j) + 1] = col_off[size_t(j)] + sz;
        }
        S->shards.assign(size_t(nd), nullptr);
        for (int s = 0; s < nd; ++s) {
            S->c0.push_back(b[size_t(s)]);
            S->c1.push_back(b[size_t(s) + 1]);
            tm_store_desc sd = d;
            sd.ncols = b[size_t(s) + 1] - b[size_t(s)];
            sd.ranks = d.ranks + 3 * d.q * b[size_t(s)];
            sd.payload = d.payload + 2 * col_off[size_t(b[size_t(s)])];
            if (d.v) sd.v = d.v + 2 * d.m2 * b[size_t(s)];  // V's columns of this shard (column-major)
            S->shards[size_t(s)] = create_store(sd, comm->devices[size_t(s)], dtype);
        }
        *out = S.release();
    });
}

TM_API int tm_sharded_create(const tm_store_desc* desc, tm_comm* comm, int dtype, tm_sharded** out) {
    return tm_sharded_create_mode(desc, comm, dtype, TM_SHARD_COLUMNS, out);
}

TM_API int tm_shard_row_cuts(int32_t q, int64_t n1, int32_t ndev, int64_t align, int64_t min_rows,
                             const double* comp_costs, int64_t* cuts) {
    return guarded([&] {
        if (q < 1 || n1 < 1 || ndev < 1 || !comp_costs || !cuts) contract("tm_shard_row_cuts: bad argument");
        const std::vector<int64_t> c =
            row_cuts(std::vector<double>(comp_costs, comp_costs + q), n1, ndev, align, min_rows);
        std::copy(c.begin(), c.end(), cuts);
    });
}

TM_API int tm_sharded_pieces(const tm_sharded* s, int32_t* npieces, int64_t* pieces) {
    return guarded([&] {
        if (!s) contract("null sharded store");
        if (npieces) *npieces = int32_t(s->pieces.size());
        if (pieces)
            for (size_t i = 0; i < s->pieces.size(); ++i) {
                pieces[4 * i] = int64_t(s->pieces[i].d);
                pieces[4 * i + 1] = s->pieces[i].k;
                pieces[4 * i + 2] = s->pieces[i].a;
                pieces[4 * i + 3] = s->pieces[i].b;
            }
    });
}

TM_API int tm_sharded_destroy(tm_sharded* s) {
    return guarded([&] { delete s; });
}

TM_API int tm_sharded_info(const tm_sharded* s, int32_t* nshards, int64_t* ranges, int64_t* device_bytes) {
    return guarded([&] {
        if (!s) contract("null sharded store");
        if (nshards) *nshards = int32_t(s->ndev());
        int64_t bytes = 0;
        for (size_t d = 0; d < s->ndev(); ++d) {
            if (ranges) {
                ranges[2 * d] = s->c0[d];
                ranges[2 * d + 1] = s->c1[d];
            }
            if (d < s->shards.size()) bytes += s->shards[d]->device_bytes;
        }
        for (const tm_sharded::Piece& pc : s->pieces) bytes += pc.st->device_bytes;
        if (device_bytes) *device_bytes = bytes;
    });
}

TM_API int tm_sharded_forward(tm_sharded* S, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y,
                              int64_t ldy, int where, void* stream, int64_t* ops) {
    return guarded([&] {
        if (!S) contract("null sharded store");
        if (xrows != S->ncols)
            contract("forward: x has " + std::to_string(xrows) + " rows, expected m = " + std::to_string(S->ncols));
        check_common(S->any_store(), p, ldx, xrows, ldy, S->rows(), where, x, y);
        std::lock_guard<std::mutex> lock(S->mu);
        if (p > 0 && S->mode == TM_SHARD_ROWS)
            rows_forward(S, x, ldx, xrows, p, y, ldy, where == TM_HOST, static_cast<cudaStream_t>(stream), false);
        else if (p > 0)
            sharded_sum(S, x, ldx, xrows, p, y, ldy, S->rows(), where == TM_HOST, static_cast<cudaStream_t>(stream),
                        false, [](tm_store* st, const void* xd, int64_t n, int64_t pp, void* yd, int64_t ld,
                                  cudaStream_t cs, const HostPipe* hp) {
                            if (n > 0)
                                forward_dev(st, xd, n, pp, yd, ld, cs, hp);
                            else
                                zero_dev(st, yd, st->rows(), pp, ld, cs);
                        });
        if (ops) add_ops(S, p, ops);
    });
}

TM_API int tm_sharded_adjoint(tm_sharded* S, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z,
                              int64_t ldz, int where, void* stream, int64_t* ops) {
    return guarded([&] {
        if (!S) contract("null sharded store");
        if (phirows != S->rows())
            contract("adjoint: phi has " + std::to_string(phirows) + " rows, expected q*n_v = " +
                     std::to_string(S->rows()));
        check_common(S->any_store(), p, ldphi, phirows, ldz, S->ncols, where, phi, z);
        std::lock_guard<std::mutex> lock(S->mu);
        if (p > 0 && S->ncols > 0 && S->mode == TM_SHARD_ROWS)
            rows_adjoint(S, phi, ldphi, p, z, ldz, where == TM_HOST, static_cast<cudaStream_t>(stream), false);
        else if (p > 0 && S->ncols > 0)
            sharded_adjoint(S, phi, ldphi, p, z, ldz, where == TM_HOST, static_cast<cudaStream_t>(stream));
        if (ops) add_ops(S, p, ops);
    });
}

TM_API int tm_sharded_aca_forward(tm_sharded* S, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y,
                                  int64_t ldy, int where, void* stream) {
    return guarded([&] {
        if (!S) contract("null sharded store");
        if (!S->m2) contract("aca_forward: store carries no ACA V factor");
        if (xrows != S->m2)
            contract("aca_forward: x has " + std::to_string(xrows) + " rows, expected " + std::to_string(S->m2));
        check_common(S->any_store(), p, ldx, xrows, ldy, S->rows(), where, x, y);
        std::lock_guard<std::mutex> lock(S->mu);
        if (p > 0 && S->mode == TM_SHARD_ROWS)
            rows_forward(S, x, ldx, xrows, p, y, ldy, where == TM_HOST, static_cast<cudaStream_t>(stream), true);
        else if (p > 0)
            sharded_sum(S, x, ldx, xrows, p, y, ldy, S->rows(), where == TM_HOST, static_cast<cudaStream_t>(stream),
                        true, [](tm_store* st, const void* xd, int64_t n, int64_t pp, void* yd, int64_t ld,
                                 cudaStream_t cs, const HostPipe* hp) {
                            if (st->ncols == 0) {
                                zero_dev(st, yd, st->rows(), pp, ld, cs);
                                return;
                            }
                            void* w = st->wbuf.get(size_t(st->ncols * pp) * st->csize());
                            aca_vhx_dev(st, xd, n, pp, w, cs);
                            forward_dev(st, w, st->ncols, pp, yd, ld, cs, hp);
                        });
    });
}

TM_API int tm_sharded_aca_adjoint(tm_sharded* S, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z,
                                  int64_t ldz, int where, void* stream) {
    return guarded([&] {
        if (!S) contract("null sharded store");
        if (!S->m2) contract("aca_adjoint: store carries no ACA V factor");
        if (phirows != S->rows())
            contract("aca_adjoint: phi has " + std::to_string(phirows) + " rows, expected " +
                     std::to_string(S->rows()));
        check_common(S->any_store(), p, ldphi, phirows, ldz, S->m2, where, phi, z);
        std::lock_guard<std::mutex> lock(S->mu);
        if (p > 0 && S->mode == TM_SHARD_ROWS)
            rows_adjoint(S, phi, ldphi, p, z, ldz, where == TM_HOST, static_cast<cudaStream_t>(stream), true);
        else if (p > 0)
            sharded_sum(S, phi, ldphi, phirows, p, z, ldz, S->m2, where == TM_HOST,
                        static_cast<cudaStream_t>(stream), true,
                        [](tm_store* st, const void* pd, int64_t n, int64_t pp, void* zd, int64_t ld, cudaStream_t cs,
                           const HostPipe*) {
                            if (st->ncols == 0) {
                                zero_dev(st, zd, st->m2, pp, ld, cs);
                                return;
                            }
                            void* t = st->wbuf.get(size_t(st->ncols * pp) * st->csize());
                            adjoint_dev(st, pd, n, pp, t, st->ncols, cs);
                            aca_vt_dev(st, t, pp, zd, ld, cs);
                        });
    });
}

}  // extern "C"
