/*
 * tuckmat_b200 — C ABI of the B200-native Tucker-compressed coupling matvec.
 *
 * Drop-in boundary for the reference library's hot path
 * (/root/reference/proj/include/tuckmat/matvec.hpp).  The reference exposes
 * a header-only C++ API with no FFI; each entry point below replaces one
 * reference function, cited as file:line (paths relative to
 * /root/reference/proj).  The C++ drop-in that re-declares the reference
 * signatures on top of this ABI is include/tuckmat_b200/tuckmat.hpp.
 *
 * Conventions
 *   - Complex scalars are interleaved (re, im) pairs: float for TM_C64
 *     stores, double for TM_C128 stores.  Host-side store payloads are
 *     always complex128 (the reference's only scalar type,
 *     include/tuckmat/tensor.hpp:14); a TM_C64 store rounds them once.
 *   - Multivectors are column-major with a leading dimension (elements),
 *     like Eigen::MatrixXcd (include/tuckmat/matvec.hpp:13).
 *   - Rows of the coupling matrix are component-major, voxel index
 *     f1-fastest (src/compress.cpp:52-65).
 *   - Every call returns a tm_status; on failure tm_last_error() returns a
 *     thread-local message.  Status codes map one-to-one onto the reference
 *     exception types (include/tuckmat/errors.hpp:10-48).
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with TM_CUDA_ERROR.
 *   - A store is immutable after creation.  Products on one store share
 *     device work buffers: they are serialised on the host by an internal
 *     mutex and on the device by a per-store completion event (every
 *     product's stream waits for the previous product's event, whatever
 *     stream or TM_HOST / TM_DEVICE mode it used).  Products on different
 *     stores may run concurrently.
 */
#ifndef TUCKMAT_B200_H
#define TUCKMAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TM_API __attribute__((visibility("default")))
#else
#define TM_API
#endif

typedef enum {
    TM_OK = 0,
    TM_CONTRACT_VIOLATION = 1, /* tuckmat::ContractViolation  (errors.hpp:16-19) */
    TM_CAPACITY_ERROR = 2,     /* tuckmat::CapacityError      (errors.hpp:27-30) */
    TM_PARSE_ERROR = 3,        /* tuckmat::ParseError         (errors.hpp:39-45) */
    TM_SINGULARITY_ERROR = 4,  /* tuckmat::SingularityError   (errors.hpp:21-24) */
    TM_CUDA_ERROR = 6,         /* device / driver failure (no reference analogue) */
    TM_ERROR = 9               /* tuckmat::Error              (errors.hpp:10-13) */
} tm_status;

typedef enum { TM_C64 = 0, TM_C128 = 1 } tm_dtype;

typedef enum { TM_HOST = 0, TM_DEVICE = 1 } tm_where;

typedef struct tm_store tm_store;

/*
 * Store description.  Mirrors CompressedCoupling (include/tuckmat/compress.hpp:14-25)
 * — `ncols` = m, tensors columns[j][k] — or, for an ACA store, the Tucker U
 * of AcaFactors (include/tuckmat/aca.hpp:24-41) — `ncols` = r_c, tensors
 * tucker_u[k][l] listed l-major — plus V.
 *
 * ranks:   ncols*q*3 int32, [col][comp][mode].
 * payload: per tensor, in [col][comp] order, the CTC1 payload layout
 *          (src/io.cpp:121-129): core r1*r2*r3 f1-fastest, then U1 (n1 x r1),
 *          U2, U3 column-major; complex128 pairs.
 * v:       ACA only (else NULL): V, m2 x r_c column-major complex128.
 */
typedef struct {
    int32_t q;
    int64_t ncols;
    int64_t dims[3];
    const int32_t* ranks;
    const double* payload;
    int32_t payload_on_device; /* payload is a device pointer on `device` */
    const double* v;
    int64_t m2;
    int32_t v_on_device;
} tm_store_desc;

/* Build the device-resident store (replaces holding CompressedCoupling /
 * AcaFactors in host memory; K6 "pack_store").  device = CUDA ordinal. */
TM_API int tm_store_create(const tm_store_desc* desc, int device, int dtype, tm_store** out);

/* Native ingest of a CTC1 / CTA1 file straight into device memory
 * (replaces load_ctc1 / load_cta1, src/io.cpp:212-230, 249-279). */
TM_API int tm_store_load_ctc1(const char* path, int device, int dtype, tm_store** out);
TM_API int tm_store_load_cta1(const char* path, int device, int dtype, tm_store** out);

/* Dense-U ACA store: AcaFactors with `dense_u` set and `tucker_u` empty
 * (include/tuckmat/aca.hpp:24-41; the `fac.dense_u * w` branches of
 * aca_forward / aca_adjoint, src/matvec.cpp:158,173).  u: m1 x r, v: m2 x r,
 * column-major complex128, host pointers (device pointers on `device` with
 * on_device = 1).  Only tm_aca_forward / tm_aca_adjoint apply to it. */
TM_API int tm_store_create_dense_aca(const double* u, int64_t m1, const double* v, int64_t m2, int64_t r,
                                     int on_device, int device, int dtype, tm_store** out);

TM_API int tm_store_destroy(tm_store* s);

/* q, ncols (m or r_c), dims, dtype, m2 (0 unless ACA), device bytes held. */
TM_API int tm_store_info(const tm_store* s, int32_t* q, int64_t* ncols, int64_t* dims3, int32_t* dtype,
                         int64_t* m2, int64_t* device_bytes);

/* Which kernels the store's products run: 1 = tcgen05 tensor-core kernels
 * (c64 stores with every rank <= 32 whose factor slots fit the shared-memory
 * plan), 0 = CUDA-core kernels (c128, larger ranks, TMB_DISABLE_TC=1);
 * forward 2 = tcgen05 with its A operand (W = U1 x_1 G x_2 U2 as fp16
 * splits) streamed from the store's precomputed W arena, no producer warps;
 * adjoint 3 = the adjoint as one tcgen05 GEMM on the transposed arena,
 * G = conj(W)^T Phi, then z = sum conj(U3) G.  The arenas are built when the
 * whole store's fit $TMB_WARENA_GB (default 24) and half the free memory;
 * TMB_WARENA=0 (both) / TMB_ADJ_GEMM=0 (the GEMM adjoint) switch them off. */
TM_API int tm_store_kernels(const tm_store* s, int32_t* forward_tc, int32_t* adjoint_tc);

/*
 * Y = Zbc X  — forward(cc, x, workers, ops) (src/matvec.cpp:132-138) and
 * stacked_forward (src/matvec.cpp:17-65).  x: xrows x p (xrows must equal
 * ncols), y: q*n_v x p.  where = TM_HOST: x, y are host pointers, the call
 * copies in, computes and copies out before returning.  where = TM_DEVICE:
 * x, y are device pointers on the store's device and the work is enqueued
 * on `stream` (a cudaStream_t, NULL = legacy default stream).  ops, if not
 * NULL, is {decompress_madds, accumulate_madds} and is incremented (+=) as
 * the reference does (src/matvec.cpp:60-63).
 */
TM_API int tm_forward(tm_store* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y, int64_t ldy,
                      int where, void* stream, int64_t* ops);

/* The forward restricted to components [k0, k1): rows k n_v .. (k+1) n_v - 1 of
 * y for k in the range are written, the other rows untouched; device
 * pointers, enqueued on `stream`.  Lets a one-process-per-GPU driver reduce
 * component k of the partial y while component k + 1 computes
 * (sharded.py). */
TM_API int tm_forward_components(tm_store* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y,
                                 int64_t ldy, int32_t k0, int32_t k1, void* stream);

/* Z = Zbc^H Phi — adjoint(cc, phi, workers, ops) (src/matvec.cpp:140-148)
 * and stacked_adjoint (src/matvec.cpp:67-102).  phi: q*n_v x p, z: ncols x p. */
TM_API int tm_adjoint(tm_store* s, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z,
                      int64_t ldz, int where, void* stream, int64_t* ops);

/* ACA products (src/matvec.cpp:150-175): y = U (V^H x), z = V (U^H phi).
 * x: m2 x p, y: q*n_v x p; phi: q*n_v x p, z: m2 x p.  No OpCounts, as in
 * the reference (include/tuckmat/matvec.hpp:54-57). */
TM_API int tm_aca_forward(tm_store* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y, int64_t ldy,
                          int where, void* stream);
TM_API int tm_aca_adjoint(tm_store* s, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z,
                          int64_t ldz, int where, void* stream);

/* assemble_column (src/scene.cpp:127-150) for a batch of source columns on
 * the device (complex128), the field evaluation of the GPU compressor:
 * origin3 / spacing / dims3 the voxel grid, q = 3 (PWC) or 12 (PWL moments),
 * op = 0 (E-field, src/scene.cpp:84-103) or 1 (H-field, :105-118), k0 the
 * wavenumber; src a device array of m x 7 doubles {midpoint xyz, unit
 * direction xyz, weight}; cols a host array of nb column indices; out a
 * device array of nb x q x n_v complex128 (component-major rows, voxel
 * f1-fastest).  TM_SINGULARITY_ERROR if an evaluation point hits a source. */
TM_API int tm_assemble_columns(const double* origin3, double spacing, const int64_t* dims3, int q, int op, double k0,
                               const double* src, int64_t m, const int64_t* cols, int64_t nb, void* out,
                               void* stream);

/* Rows of the stored operator at the requested global rows (host array,
 * rows[r] = k*n_v + v, v = i1 + n1*(i2 + n2*i3)): out[r + ldout*j] =
 * T_jk[v] for every column j — element() (src/tensor.cpp:183-196) per
 * column, i.e. row_of_compressed_u (src/aca.cpp:234-244) for an ACA store.
 * out is nrows x ncols, host or device per `where`.  An index outside
 * [0, q*n_v) is a contract violation ("element: index out of range"). */
TM_API int tm_rows(tm_store* s, const int64_t* rows, int64_t nrows, void* out, int64_t ldout, int where,
                   void* stream);

/* Exact OpCounts of one product at p right-hand sides, without running it
 * (reconstruct_madds, src/matvec.cpp:10-15; accumulate term :51,95). */
TM_API int tm_opcounts(const tm_store* s, int64_t p, int64_t* decompress_madds, int64_t* accumulate_madds);

/* ------------------------------------------------------------ multi-GPU --
 * Column sharding over the GPUs of one box, driven by
 * one host thread through a single-process NCCL communicator
 * (ncclCommInitAll).  Replaces the reference's worker pool over columns
 * (parallel_for, src/parallel.cpp:13-48; stacked_forward's per-worker
 * partials summed serially, src/matvec.cpp:30-38,58-59): each GPU holds a
 * contiguous, cost-balanced column range (all q components) as a regular
 * store; the forward's partial y is reduced to the root GPU (devices[0]) per
 * component as soon as every GPU has finished that component, overlapping
 * the later components' waves; the adjoint broadcasts Phi and gathers the
 * rows of z (no reduction: rows are independent, src/matvec.cpp:78-96).
 * ACA stores shard U with the matching columns of V.  NCCL is loaded at run
 * time by tm_comm_init (the copy already in the process, $TMB_NCCL_LIB, or
 * libnccl.so.2).  A device list that repeats a device makes an EMULATED
 * communicator (collectives as device-local copies / adds): a functional
 * check of the sharded orchestration on one GPU, not a measurement. */
typedef struct tm_comm tm_comm;
typedef struct tm_sharded tm_sharded;

/* Partition modes of a sharded store.  TM_SHARD_COLUMNS: as above.
 * TM_SHARD_ROWS: row (voxel-slab) sharding, the alternative of SURVEY §8e —
 * the q * n1 (component, i1) slabs of the output are cut into one contiguous
 * cost-balanced range per GPU (cuts inside a component on multiples of 8 i1
 * rows, at least max r1 rows per piece); each (component k, i1 rows [a, b))
 * piece is a one-component store on the sub-grid (b - a) x n2 x n3 with all
 * columns (U1 rows sliced: the same operator restricted to those voxels).
 * The forward has no reduction (each GPU copies its rows of y into the
 * output, peer to peer for a device output); the adjoint reads only its
 * GPU's rows of Phi and reduces the m x p partial z (ACA: m2 x p).  Every
 * GPU holds ~1/N of the store and of Phi. */
typedef enum { TM_SHARD_COLUMNS = 0, TM_SHARD_ROWS = 1 } tm_shard_mode;

TM_API int tm_comm_init(int ndev, const int* devices, tm_comm** out);
TM_API int tm_comm_finalize(tm_comm* comm);
TM_API int tm_comm_info(const tm_comm* comm, int32_t* ndev, int32_t* emulated);

/* desc as for tm_store_create, host payload / V only; shard d lives on
 * devices[d].  ranges (optional, 2 * nshards) receives each shard's [c0, c1). */
TM_API int tm_sharded_create(const tm_store_desc* desc, tm_comm* comm, int dtype, tm_sharded** out);
TM_API int tm_sharded_create_mode(const tm_store_desc* desc, tm_comm* comm, int dtype, int mode, tm_sharded** out);
TM_API int tm_sharded_destroy(tm_sharded* s);
/* ranges: columns mode [c0, c1) per shard; rows mode the shard's slab range
 * [r0, r1) of global slab indices k * n1 + i1. */
TM_API int tm_sharded_info(const tm_sharded* s, int32_t* nshards, int64_t* ranges, int64_t* device_bytes);
/* Rows mode: the pieces (4 int64 each: shard index, k, a, b), in shard order. */
TM_API int tm_sharded_pieces(const tm_sharded* s, int32_t* npieces, int64_t* pieces);
/* The row partition rule on its own (host only, no device needed): ndev + 1
 * cut points over [0, q * n1) from per-component costs. */
TM_API int tm_shard_row_cuts(int32_t q, int64_t n1, int32_t ndev, int64_t align, int64_t min_rows,
                             const double* comp_costs, int64_t* cuts);

/* As tm_forward / tm_adjoint / tm_aca_*; with TM_DEVICE the inputs and
 * outputs live on devices[0] and the work is ordered after / before
 * `stream` (a cudaStream_t of devices[0]). */
TM_API int tm_sharded_forward(tm_sharded* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y,
                              int64_t ldy, int where, void* stream, int64_t* ops);
TM_API int tm_sharded_adjoint(tm_sharded* s, const void* phi, int64_t ldphi, int64_t phirows, int64_t p, void* z,
                              int64_t ldz, int where, void* stream, int64_t* ops);
TM_API int tm_sharded_aca_forward(tm_sharded* s, const void* x, int64_t ldx, int64_t xrows, int64_t p, void* y,
                                  int64_t ldy, int where, void* stream);
TM_API int tm_sharded_aca_adjoint(tm_sharded* s, const void* phi, int64_t ldphi, int64_t phirows, int64_t p,
                                  void* z, int64_t ldz, int where, void* stream);

/* Thread-local message of the last failed call on this thread. */
TM_API const char* tm_last_error(void);

/* Number of CUDA kernels this library has launched in this process
 * (instrumentation for the bench's gpu_launches claim). */
TM_API int64_t tm_launch_count(void);

/* ABI version (bumped on incompatible changes). */
TM_API int tm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TUCKMAT_B200_H */
