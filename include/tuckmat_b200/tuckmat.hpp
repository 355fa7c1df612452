// C++ drop-in for the reference tuckmat matvec API, running on B200.
//
// Re-declares, with the same names, argument order, defaults and exception
// types, the hot-path API of the reference library
//   /root/reference/proj/include/tuckmat/matvec.hpp:13-63   (forward, adjoint,
//       aca_forward, aca_adjoint, stacked_forward, stacked_adjoint, OpCounts,
//       TuckerColumns, reconstruct_madds)
// and the value types it consumes
//   include/tuckmat/tensor.hpp:14-80    (Complex, Index, Dims3, Tensor3, TuckerTensor)
//   include/tuckmat/compress.hpp:14-25  (CompressedCoupling)
//   include/tuckmat/aca.hpp:24-41       (AcaFactors)
//   include/tuckmat/errors.hpp:10-48    (exception taxonomy)
//   include/tuckmat/io.hpp:19-31        (load_ctc1 / load_cta1)
// Eigen is not available, so Matrix / MultiVector are a small column-major
// complex matrix with the members the reference's call sites use.
//
// Every product runs on the GPU through the C ABI of tuckmat_b200.h; there is
// no CPU fallback.  `workers` is accepted for source compatibility (it was
// the reference's host-thread count) and ignored.  The reference's value
// types are immutable after construction (SPEC / README), so the device
// store built for a CompressedCoupling or AcaFactors is cached by object
// identity; call tuckmat::b200::clear_cache() if an object is mutated or its
// address reused for different data.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../tuckmat_b200.h"

// The drop-in's symbols are part of the library's public ABI.
#pragma GCC visibility push(default)

namespace tuckmat {

using Complex = std::complex<double>;
using Index = std::int64_t;
using Dims3 = std::array<Index, 3>;

inline Index volume(const Dims3& d) { return d[0] * d[1] * d[2]; }

// ----------------------------------------------------------------- errors --
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ContractViolation : Error {
    using Error::Error;
};
struct SingularityError : Error {
    using Error::Error;
};
struct CapacityError : Error {
    using Error::Error;
};
struct SceneError : Error {
    SceneError(const std::string& msg, std::size_t source_index) : Error(msg), source(source_index) {}
    std::size_t source;
};
struct ParseError : Error {
    ParseError(const std::string& msg, std::uint64_t offset) : Error(msg), byte_offset(offset) {}
    std::uint64_t byte_offset;
};
struct ConfigError : Error {
    using Error::Error;
};

// ---------------------------------------------------------------- matrices --
// Column-major complex matrix (Eigen::MatrixXcd stand-in).
class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), d_(static_cast<std::size_t>(rows * cols)) {}
    static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    Complex* data() { return d_.data(); }
    const Complex* data() const { return d_.data(); }
    Complex& operator()(Index r, Index c) { return d_[static_cast<std::size_t>(r + rows_ * c)]; }
    const Complex& operator()(Index r, Index c) const { return d_[static_cast<std::size_t>(r + rows_ * c)]; }
    void resize(Index rows, Index cols) {
        rows_ = rows;
        cols_ = cols;
        d_.assign(static_cast<std::size_t>(rows * cols), Complex(0));
    }
    double norm() const;

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<Complex> d_;
};

// Dense block of p right-hand sides / results (matvec.hpp:13).
using MultiVector = Matrix;

// First-index-fastest complex 3D array (tensor.hpp:24-67).
class Tensor3 {
public:
    Tensor3() = default;
    Tensor3(Index n1, Index n2, Index n3);
    explicit Tensor3(const Dims3& d) : Tensor3(d[0], d[1], d[2]) {}
    const Dims3& dims() const { return dims_; }
    Index dim(int mode) const { return dims_[static_cast<std::size_t>(mode - 1)]; }
    Index size() const { return static_cast<Index>(data_.size()); }
    bool empty() const { return data_.empty(); }
    Complex* data() { return data_.data(); }
    const Complex* data() const { return data_.data(); }
    Complex& operator[](Index i) { return data_[static_cast<std::size_t>(i)]; }
    const Complex& operator[](Index i) const { return data_[static_cast<std::size_t>(i)]; }
    Complex& operator()(Index i1, Index i2, Index i3) { return data_[static_cast<std::size_t>(linear(i1, i2, i3))]; }
    const Complex& operator()(Index i1, Index i2, Index i3) const {
        return data_[static_cast<std::size_t>(linear(i1, i2, i3))];
    }
    Index linear(Index i1, Index i2, Index i3) const { return i1 + dims_[0] * (i2 + dims_[1] * i3); }

private:
    Dims3 dims_{0, 0, 0};
    std::vector<Complex> data_;
};

// Tucker representation (tensor.hpp:71-80).
struct TuckerTensor {
    Tensor3 core;
    std::array<Matrix, 3> factors;
    Dims3 dims{0, 0, 0};
    Index rank(int mode) const { return core.dim(mode); }
};

enum class KernelOp : std::uint8_t { EField = 0, HField = 1 };

// compress.hpp:14-25
struct CompressedCoupling {
    Dims3 grid_dims{0, 0, 0};
    int q = 0;
    Index m = 0;
    KernelOp kernel_op = KernelOp::EField;
    double k0 = 0;
    double eps = 0;
    std::vector<std::vector<TuckerTensor>> columns;  // [m][q]
    Index num_voxels() const { return volume(grid_dims); }
    Index rows() const { return q * num_voxels(); }
};

// aca.hpp:24-41
struct AcaFactors {
    Matrix dense_u;                                   // (m1 x r) or empty
    std::vector<std::vector<TuckerTensor>> tucker_u;  // [q][r] or empty
    Dims3 grid_dims{0, 0, 0};
    int q = 0;
    Matrix v;  // (m2 x r)
    double eps = 0;
    double hosvd_eps = 0;
    double final_stat = 0;
    bool converged = false;
    bool compressed() const { return !tucker_u.empty(); }
    Index rank() const { return v.cols(); }
    Index rows() const { return compressed() ? q * volume(grid_dims) : dense_u.rows(); }
    Index cols() const { return v.rows(); }
};

// io.hpp:19-31
struct Cta1File {
    AcaFactors factors;
    double k0 = 0;
    KernelOp kernel_op = KernelOp::EField;
};
CompressedCoupling load_ctc1(const std::string& path);
Cta1File load_cta1(const std::string& path);

// ------------------------------------------------------------------ matvec --
struct OpCounts {
    std::int64_t decompress_madds = 0;
    std::int64_t accumulate_madds = 0;
};

std::int64_t reconstruct_madds(const TuckerTensor& tt);

struct TuckerColumns {
    std::function<const TuckerTensor&(Index col, int comp)> tensor;
    Index ncols = 0;
    int q = 0;
    Dims3 grid_dims{0, 0, 0};
    Index rows() const { return q * volume(grid_dims); }
};

MultiVector stacked_forward(const TuckerColumns& z, const MultiVector& x, int workers = 1, OpCounts* ops = nullptr);
MultiVector stacked_adjoint(const TuckerColumns& z, const MultiVector& x, int workers = 1, OpCounts* ops = nullptr);

MultiVector forward(const CompressedCoupling& cc, const MultiVector& x, int workers = 1, OpCounts* ops = nullptr);
MultiVector adjoint(const CompressedCoupling& cc, const MultiVector& phi, int workers = 1, OpCounts* ops = nullptr);

MultiVector aca_forward(const AcaFactors& fac, const MultiVector& x, int workers = 1);
MultiVector aca_adjoint(const AcaFactors& fac, const MultiVector& phi, int workers = 1);

// tensor.hpp:105 / src/tensor.cpp:183-196 and aca.hpp:57 / src/aca.cpp:234-244,
// evaluated on the device (tm_rows).  row_of_compressed_u returns a 1 x rank
// MultiVector (the reference returns Eigen::RowVectorXcd).
Complex element(const TuckerTensor& tt, Index i1, Index i2, Index i3);
MultiVector row_of_compressed_u(const AcaFactors& fac, Index i);

// ------------------------------------------------------ B200 extensions --
namespace b200 {

// Device precision used for stores the drop-in builds implicitly
// (TM_C128 by default: the reference's own arithmetic).
void set_default_dtype(int dtype);
int default_dtype();
// CUDA ordinal for implicitly built stores (default: $TUCKMAT_DEVICE or 0).
void set_device(int device);
// Drop every cached device store.
void clear_cache();

// Explicit device-resident store (no identity cache).
class DeviceStore {
public:
    DeviceStore(const CompressedCoupling& cc, int dtype = TM_C128, int device = 0);
    DeviceStore(const AcaFactors& fac, int dtype = TM_C128, int device = 0);
    DeviceStore(const TuckerColumns& z, int dtype = TM_C128, int device = 0);
    ~DeviceStore();
    DeviceStore(const DeviceStore&) = delete;
    DeviceStore& operator=(const DeviceStore&) = delete;
    tm_store* handle() const { return h_; }
    int dtype() const { return dtype_; }

private:
    tm_store* h_ = nullptr;
    int dtype_ = TM_C128;
};

MultiVector forward(const DeviceStore& s, const MultiVector& x, OpCounts* ops = nullptr);
MultiVector adjoint(const DeviceStore& s, const MultiVector& phi, OpCounts* ops = nullptr);
MultiVector aca_forward(const DeviceStore& s, const MultiVector& x);
MultiVector aca_adjoint(const DeviceStore& s, const MultiVector& phi);

// Multi-GPU: the store sharded over the GPUs of one box (tm_comm_* /
// tm_sharded_*, tuckmat_b200.h) by columns (TM_SHARD_COLUMNS) or by row
// slabs (TM_SHARD_ROWS); products take and return host blocks.
class Communicator {
public:
    explicit Communicator(const std::vector<int>& devices);
    ~Communicator();
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    tm_comm* handle() const { return h_; }

private:
    tm_comm* h_ = nullptr;
};

class ShardedStore {
public:
    ShardedStore(const CompressedCoupling& cc, Communicator& comm, int dtype = TM_C128,
                 int mode = TM_SHARD_COLUMNS);
    ShardedStore(const AcaFactors& fac, Communicator& comm, int dtype = TM_C128, int mode = TM_SHARD_COLUMNS);
    ~ShardedStore();
    ShardedStore(const ShardedStore&) = delete;
    ShardedStore& operator=(const ShardedStore&) = delete;
    tm_sharded* handle() const { return h_; }
    int dtype() const { return dtype_; }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index m2() const { return m2_; }

private:
    tm_sharded* h_ = nullptr;
    int dtype_ = TM_C128;
    Index rows_ = 0, cols_ = 0, m2_ = 0;
};

MultiVector forward(const ShardedStore& s, const MultiVector& x, OpCounts* ops = nullptr);
MultiVector adjoint(const ShardedStore& s, const MultiVector& phi, OpCounts* ops = nullptr);
MultiVector aca_forward(const ShardedStore& s, const MultiVector& x);
MultiVector aca_adjoint(const ShardedStore& s, const MultiVector& phi);

}  // namespace b200
}  // namespace tuckmat

#pragma GCC visibility pop
