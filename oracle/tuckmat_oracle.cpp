// TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the reference
// tuckmat library's compressed-matvec path.  Nothing in the product
// (paper_2103_06393_b200/) may link or call this file; only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// use it, and only as the checker or the timed CPU baseline.
//
// The reference cannot be compiled here (Eigen 3.4 is a hard find_package
// dependency, proj/CMakeLists.txt:10, and is absent), so this is a
// restatement of its algorithms with hand-written loops in place of Eigen's
// GEMMs.  Each function cites the reference lines it follows
// (paths are relative to /root/reference/proj).
//
// Exposed through a plain C ABI (orc_*) for ctypes.  Complex scalars are
// interleaved (re, im) float64 pairs everywhere.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using Complex = std::complex<double>;
using Index = std::int64_t;

// ---------------------------------------------------------------- errors --
// Status codes mirror include/tuckmat/errors.hpp:10-48 of the reference.
enum Status : int {
    kOk = 0,
    kContractViolation = 1,
    kCapacityError = 2,
    kParseError = 3,
    kSingularityError = 4,
    kSceneError = 5,
    kError = 9,
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct ContractViolation : Error {
    explicit ContractViolation(const std::string& m) : Error(kContractViolation, m) {}
};

thread_local std::string g_last_error;

// ---------------------------------------------------------------- tensor --
// Tensor3: first index fastest, (i1,i2,i3) at i1 + n1*(i2 + n2*i3)
// (include/tuckmat/tensor.hpp:24-67).
struct Tensor3 {
    Index n[3] = {0, 0, 0};
    std::vector<Complex> d;
    Tensor3() = default;
    Tensor3(Index a, Index b, Index c) : n{a, b, c}, d(static_cast<std::size_t>(a * b * c)) {
        if (a <= 0 || b <= 0 || c <= 0)
            throw ContractViolation("Tensor3: dimensions must be positive");
    }
    Index size() const { return n[0] * n[1] * n[2]; }
    Complex* data() { return d.data(); }
    const Complex* data() const { return d.data(); }
};

// Column-major factor (rows x cols), like Eigen::MatrixXcd.
struct Matrix {
    Index rows = 0, cols = 0;
    std::vector<Complex> d;
    Matrix() = default;
    Matrix(Index r, Index c) : rows(r), cols(c), d(static_cast<std::size_t>(r * c)) {}
    Complex& operator()(Index r, Index c) { return d[static_cast<std::size_t>(r + rows * c)]; }
    const Complex& operator()(Index r, Index c) const { return d[static_cast<std::size_t>(r + rows * c)]; }
};

// TuckerTensor: core (r1,r2,r3) + factors[g] (n_g x r_g)
// (include/tuckmat/tensor.hpp:71-80).
struct TuckerTensor {
    Tensor3 core;
    Matrix factors[3];
    Index dims[3] = {0, 0, 0};
};

// mode_product (src/tensor.cpp:89-120): out(i,b,c) = sum_a t(a,b,c) m(i,a)
// for mode 1 and analogously for modes 2 and 3.  Mode 1 is the GEMM
// (r x n1)(n1 x n2n3), mode 2 is n3 slab GEMMs slab*m^T, mode 3 is
// (n1n2 x n3) m^T.
Tensor3 mode_product(const Tensor3& t, const Matrix& m, int mode) {
    if (mode < 1 || mode > 3)
        throw ContractViolation("tensor mode must be 1, 2 or 3, got " + std::to_string(mode));
    if (m.cols != t.n[mode - 1])
        throw ContractViolation("mode_product: matrix has " + std::to_string(m.cols) +
                                " columns but tensor extent along mode " +
                                std::to_string(mode) + " is " + std::to_string(t.n[mode - 1]));
    const Index n1 = t.n[0], n2 = t.n[1], n3 = t.n[2];
    const Index r = m.rows;
    Index od[3] = {n1, n2, n3};
    od[mode - 1] = r;
    Tensor3 out(od[0], od[1], od[2]);
    Complex* o = out.data();
    const Complex* a = t.data();
    const Complex* mm = m.d.data();
    switch (mode) {
    case 1:
        // out (r x n2n3) = m (r x n1) * t (n1 x n2n3)
        for (Index c = 0; c < n2 * n3; ++c) {
            Complex* oc = o + r * c;
            const Complex* tc = a + n1 * c;
            for (Index k = 0; k < n1; ++k) {
                const Complex tk = tc[k];
                const Complex* mk = mm + r * k;
                for (Index i = 0; i < r; ++i) oc[i] += mk[i] * tk;
            }
        }
        break;
    case 2:
        // per i3 slab: out (n1 x r) = t (n1 x n2) * m^T (n2 x r)
        for (Index i3 = 0; i3 < n3; ++i3) {
            const Complex* ts = a + n1 * n2 * i3;
            Complex* os = o + n1 * r * i3;
            for (Index i = 0; i < r; ++i) {
                Complex* oi = os + n1 * i;
                for (Index b = 0; b < n2; ++b) {
                    const Complex mib = mm[i + r * b];
                    const Complex* tb = ts + n1 * b;
                    for (Index i1 = 0; i1 < n1; ++i1) oi[i1] += tb[i1] * mib;
                }
            }
        }
        break;
    default: {
        // out (n1n2 x r) = t (n1n2 x n3) * m^T (n3 x r)
        const Index pl = n1 * n2;
        for (Index i = 0; i < r; ++i) {
            Complex* oi = o + pl * i;
            for (Index c = 0; c < n3; ++c) {
                const Complex mic = mm[i + r * c];
                const Complex* tc = a + pl * c;
                for (Index v = 0; v < pl; ++v) oi[v] += tc[v] * mic;
            }
        }
        break;
    }
    }
    return out;
}

// reconstruct (src/tensor.cpp:176-181): core x1 U1 x2 U2 x3 U3.
Tensor3 reconstruct(const TuckerTensor& tt) {
    Tensor3 out = mode_product(tt.core, tt.factors[0], 1);
    out = mode_product(out, tt.factors[1], 2);
    out = mode_product(out, tt.factors[2], 3);
    return out;
}

// element (src/tensor.cpp:183-196): one entry in O(r1 r2 r3).
Complex element(const TuckerTensor& tt, Index i1, Index i2, Index i3) {
    if (i1 < 0 || i1 >= tt.dims[0] || i2 < 0 || i2 >= tt.dims[1] || i3 < 0 || i3 >= tt.dims[2])
        throw ContractViolation("element: index out of range");
    const Index r1 = tt.core.n[0], r2 = tt.core.n[1], r3 = tt.core.n[2];
    std::vector<Complex> w(static_cast<std::size_t>(r2 * r3));
    for (Index c = 0; c < r2 * r3; ++c) {
        Complex s = 0;
        for (Index a = 0; a < r1; ++a) s += tt.factors[0](i1, a) * tt.core.d[a + r1 * c];
        w[c] = s;
    }
    Complex out = 0;
    for (Index c3 = 0; c3 < r3; ++c3) {
        Complex s = 0;
        for (Index b = 0; b < r2; ++b) s += tt.factors[1](i2, b) * w[b + r2 * c3];
        out += s * tt.factors[2](i3, c3);
    }
    return out;
}

// reconstruct_madds (src/matvec.cpp:10-15).
std::int64_t reconstruct_madds(const TuckerTensor& tt) {
    const Index n1 = tt.dims[0], n2 = tt.dims[1], n3 = tt.dims[2];
    const Index r1 = tt.core.n[0], r2 = tt.core.n[1], r3 = tt.core.n[2];
    return std::int64_t(n1) * r1 * r2 * r3 + std::int64_t(n1) * n2 * r2 * r3 +
           std::int64_t(n1) * n2 * n3 * r3;
}

// -------------------------------------------------------------- parallel --
// parallel_for (src/parallel.cpp:13-48): inline + ordered when workers <= 1,
// else an atomic work queue over std::thread; the first error is rethrown.
template <class Fn>
void parallel_for(std::size_t n, int workers, Fn&& fn) {
    if (n == 0) return;
    if (workers <= 1 || n == 1) {
        for (std::size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    const std::size_t nthreads = std::min<std::size_t>(static_cast<std::size_t>(workers), n);
    std::atomic<std::size_t> next{0};
    std::exception_ptr first_error;
    std::mutex mu;
    auto body = [&]() {
        for (;;) {
            const std::size_t i = next.fetch_add(1);
            if (i >= n) return;
            try {
                fn(i);
            } catch (...) {
                std::lock_guard<std::mutex> lock(mu);
                if (!first_error) first_error = std::current_exception();
                next.store(n);
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    pool.reserve(nthreads);
    for (std::size_t k = 0; k < nthreads; ++k) pool.emplace_back(body);
    for (auto& th : pool) th.join();
    if (first_error) std::rethrow_exception(first_error);
}

// ----------------------------------------------------------------- store --
// A TuckerColumns view (include/tuckmat/matvec.hpp:28-35): ncols columns of
// q tensors each.  Tensor (col j, comp k) lives at index j*q + k, which is
// the CTC1 payload order (src/io.cpp:204-208) and, for an ACA U store, the
// CTA1 order tucker_u[k][l] written l-major (src/io.cpp:240-243).
struct Store {
    int q = 0;
    Index ncols = 0;
    Index dims[3] = {0, 0, 0};
    std::vector<TuckerTensor> t;
    Index nv() const { return dims[0] * dims[1] * dims[2]; }
    Index rows() const { return q * nv(); }
    const TuckerTensor& at(Index j, int k) const { return t[static_cast<std::size_t>(j * q + k)]; }
};

// Dense column-major multivector (Eigen::MatrixXcd stand-in).
struct MV {
    Index rows, cols;
    Complex* p;
    Complex& operator()(Index r, Index c) { return p[r + rows * c]; }
    const Complex& operator()(Index r, Index c) const { return p[r + rows * c]; }
};

// stacked_forward (src/matvec.cpp:17-65): min(workers, ncols) workers, each
// zeroing a private rows x p partial, pulling columns from an atomic queue,
// reconstructing each of the q tensors and adding vec(T) x(j,:); partials
// summed in worker order at the end.
void stacked_forward(const Store& z, const MV& x, MV& y, int workers, std::int64_t* ops) {
    if (x.rows != z.ncols)
        throw ContractViolation("stacked_forward: x has " + std::to_string(x.rows) +
                                " rows, expected " + std::to_string(z.ncols));
    const Index nv = z.nv();
    const Index rows = z.rows();
    const Index p = x.cols;
    const int nworkers = std::max<int>(1, std::min<Index>(workers, z.ncols));
    std::vector<std::vector<Complex>> partial(static_cast<std::size_t>(nworkers));
    std::atomic<Index> next{0};
    std::atomic<std::int64_t> dec_ops{0}, acc_ops{0};
    parallel_for(static_cast<std::size_t>(nworkers), nworkers, [&](std::size_t w) {
        std::vector<Complex>& yw = partial[w];
        yw.assign(static_cast<std::size_t>(rows * p), Complex(0));
        std::int64_t my_dec = 0, my_acc = 0;
        for (;;) {
            const Index j = next.fetch_add(1);
            if (j >= z.ncols) break;
            for (int k = 0; k < z.q; ++k) {
                const TuckerTensor& tt = z.at(j, k);
                const Tensor3 dense = reconstruct(tt);
                const Complex* dv = dense.data();
                for (Index c = 0; c < p; ++c) {
                    const Complex xc = x(j, c);
                    Complex* yc = yw.data() + rows * c + k * nv;
                    for (Index v = 0; v < nv; ++v) yc[v] += dv[v] * xc;
                }
                my_dec += reconstruct_madds(tt);
                my_acc += std::int64_t(nv) * p;
            }
        }
        dec_ops += my_dec;
        acc_ops += my_acc;
    });
    std::memcpy(y.p, partial[0].data(), sizeof(Complex) * static_cast<std::size_t>(rows * p));
    for (std::size_t w = 1; w < partial.size(); ++w)
        for (Index i = 0; i < rows * p; ++i) y.p[i] += partial[w][static_cast<std::size_t>(i)];
    if (ops) {
        ops[0] += dec_ops.load();
        ops[1] += acc_ops.load();
    }
}

// stacked_adjoint (src/matvec.cpp:67-102): per column j (parallel_for),
// row(j) = sum_k vec(T_jk)^H x_k.  Deterministic per row.
void stacked_adjoint(const Store& z, const MV& x, MV& y, int workers, std::int64_t* ops) {
    if (x.rows != z.rows())
        throw ContractViolation("stacked_adjoint: x has " + std::to_string(x.rows) +
                                " rows, expected " + std::to_string(z.rows()));
    const Index nv = z.nv();
    const Index p = x.cols;
    std::atomic<std::int64_t> dec_ops{0}, acc_ops{0};
    parallel_for(static_cast<std::size_t>(z.ncols), workers, [&](std::size_t jz) {
        const Index j = static_cast<Index>(jz);
        std::vector<Complex> row(static_cast<std::size_t>(p), Complex(0));
        std::int64_t my_dec = 0;
        for (int k = 0; k < z.q; ++k) {
            const TuckerTensor& tt = z.at(j, k);
            const Tensor3 dense = reconstruct(tt);
            const Complex* dv = dense.data();
            for (Index c = 0; c < p; ++c) {
                const Complex* xc = x.p + x.rows * c + k * nv;
                Complex s = 0;
                for (Index v = 0; v < nv; ++v) s += std::conj(dv[v]) * xc[v];
                row[c] += s;
            }
            my_dec += reconstruct_madds(tt);
        }
        for (Index c = 0; c < p; ++c) y(j, c) = row[c];
        dec_ops += my_dec;
        acc_ops += std::int64_t(z.q) * nv * p;
    });
    if (ops) {
        ops[0] += dec_ops.load();
        ops[1] += acc_ops.load();
    }
}

// ----------------------------------------------------------------- scene --
// Kernels follow src/scene.cpp:76-118; assembly src/scene.cpp:127-150.
constexpr double kSingularRadius = 1e-12;
struct Vec3 {
    double x, y, z;
};
struct Source {
    double mid[3];
    double dir[3];
    double weight;
};
struct Scene {
    double origin[3];
    double spacing;
    Index dims[3];
    int op;  // 0 = EField, 1 = HField
    double k0;
    int q;   // 3 = PWC (reference), 12 = PWL stand-in (this build's extension)
    const Source* src;
    Index nsrc;
    Vec3 center(Index i1, Index i2, Index i3) const {
        return {origin[0] + spacing * (double(i1) + 0.5), origin[1] + spacing * (double(i2) + 0.5),
                origin[2] + spacing * (double(i3) + 0.5)};
    }
};

struct SingularityError : Error {
    explicit SingularityError(const std::string& m) : Error(kSingularityError, m) {}
};

// efield_kernel (src/scene.cpp:84-103): curl curl (g w p) = A p + B (rhat.p) rhat.
void efield(const Source& s, const Vec3& obs, double k0, Complex out[3]) {
    if (!(k0 > 0)) throw ContractViolation("efield_kernel: k0 must be positive");
    const double rv[3] = {obs.x - s.mid[0], obs.y - s.mid[1], obs.z - s.mid[2]};
    const double R = std::sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
    if (R < kSingularRadius) throw SingularityError("efield_kernel: observation point hits the source");
    const double rh[3] = {rv[0] / R, rv[1] / R, rv[2] / R};
    const Complex g = std::polar(1.0 / (4.0 * std::numbers::pi * R), -k0 * R);
    const double R2 = R * R;
    const Complex a = g * Complex(k0 * k0 - 1.0 / R2, -k0 / R);
    const Complex b = g * Complex(-(k0 * k0) + 3.0 / R2, 3.0 * k0 / R);
    const double pr = rh[0] * s.dir[0] + rh[1] * s.dir[1] + rh[2] * s.dir[2];
    for (int c = 0; c < 3; ++c) out[c] = s.weight * (a * s.dir[c] + b * pr * rh[c]);
}

// hfield_kernel (src/scene.cpp:105-118): curl (g w p) = grad g x (w p).
void hfield(const Source& s, const Vec3& obs, double k0, Complex out[3]) {
    if (k0 < 0) throw ContractViolation("hfield_kernel: k0 must be non-negative");
    const double rv[3] = {obs.x - s.mid[0], obs.y - s.mid[1], obs.z - s.mid[2]};
    const double R = std::sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
    if (R < kSingularRadius) throw SingularityError("hfield_kernel: observation point hits the source");
    const double rh[3] = {rv[0] / R, rv[1] / R, rv[2] / R};
    const Complex g = std::polar(1.0 / (4.0 * std::numbers::pi * R), -k0 * R);
    const Complex gc = -g * Complex(1.0 / R, k0);
    const double cr[3] = {rh[1] * s.dir[2] - rh[2] * s.dir[1], rh[2] * s.dir[0] - rh[0] * s.dir[2],
                          rh[0] * s.dir[1] - rh[1] * s.dir[0]};
    for (int c = 0; c < 3; ++c) out[c] = (s.weight * gc) * cr[c];
}

void eval_kernel(const Scene& sc, const Source& s, const Vec3& obs, Complex out[3]) {
    if (sc.op == 0)
        efield(s, obs, sc.k0, out);
    else
        hfield(s, obs, sc.k0, out);
}

// Field samples of one voxel.  q = 3 is the reference's point-collocated
// piecewise-constant column (src/scene.cpp:141-147).  q = 12 is this
// build's piecewise-linear stand-in (the reference rejects q != 3,
// src/scene.cpp:47-48): component k = 4*c + mu holds the 2x2x2 Gauss
// moment of field component c against mu in {1, x~, y~, z~}, with
// x~ = (x - x_center)/h.
void voxel_field(const Scene& sc, const Source& s, Index i1, Index i2, Index i3, Complex* out) {
    const Vec3 c = sc.center(i1, i2, i3);
    if (sc.q == 3) {
        eval_kernel(sc, s, c, out);
        return;
    }
    for (int k = 0; k < 12; ++k) out[k] = 0;
    const double off = 0.5 / std::sqrt(3.0);  // Gauss nodes at +-h/(2 sqrt 3)
    for (int gz = 0; gz < 2; ++gz)
        for (int gy = 0; gy < 2; ++gy)
            for (int gx = 0; gx < 2; ++gx) {
                const double lx = gx ? off : -off, ly = gy ? off : -off, lz = gz ? off : -off;
                const Vec3 pt{c.x + sc.spacing * lx, c.y + sc.spacing * ly, c.z + sc.spacing * lz};
                Complex f[3];
                eval_kernel(sc, s, pt, f);
                const double phi[4] = {1.0, lx, ly, lz};
                for (int cc = 0; cc < 3; ++cc)
                    for (int mu = 0; mu < 4; ++mu) out[4 * cc + mu] += 0.125 * phi[mu] * f[cc];
            }
}

// assemble_column (src/scene.cpp:127-150): q grid tensors, f1-fastest,
// written component-major into out (q * n_v).
void assemble_column(const Scene& sc, Index j, Complex* out) {
    if (j < 0 || j >= sc.nsrc)
        throw ContractViolation("assemble_column: source index " + std::to_string(j) + " out of range");
    const Index nv = sc.dims[0] * sc.dims[1] * sc.dims[2];
    const Source& s = sc.src[j];
    Complex f[12];
    Index v = 0;
    for (Index i3 = 0; i3 < sc.dims[2]; ++i3)
        for (Index i2 = 0; i2 < sc.dims[1]; ++i2)
            for (Index i1 = 0; i1 < sc.dims[0]; ++i1, ++v) {
                voxel_field(sc, s, i1, i2, i3, f);
                for (int k = 0; k < sc.q; ++k) out[k * nv + v] = f[k];
            }
}

// -------------------------------------------------------------------- io --
// The CTC1/CTA1 byte layout of src/io.cpp:121-194 is restated in Python
// (oracle/oracle.py) for fixtures; the flat payload handed to orc_store_create
// is exactly the CTC1 per-tensor payload: core f1-fastest, then U1, U2, U3
// column-major, each complex as an (re, im) float64 pair.

Store* build_store(int q, Index ncols, const Index* dims, const std::int32_t* ranks,
                   const double* payload) {
    if (q < 1 || ncols < 0 || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
        throw ContractViolation("store: non-positive dimensions");
    auto* s = new Store;
    s->q = q;
    s->ncols = ncols;
    for (int g = 0; g < 3; ++g) s->dims[g] = dims[g];
    s->t.resize(static_cast<std::size_t>(ncols * q));
    const Complex* src = reinterpret_cast<const Complex*>(payload);
    std::size_t off = 0;
    for (Index i = 0; i < ncols * q; ++i) {
        TuckerTensor& tt = s->t[static_cast<std::size_t>(i)];
        const std::int32_t* r = ranks + 3 * i;
        for (int g = 0; g < 3; ++g) {
            if (r[g] < 1 || r[g] > dims[g]) {
                delete s;
                throw ContractViolation("store: tucker rank out of range for mode " + std::to_string(g + 1));
            }
            tt.dims[g] = dims[g];
        }
        tt.core = Tensor3(r[0], r[1], r[2]);
        std::memcpy(tt.core.data(), src + off, sizeof(Complex) * static_cast<std::size_t>(tt.core.size()));
        off += static_cast<std::size_t>(tt.core.size());
        for (int g = 0; g < 3; ++g) {
            tt.factors[g] = Matrix(dims[g], r[g]);
            std::memcpy(tt.factors[g].d.data(), src + off, sizeof(Complex) * tt.factors[g].d.size());
            off += tt.factors[g].d.size();
        }
    }
    return s;
}

}  // namespace orc

// ================================================================= C ABI ==
using namespace orc;

namespace {
template <class F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "allocation failed";
        return kCapacityError;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return kError;
    }
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_last_error.c_str(); }

int orc_store_create(int q, std::int64_t ncols, const std::int64_t* dims, const std::int32_t* ranks,
                     const double* payload, void** out) {
    return guarded([&] { *out = build_store(q, ncols, dims, ranks, payload); });
}

void orc_store_destroy(void* h) { delete static_cast<Store*>(h); }

// forward (src/matvec.cpp:132-138): x is m x p, y is q n_v x p (col-major).
int orc_forward(void* h, const double* x, std::int64_t xrows, std::int64_t p, double* y, int workers,
                std::int64_t* ops) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        if (xrows != s.ncols)
            throw ContractViolation("forward: x has " + std::to_string(xrows) + " rows, expected m = " +
                                    std::to_string(s.ncols));
        MV xv{xrows, p, reinterpret_cast<Complex*>(const_cast<double*>(x))};
        MV yv{s.rows(), p, reinterpret_cast<Complex*>(y)};
        stacked_forward(s, xv, yv, workers, ops);
    });
}

// adjoint (src/matvec.cpp:140-148): phi is q n_v x p, z is m x p.
int orc_adjoint(void* h, const double* phi, std::int64_t phirows, std::int64_t p, double* z, int workers,
                std::int64_t* ops) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        if (phirows != s.rows())
            throw ContractViolation("adjoint: phi has " + std::to_string(phirows) +
                                    " rows, expected q*n_v = " + std::to_string(s.rows()));
        MV xv{phirows, p, reinterpret_cast<Complex*>(const_cast<double*>(phi))};
        MV zv{s.ncols, p, reinterpret_cast<Complex*>(z)};
        stacked_adjoint(s, xv, zv, workers, ops);
    });
}

// aca_forward (src/matvec.cpp:150-160): w = V^H x (r_c x p), then
// stacked_forward over the Tucker U columns.  V is m2 x r_c col-major.
int orc_aca_forward(void* h, const double* v, std::int64_t m2, const double* x, std::int64_t xrows,
                    std::int64_t p, double* y, int workers) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        if (xrows != m2)
            throw ContractViolation("aca_forward: x has " + std::to_string(xrows) + " rows, expected " +
                                    std::to_string(m2));
        const Complex* V = reinterpret_cast<const Complex*>(v);
        const Complex* X = reinterpret_cast<const Complex*>(x);
        const Index rc = s.ncols;
        std::vector<Complex> w(static_cast<std::size_t>(rc * p));
        for (Index c = 0; c < p; ++c)
            for (Index l = 0; l < rc; ++l) {
                Complex acc = 0;
                for (Index i = 0; i < m2; ++i) acc += std::conj(V[i + m2 * l]) * X[i + m2 * c];
                w[static_cast<std::size_t>(l + rc * c)] = acc;
            }
        MV wv{rc, p, w.data()};
        MV yv{s.rows(), p, reinterpret_cast<Complex*>(y)};
        stacked_forward(s, wv, yv, workers, nullptr);
    });
}

// aca_adjoint (src/matvec.cpp:162-175): t = stacked_adjoint(U, phi), z = V t.
int orc_aca_adjoint(void* h, const double* v, std::int64_t m2, const double* phi, std::int64_t phirows,
                    std::int64_t p, double* z, int workers) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        if (phirows != s.rows())
            throw ContractViolation("aca_adjoint: phi has " + std::to_string(phirows) + " rows, expected " +
                                    std::to_string(s.rows()));
        const Index rc = s.ncols;
        std::vector<Complex> t(static_cast<std::size_t>(rc * p));
        MV xv{phirows, p, reinterpret_cast<Complex*>(const_cast<double*>(phi))};
        MV tv{rc, p, t.data()};
        stacked_adjoint(s, xv, tv, workers, nullptr);
        const Complex* V = reinterpret_cast<const Complex*>(v);
        Complex* Z = reinterpret_cast<Complex*>(z);
        for (Index c = 0; c < p; ++c)
            for (Index i = 0; i < m2; ++i) {
                Complex acc = 0;
                for (Index l = 0; l < rc; ++l) acc += V[i + m2 * l] * t[static_cast<std::size_t>(l + rc * c)];
                Z[i + m2 * c] = acc;
            }
    });
}

// OpCounts of one product at p right-hand sides (src/matvec.cpp:50-51,60-63).
int orc_opcounts(void* h, std::int64_t p, std::int64_t* dec, std::int64_t* acc) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        std::int64_t d = 0;
        for (const auto& tt : s.t) d += reconstruct_madds(tt);
        *dec = d;
        *acc = std::int64_t(s.ncols) * s.q * s.nv() * p;
    });
}

int orc_reconstruct(void* h, std::int64_t j, int k, double* out) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        if (j < 0 || j >= s.ncols || k < 0 || k >= s.q) throw ContractViolation("reconstruct: index out of range");
        const Tensor3 t = reconstruct(s.at(j, k));
        std::memcpy(out, t.data(), sizeof(Complex) * static_cast<std::size_t>(t.size()));
    });
}

int orc_element(void* h, std::int64_t j, int k, std::int64_t i1, std::int64_t i2, std::int64_t i3, double* out) {
    return guarded([&] {
        const Store& s = *static_cast<Store*>(h);
        if (j < 0 || j >= s.ncols || k < 0 || k >= s.q) throw ContractViolation("element: column out of range");
        const Complex e = element(s.at(j, k), i1, i2, i3);
        out[0] = e.real();
        out[1] = e.imag();
    });
}

// mode_product on raw buffers: t is (n1,n2,n3) f1-fastest, m is (mrows x
// extent) col-major.
int orc_mode_product(const double* t, const std::int64_t* tdims, const double* m, std::int64_t mrows,
                     std::int64_t mcols, int mode, double* out) {
    return guarded([&] {
        Tensor3 tt(tdims[0], tdims[1], tdims[2]);
        std::memcpy(static_cast<void*>(tt.data()), t, sizeof(Complex) * static_cast<std::size_t>(tt.size()));
        Matrix mm(mrows, mcols);
        std::memcpy(static_cast<void*>(mm.d.data()), m, sizeof(Complex) * mm.d.size());
        const Tensor3 o = mode_product(tt, mm, mode);
        std::memcpy(out, o.data(), sizeof(Complex) * static_cast<std::size_t>(o.size()));
    });
}

// Scene assembly: `src` is nsrc records of 7 doubles (mid xyz, dir xyz, w).
int orc_assemble_column(const double* origin, double spacing, const std::int64_t* dims, int op, double k0, int q,
                        const double* src, std::int64_t nsrc, std::int64_t j, double* out) {
    return guarded([&] {
        if (q != 3 && q != 12) throw ContractViolation("assemble: q must be 3 (PWC) or 12 (PWL)");
        static_assert(sizeof(Source) == 7 * sizeof(double));
        Scene sc{{origin[0], origin[1], origin[2]}, spacing, {dims[0], dims[1], dims[2]}, op, k0, q,
                 reinterpret_cast<const Source*>(src), nsrc};
        assemble_column(sc, j, reinterpret_cast<Complex*>(out));
    });
}

// Dense (q n_v x m) matrix, columns assembled in parallel (assemble_full,
// src/scene.cpp:156-175).
int orc_assemble_full(const double* origin, double spacing, const std::int64_t* dims, int op, double k0, int q,
                      const double* src, std::int64_t nsrc, int workers, double* out) {
    return guarded([&] {
        if (q != 3 && q != 12) throw ContractViolation("assemble: q must be 3 (PWC) or 12 (PWL)");
        Scene sc{{origin[0], origin[1], origin[2]}, spacing, {dims[0], dims[1], dims[2]}, op, k0, q,
                 reinterpret_cast<const Source*>(src), nsrc};
        const Index rows = q * dims[0] * dims[1] * dims[2];
        Complex* o = reinterpret_cast<Complex*>(out);
        parallel_for(static_cast<std::size_t>(nsrc), workers,
                     [&](std::size_t j) { assemble_column(sc, static_cast<Index>(j), o + rows * static_cast<Index>(j)); });
    });
}

// Single kernel evaluation (eval_kernel, src/scene.cpp:120-125).
int orc_eval_kernel(int op, double k0, const double* src7, const double* obs, double* out6) {
    return guarded([&] {
        Scene sc{};
        sc.op = op;
        sc.k0 = k0;
        Complex f[3];
        eval_kernel(sc, *reinterpret_cast<const Source*>(src7), Vec3{obs[0], obs[1], obs[2]}, f);
        for (int c = 0; c < 3; ++c) {
            out6[2 * c] = f[c].real();
            out6[2 * c + 1] = f[c].imag();
        }
    });
}

// random_multivector (src/experiments.cpp:26-33): mt19937_64 seeded with
// `seed`, normal_distribution(0,1), re then im, column-major.
void orc_random_multivector(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    for (std::int64_t c = 0; c < cols; ++c)
        for (std::int64_t r = 0; r < rows; ++r) {
            const double re = dist(rng);
            const double im = dist(rng);
            out[2 * (r + rows * c)] = re;
            out[2 * (r + rows * c) + 1] = im;
        }
}

// randn_c helper of tests/oracles.hpp:17-22 (one fresh distribution per
// draw, as the reference's test oracle does).
void orc_randn_tests(std::int64_t n, std::uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    for (std::int64_t i = 0; i < n; ++i) {
        std::normal_distribution<double> d(0.0, 1.0);
        out[2 * i] = d(rng);
        out[2 * i + 1] = d(rng);
    }
}

}  // extern "C"
