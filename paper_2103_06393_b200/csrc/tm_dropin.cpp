// C++ drop-in of the reference matvec API on top of the C ABI
// (include/tuckmat_b200/tuckmat.hpp).  Host glue only: flatten the
// reference value types into a tm_store_desc, keep the device store cached
// by content (a hash of the factors), convert MultiVector blocks to the store precision and
// map status codes back onto the reference exception types.
#include "../../include/tuckmat_b200/tuckmat.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <thread>

#include "tm_io_internal.hpp"

namespace tuckmat {

double Matrix::norm() const {
    double s = 0;
    for (const Complex& z : d_) s += std::norm(z);
    return std::sqrt(s);
}

Tensor3::Tensor3(Index n1, Index n2, Index n3) : dims_{n1, n2, n3} {
    if (n1 <= 0 || n2 <= 0 || n3 <= 0) throw ContractViolation("Tensor3: dimensions must be positive");
    data_.assign(static_cast<std::size_t>(n1 * n2 * n3), Complex(0));
}

std::int64_t reconstruct_madds(const TuckerTensor& tt) {
    const Index n1 = tt.dims[0], n2 = tt.dims[1], n3 = tt.dims[2];
    const Index r1 = tt.core.dim(1), r2 = tt.core.dim(2), r3 = tt.core.dim(3);
    return std::int64_t(n1) * r1 * r2 * r3 + std::int64_t(n1) * n2 * r2 * r3 + std::int64_t(n1) * n2 * n3 * r3;
}

namespace {

[[noreturn]] void rethrow(int st) {
    const std::string msg = tm_last_error();
    switch (st) {
    case TM_CONTRACT_VIOLATION:
        throw ContractViolation(msg);
    case TM_CAPACITY_ERROR:
        throw CapacityError(msg);
    case TM_PARSE_ERROR: {
        std::uint64_t off = 0;
        const auto p = msg.rfind("(byte offset ");
        if (p != std::string::npos) off = std::strtoull(msg.c_str() + p + 13, nullptr, 10);
        throw ParseError(msg, off);
    }
    default:
        throw Error(msg);
    }
}

void check(int st) {
    if (st != TM_OK) rethrow(st);
}

struct Flat {
    std::vector<std::int32_t> ranks;
    std::vector<double> payload;
};

void append_tensor(Flat& f, const TuckerTensor& tt, const Dims3& dims) {
    for (int g = 0; g < 3; ++g) {
        if (tt.factors[g].rows() != dims[g] || tt.factors[g].cols() != tt.core.dim(g + 1))
            throw ContractViolation("TuckerTensor factor " + std::to_string(g + 1) + " does not match the core");
        f.ranks.push_back(static_cast<std::int32_t>(tt.core.dim(g + 1)));
    }
    auto put = [&](const Complex* p, Index n) {
        for (Index i = 0; i < n; ++i) {
            f.payload.push_back(p[i].real());
            f.payload.push_back(p[i].imag());
        }
    };
    put(tt.core.data(), tt.core.size());
    for (int g = 0; g < 3; ++g) put(tt.factors[g].data(), tt.factors[g].size());
}

// Flattens the columns (and V) into a tm_store_desc and hands it to `create`
// (tm_store_create or tm_sharded_create).
template <typename Create>
void with_desc(int q, Index ncols, const Dims3& dims, const std::function<const TuckerTensor&(Index, int)>& at,
               const Matrix* v, Create create) {
    Flat f;
    for (Index j = 0; j < ncols; ++j)
        for (int k = 0; k < q; ++k) append_tensor(f, at(j, k), dims);
    std::vector<double> vbuf;
    tm_store_desc d{};
    d.q = q;
    d.ncols = ncols;
    for (int g = 0; g < 3; ++g) d.dims[g] = dims[g];
    d.ranks = f.ranks.data();
    d.payload = f.payload.data();
    if (v) {
        vbuf.reserve(static_cast<std::size_t>(2 * v->size()));
        for (Index i = 0; i < v->size(); ++i) {
            vbuf.push_back(v->data()[i].real());
            vbuf.push_back(v->data()[i].imag());
        }
        d.v = vbuf.data();
        d.m2 = v->rows();
    }
    create(d);
}

tm_store* make_store(int q, Index ncols, const Dims3& dims,
                     const std::function<const TuckerTensor&(Index, int)>& at, const Matrix* v, int dtype,
                     int device) {
    tm_store* h = nullptr;
    with_desc(q, ncols, dims, at, v, [&](const tm_store_desc& d) { check(tm_store_create(&d, device, dtype, &h)); });
    return h;
}

// ---- content-keyed store cache -------------------------------------------
// The reference's value types are immutable and passed by const& on every
// call (src/matvec.cpp:132-175), so the drop-in keeps the device store it
// built for a given CONTENT: the key is a 64-bit hash of every tensor's
// ranks and payload (and V), plus shape, dtype and device.  An object whose
// address is reused for different data (a loop that rebuilds its factors)
// hashes differently and gets a fresh store; identical content in another
// object reuses the store.  Least-recently-used eviction bounds the device
// memory held ($TUCKMAT_STORE_CACHE stores, default 4).
struct Key {
    std::uint64_t hash;
    Index ncols, m2;
    int q, dtype, device, kind;
    Index d0, d1, d2;
    bool operator==(const Key& o) const {
        return hash == o.hash && ncols == o.ncols && m2 == o.m2 && q == o.q && dtype == o.dtype &&
               device == o.device && kind == o.kind && d0 == o.d0 && d1 == o.d1 && d2 == o.d2;
    }
};

std::mutex g_mu;
std::list<std::pair<Key, std::shared_ptr<tm_store>>> g_cache;  // front = most recently used
int g_dtype = TM_C128;
int g_device = -1;

int current_device() {
    if (g_device >= 0) return g_device;
    if (const char* e = std::getenv("TUCKMAT_DEVICE")) return std::atoi(e);
    return 0;
}

std::size_t cache_capacity() {
    if (const char* e = std::getenv("TUCKMAT_STORE_CACHE")) {
        const long v = std::atol(e);
        if (v >= 0) return std::size_t(v);
    }
    return 4;
}

inline std::uint64_t mix(std::uint64_t h, std::uint64_t w) {
    h ^= w + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    return h * 0xBF58476D1CE4E5B9ull;
}

std::uint64_t hash_words(std::uint64_t h, const void* p, std::size_t bytes) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    std::size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        std::uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = mix(h, w);
    }
    std::uint64_t tail = 0;
    std::memcpy(&tail, b + i, bytes - i);
    return mix(h, tail ^ bytes);
}

std::uint64_t hash_tensor(const TuckerTensor& tt) {
    std::uint64_t h = 0x12345678ull;
    for (int g = 0; g < 3; ++g) h = mix(h, std::uint64_t(tt.core.dim(g + 1)) | (std::uint64_t(tt.factors[g].rows()) << 32));
    h = hash_words(h, tt.core.data(), sizeof(Complex) * std::size_t(tt.core.size()));
    for (int g = 0; g < 3; ++g) h = hash_words(h, tt.factors[g].data(), sizeof(Complex) * std::size_t(tt.factors[g].size()));
    return h;
}

// Hash of ncols x q tensors, computed per tensor on a few threads (a
// config-4 store is 6 GB of complex128) and combined in tensor order.
std::uint64_t hash_columns(int q, Index ncols, const std::function<const TuckerTensor&(Index, int)>& at) {
    const Index nt = ncols * q;
    std::vector<std::uint64_t> ht(static_cast<std::size_t>(nt));
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nth = nt > 64 ? hw : 1;
    std::atomic<Index> next{0};
    auto work = [&]() {
        for (;;) {
            const Index t0 = next.fetch_add(16);
            if (t0 >= nt) return;
            for (Index t = t0; t < std::min(nt, t0 + 16); ++t) ht[std::size_t(t)] = hash_tensor(at(t / q, int(t % q)));
        }
    };
    std::vector<std::thread> pool;
    for (unsigned i = 1; i < nth; ++i) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    std::uint64_t h = mix(0xC0FFEEull, std::uint64_t(nt));
    for (std::uint64_t v : ht) h = mix(h, v);
    return h;
}

std::shared_ptr<tm_store> cached(const Key& key, const std::function<tm_store*()>& make) {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
        if (it->first == key) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front().second;
        }
    std::shared_ptr<tm_store> s(make(), [](tm_store* p) { tm_store_destroy(p); });
    const std::size_t cap = cache_capacity();
    if (cap == 0) return s;  // caching disabled: the store lives as long as the call
    g_cache.emplace_front(key, s);
    while (g_cache.size() > cap) g_cache.pop_back();  // in-flight users keep their shared_ptr
    return s;
}

// ---- products through the C ABI -------------------------------------------
// dtype-converting host call: MultiVector is complex128; a TM_C64 store takes
// complex64 blocks.
template <typename Call>
MultiVector run(tm_store* s, int dtype, const MultiVector& in, Index outrows, Call call) {
    const Index p = in.cols();
    MultiVector out(outrows, p);
    if (dtype == TM_C128) {
        check(call(in.data(), std::max<Index>(in.rows(), 1), out.data(), std::max<Index>(outrows, 1)));
        return out;
    }
    std::vector<std::complex<float>> a(static_cast<std::size_t>(in.size())), b(static_cast<std::size_t>(outrows * p));
    for (Index i = 0; i < in.size(); ++i) a[static_cast<std::size_t>(i)] = std::complex<float>(in.data()[i]);
    check(call(a.data(), std::max<Index>(in.rows(), 1), b.data(), std::max<Index>(outrows, 1)));
    for (Index i = 0; i < outrows * p; ++i) out.data()[i] = Complex(b[static_cast<std::size_t>(i)]);
    (void)s;
    return out;
}

Index store_rows(tm_store* s) {
    std::int32_t q = 0;
    std::int64_t ncols = 0, dims[3] = {0, 0, 0};
    check(tm_store_info(s, &q, &ncols, dims, nullptr, nullptr, nullptr));
    return q * dims[0] * dims[1] * dims[2];
}

Index store_cols(tm_store* s) {
    std::int64_t ncols = 0;
    check(tm_store_info(s, nullptr, &ncols, nullptr, nullptr, nullptr, nullptr));
    return ncols;
}

Index store_m2(tm_store* s) {
    std::int64_t m2 = 0;
    check(tm_store_info(s, nullptr, nullptr, nullptr, nullptr, &m2, nullptr));
    return m2;
}

MultiVector fwd(tm_store* s, int dtype, const MultiVector& x, OpCounts* ops) {
    std::int64_t o[2] = {0, 0};
    MultiVector y = run(s, dtype, x, store_rows(s), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_forward(s, in, ldi, x.rows(), x.cols(), out, ldo, TM_HOST, nullptr, o);
    });
    if (ops) {
        ops->decompress_madds += o[0];
        ops->accumulate_madds += o[1];
    }
    return y;
}

MultiVector adj(tm_store* s, int dtype, const MultiVector& phi, OpCounts* ops) {
    std::int64_t o[2] = {0, 0};
    MultiVector z = run(s, dtype, phi, store_cols(s), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_adjoint(s, in, ldi, phi.rows(), phi.cols(), out, ldo, TM_HOST, nullptr, o);
    });
    if (ops) {
        ops->decompress_madds += o[0];
        ops->accumulate_madds += o[1];
    }
    return z;
}

MultiVector aca_fwd(tm_store* s, int dtype, const MultiVector& x) {
    return run(s, dtype, x, store_rows(s), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_aca_forward(s, in, ldi, x.rows(), x.cols(), out, ldo, TM_HOST, nullptr);
    });
}

MultiVector aca_adj(tm_store* s, int dtype, const MultiVector& phi) {
    return run(s, dtype, phi, store_m2(s), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_aca_adjoint(s, in, ldi, phi.rows(), phi.cols(), out, ldo, TM_HOST, nullptr);
    });
}

Key key_of(int kind, int q, Index ncols, const Dims3& dims, Index m2, std::uint64_t h) {
    return Key{h, ncols, m2, q, g_dtype, current_device(), kind, dims[0], dims[1], dims[2]};
}

std::shared_ptr<tm_store> store_of(const TuckerColumns& z) {
    const std::uint64_t h = hash_columns(z.q, z.ncols, z.tensor);
    return cached(key_of(0, z.q, z.ncols, z.grid_dims, 0, h),
                  [&] { return make_store(z.q, z.ncols, z.grid_dims, z.tensor, nullptr, g_dtype, current_device()); });
}

std::shared_ptr<tm_store> store_of(const CompressedCoupling& cc) {
    if (static_cast<Index>(cc.columns.size()) != cc.m) throw ContractViolation("CompressedCoupling: columns != m");
    for (const auto& col : cc.columns)
        if (static_cast<int>(col.size()) != cc.q) throw ContractViolation("CompressedCoupling: column with wrong component count");
    TuckerColumns z;
    z.tensor = [&](Index j, int k) -> const TuckerTensor& {
        return cc.columns[static_cast<std::size_t>(j)][static_cast<std::size_t>(k)];
    };
    z.ncols = cc.m;
    z.q = cc.q;
    z.grid_dims = cc.grid_dims;
    return store_of(z);
}

std::shared_ptr<tm_store> store_of(const AcaFactors& f) {
    auto at = [&](Index l, int k) -> const TuckerTensor& {
        return f.tucker_u[static_cast<std::size_t>(k)][static_cast<std::size_t>(l)];
    };
    if (static_cast<int>(f.tucker_u.size()) != f.q) throw ContractViolation("AcaFactors: tucker_u needs q rows");
    for (const auto& row : f.tucker_u)
        if (static_cast<Index>(row.size()) != f.rank()) throw ContractViolation("AcaFactors: tucker_u rows need r_c tensors");
    std::uint64_t h = hash_columns(f.q, f.rank(), at);
    h = hash_words(h, f.v.data(), sizeof(Complex) * std::size_t(f.v.size()));
    return cached(key_of(1, f.q, f.rank(), f.grid_dims, f.v.rows(), h),
                  [&] { return make_store(f.q, f.rank(), f.grid_dims, at, &f.v, g_dtype, current_device()); });
}

// AcaFactors with a dense U (aca_forward / aca_adjoint's `fac.dense_u`
// branches, src/matvec.cpp:158,173): a dense-U device store.
std::shared_ptr<tm_store> dense_store_of(const AcaFactors& f) {
    if (f.dense_u.cols() != f.v.cols()) throw ContractViolation("AcaFactors: dense_u and v column counts differ");
    std::uint64_t h = hash_words(0xDE05Eull, f.dense_u.data(), sizeof(Complex) * std::size_t(f.dense_u.size()));
    h = hash_words(h, f.v.data(), sizeof(Complex) * std::size_t(f.v.size()));
    const Dims3 d{f.dense_u.rows(), 1, 1};
    return cached(key_of(2, 1, f.rank(), d, f.v.rows(), h), [&] {
        tm_store* st = nullptr;
        check(tm_store_create_dense_aca(reinterpret_cast<const double*>(f.dense_u.data()), f.dense_u.rows(),
                                        reinterpret_cast<const double*>(f.v.data()), f.v.rows(), f.rank(), 0,
                                        current_device(), g_dtype, &st));
        return st;
    });
}

}  // namespace

// ---- reference API ----------------------------------------------------------
MultiVector forward(const CompressedCoupling& cc, const MultiVector& x, int, OpCounts* ops) {
    if (x.rows() != cc.m)
        throw ContractViolation("forward: x has " + std::to_string(x.rows()) + " rows, expected m = " +
                                std::to_string(cc.m));
    auto s = store_of(cc);
    return fwd(s.get(), g_dtype, x, ops);
}

MultiVector adjoint(const CompressedCoupling& cc, const MultiVector& phi, int, OpCounts* ops) {
    if (phi.rows() != cc.rows())
        throw ContractViolation("adjoint: phi has " + std::to_string(phi.rows()) + " rows, expected q*n_v = " +
                                std::to_string(cc.rows()));
    auto s = store_of(cc);
    return adj(s.get(), g_dtype, phi, ops);
}

MultiVector stacked_forward(const TuckerColumns& z, const MultiVector& x, int, OpCounts* ops) {
    if (x.rows() != z.ncols)
        throw ContractViolation("stacked_forward: x has " + std::to_string(x.rows()) + " rows, expected " +
                                std::to_string(z.ncols));
    auto s = store_of(z);
    return fwd(s.get(), g_dtype, x, ops);
}

MultiVector stacked_adjoint(const TuckerColumns& z, const MultiVector& x, int, OpCounts* ops) {
    if (x.rows() != z.rows())
        throw ContractViolation("stacked_adjoint: x has " + std::to_string(x.rows()) + " rows, expected " +
                                std::to_string(z.rows()));
    auto s = store_of(z);
    return adj(s.get(), g_dtype, x, ops);
}

namespace {
// One row of a store through tm_rows, in the store's dtype, as complex<double>.
std::vector<Complex> store_row(tm_store* s, int dtype, Index row, Index ncols) {
    std::vector<Complex> r(static_cast<std::size_t>(ncols));
    const std::int64_t idx = row;
    if (dtype == TM_C128) {
        check(tm_rows(s, &idx, 1, r.data(), 1, TM_HOST, nullptr));
    } else {
        std::vector<std::complex<float>> f(static_cast<std::size_t>(ncols));
        check(tm_rows(s, &idx, 1, f.data(), 1, TM_HOST, nullptr));
        for (std::size_t i = 0; i < f.size(); ++i) r[i] = Complex(f[i].real(), f[i].imag());
    }
    return r;
}
}  // namespace

Complex element(const TuckerTensor& tt, Index i1, Index i2, Index i3) {
    const Dims3 d = tt.dims;
    if (i1 < 0 || i1 >= d[0] || i2 < 0 || i2 >= d[1] || i3 < 0 || i3 >= d[2])
        throw ContractViolation("element: index out of range");
    TuckerColumns z;
    z.ncols = 1;
    z.q = 1;
    z.grid_dims = d;
    z.tensor = [&](Index, int) -> const TuckerTensor& { return tt; };
    auto s = store_of(z);
    return store_row(s.get(), g_dtype, i1 + d[0] * (i2 + d[1] * i3), 1)[0];
}

MultiVector row_of_compressed_u(const AcaFactors& fac, Index i) {
    if (!fac.compressed()) throw ContractViolation("row_of_compressed_u: U is stored dense");
    if (i < 0 || i >= fac.rows()) throw ContractViolation("element: index out of range");
    auto s = store_of(fac);
    const std::vector<Complex> r = store_row(s.get(), g_dtype, i, fac.rank());
    MultiVector out(1, fac.rank());
    for (Index l = 0; l < fac.rank(); ++l) out(0, l) = r[static_cast<std::size_t>(l)];
    return out;
}

MultiVector aca_forward(const AcaFactors& fac, const MultiVector& x, int) {
    if (x.rows() != fac.cols())
        throw ContractViolation("aca_forward: x has " + std::to_string(x.rows()) + " rows, expected " +
                                std::to_string(fac.cols()));
    auto s = fac.compressed() ? store_of(fac) : dense_store_of(fac);
    return aca_fwd(s.get(), g_dtype, x);
}

MultiVector aca_adjoint(const AcaFactors& fac, const MultiVector& phi, int) {
    if (phi.rows() != fac.rows())
        throw ContractViolation("aca_adjoint: phi has " + std::to_string(phi.rows()) + " rows, expected " +
                                std::to_string(fac.rows()));
    auto s = fac.compressed() ? store_of(fac) : dense_store_of(fac);
    return aca_adj(s.get(), g_dtype, phi);
}

// ---- io ------------------------------------------------------------------
namespace {

std::vector<std::vector<TuckerTensor>> unpack(const tmb_io::Parsed& p, bool aca) {
    const Dims3 dims{p.dims[0], p.dims[1], p.dims[2]};
    std::vector<std::vector<TuckerTensor>> out;
    if (aca)
        out.assign(p.q, std::vector<TuckerTensor>(p.m));
    else
        out.assign(p.m, std::vector<TuckerTensor>(p.q));
    std::size_t off = 0;
    const Complex* src = reinterpret_cast<const Complex*>(p.payload.data());
    for (std::uint32_t j = 0; j < p.m; ++j)
        for (std::uint32_t k = 0; k < p.q; ++k) {
            TuckerTensor& tt = aca ? out[k][j] : out[j][k];
            const std::int32_t* r = &p.ranks[3 * (std::size_t(j) * p.q + k)];
            tt.dims = dims;
            tt.core = Tensor3(r[0], r[1], r[2]);
            for (Index i = 0; i < tt.core.size(); ++i) tt.core[i] = src[off++];
            for (int g = 0; g < 3; ++g) {
                tt.factors[g] = Matrix(dims[g], r[g]);
                for (Index i = 0; i < tt.factors[g].size(); ++i) tt.factors[g].data()[i] = src[off++];
            }
        }
    return out;
}

template <typename F>
auto parse_or_throw(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const tmb_io::ParseFail& e) {
        throw ParseError(e.what(), e.offset);
    }
}

}  // namespace

CompressedCoupling load_ctc1(const std::string& path) {
    return parse_or_throw([&] {
        const tmb_io::Parsed p = tmb_io::parse(path, false);
        CompressedCoupling cc;
        cc.grid_dims = {p.dims[0], p.dims[1], p.dims[2]};
        cc.q = int(p.q);
        cc.m = p.m;
        cc.kernel_op = static_cast<KernelOp>(p.op);
        cc.k0 = p.k0;
        cc.eps = p.eps;
        cc.columns = unpack(p, false);
        return cc;
    });
}

Cta1File load_cta1(const std::string& path) {
    return parse_or_throw([&] {
        const tmb_io::Parsed p = tmb_io::parse(path, true);
        Cta1File f;
        f.k0 = p.k0;
        f.kernel_op = static_cast<KernelOp>(p.op);
        AcaFactors& fac = f.factors;
        fac.grid_dims = {p.dims[0], p.dims[1], p.dims[2]};
        fac.q = int(p.q);
        fac.eps = p.eps;
        fac.tucker_u = unpack(p, true);
        fac.v = Matrix(Index(p.m2), Index(p.m));
        const Complex* v = reinterpret_cast<const Complex*>(p.v.data());
        for (Index i = 0; i < fac.v.size(); ++i) fac.v.data()[i] = v[i];
        return f;
    });
}

// ---- B200 extensions ----------------------------------------------------
namespace b200 {

void set_default_dtype(int dtype) {
    if (dtype != TM_C64 && dtype != TM_C128) throw ContractViolation("dtype must be TM_C64 or TM_C128");
    g_dtype = dtype;
}
int default_dtype() { return g_dtype; }
void set_device(int device) { g_device = device; }
void clear_cache() {
    std::lock_guard<std::mutex> lock(g_mu);
    g_cache.clear();
}

DeviceStore::DeviceStore(const CompressedCoupling& cc, int dtype, int device) : dtype_(dtype) {
    h_ = make_store(
        cc.q, cc.m, cc.grid_dims,
        [&](Index j, int k) -> const TuckerTensor& {
            return cc.columns[static_cast<std::size_t>(j)][static_cast<std::size_t>(k)];
        },
        nullptr, dtype, device);
}

DeviceStore::DeviceStore(const AcaFactors& f, int dtype, int device) : dtype_(dtype) {
    h_ = make_store(
        f.q, f.rank(), f.grid_dims,
        [&](Index l, int k) -> const TuckerTensor& {
            return f.tucker_u[static_cast<std::size_t>(k)][static_cast<std::size_t>(l)];
        },
        &f.v, dtype, device);
}

DeviceStore::DeviceStore(const TuckerColumns& z, int dtype, int device) : dtype_(dtype) {
    h_ = make_store(z.q, z.ncols, z.grid_dims, z.tensor, nullptr, dtype, device);
}

DeviceStore::~DeviceStore() {
    if (h_) tm_store_destroy(h_);
}

MultiVector forward(const DeviceStore& s, const MultiVector& x, OpCounts* ops) {
    return fwd(s.handle(), s.dtype(), x, ops);
}
MultiVector adjoint(const DeviceStore& s, const MultiVector& phi, OpCounts* ops) {
    return adj(s.handle(), s.dtype(), phi, ops);
}
MultiVector aca_forward(const DeviceStore& s, const MultiVector& x) { return aca_fwd(s.handle(), s.dtype(), x); }
MultiVector aca_adjoint(const DeviceStore& s, const MultiVector& phi) { return aca_adj(s.handle(), s.dtype(), phi); }

// ---- multi-GPU ---------------------------------------------------------
Communicator::Communicator(const std::vector<int>& devices) {
    check(tm_comm_init(int(devices.size()), devices.data(), &h_));
}
Communicator::~Communicator() {
    if (h_) tm_comm_finalize(h_);
}

ShardedStore::ShardedStore(const CompressedCoupling& cc, Communicator& comm, int dtype, int mode) : dtype_(dtype) {
    with_desc(
        cc.q, cc.m, cc.grid_dims,
        [&](Index j, int k) -> const TuckerTensor& {
            return cc.columns[static_cast<std::size_t>(j)][static_cast<std::size_t>(k)];
        },
        nullptr, [&](const tm_store_desc& d) { check(tm_sharded_create_mode(&d, comm.handle(), dtype, mode, &h_)); });
    rows_ = cc.rows();
    cols_ = cc.m;
}

ShardedStore::ShardedStore(const AcaFactors& f, Communicator& comm, int dtype, int mode) : dtype_(dtype) {
    if (!f.compressed()) throw ContractViolation("ShardedStore: AcaFactors needs a Tucker-compressed U");
    with_desc(
        f.q, f.rank(), f.grid_dims,
        [&](Index l, int k) -> const TuckerTensor& {
            return f.tucker_u[static_cast<std::size_t>(k)][static_cast<std::size_t>(l)];
        },
        &f.v, [&](const tm_store_desc& d) { check(tm_sharded_create_mode(&d, comm.handle(), dtype, mode, &h_)); });
    rows_ = f.rows();
    cols_ = f.rank();
    m2_ = f.cols();
}

ShardedStore::~ShardedStore() {
    if (h_) tm_sharded_destroy(h_);
}

MultiVector forward(const ShardedStore& s, const MultiVector& x, OpCounts* ops) {
    std::int64_t o[2] = {0, 0};
    MultiVector y = run(nullptr, s.dtype(), x, s.rows(), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_sharded_forward(s.handle(), in, ldi, x.rows(), x.cols(), out, ldo, TM_HOST, nullptr, o);
    });
    if (ops) {
        ops->decompress_madds += o[0];
        ops->accumulate_madds += o[1];
    }
    return y;
}
MultiVector adjoint(const ShardedStore& s, const MultiVector& phi, OpCounts* ops) {
    std::int64_t o[2] = {0, 0};
    MultiVector z = run(nullptr, s.dtype(), phi, s.cols(), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_sharded_adjoint(s.handle(), in, ldi, phi.rows(), phi.cols(), out, ldo, TM_HOST, nullptr, o);
    });
    if (ops) {
        ops->decompress_madds += o[0];
        ops->accumulate_madds += o[1];
    }
    return z;
}
MultiVector aca_forward(const ShardedStore& s, const MultiVector& x) {
    return run(nullptr, s.dtype(), x, s.rows(), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_sharded_aca_forward(s.handle(), in, ldi, x.rows(), x.cols(), out, ldo, TM_HOST, nullptr);
    });
}
MultiVector aca_adjoint(const ShardedStore& s, const MultiVector& phi) {
    return run(nullptr, s.dtype(), phi, s.m2(), [&](const void* in, Index ldi, void* out, Index ldo) {
        return tm_sharded_aca_adjoint(s.handle(), in, ldi, phi.rows(), phi.cols(), out, ldo, TM_HOST, nullptr);
    });
}

}  // namespace b200
}  // namespace tuckmat
