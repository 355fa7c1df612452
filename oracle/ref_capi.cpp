// TEST INFRASTRUCTURE ONLY — C face of the reference library compiled from
// /root/reference/proj/src/*.cpp UNCHANGED (oracle/Makefile target `ref`,
// Eigen and doctest replaced by the shims under oracle/eigen_shim and
// oracle/doctest_shim).  It is the parity anchor of the tests: the GPU path
// and the CPU restatement (oracle/tuckmat_oracle.cpp) are both compared with
// the reference's own forward / adjoint / aca_* / compress_matrix /
// tucker_aca / load_ctc1 / load_cta1 through these entry points.  Nothing in
// the product links or loads this library.
//
// Complex buffers are interleaved (re, im) doubles, column-major, like
// Eigen::MatrixXcd.  Every entry returns 0 or a nonzero error code with the
// message in ref_last_error().
#include <cstdint>
#include <cstring>
#include <string>

#include "tuckmat/aca.hpp"
#include "tuckmat/compress.hpp"
#include "tuckmat/io.hpp"
#include "tuckmat/matvec.hpp"
#include "tuckmat/scene.hpp"

using namespace tuckmat;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 5;
    } catch (const ContractViolation& e) {
        g_err = e.what();
        return 2;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 3;
    } catch (const SingularityError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

MultiVector from_buf(const double* b, std::int64_t rows, std::int64_t cols) {
    MultiVector m(rows, cols);
    std::memcpy(static_cast<void*>(m.data()), b, sizeof(Complex) * static_cast<size_t>(rows * cols));
    return m;
}

void to_buf(const MultiVector& m, double* b) {
    std::memcpy(b, static_cast<const void*>(m.data()), sizeof(Complex) * static_cast<size_t>(m.rows() * m.cols()));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// load_ctc1 (proj/src/io.cpp:198-219) -> CompressedCoupling*
int ref_load_ctc1(const char* path, void** out) {
    return guarded([&] { *out = new CompressedCoupling(load_ctc1(path)); });
}

// load_cta1 (proj/src/io.cpp:239-279) -> Cta1File*
int ref_load_cta1(const char* path, void** out) {
    return guarded([&] { *out = new Cta1File(load_cta1(path)); });
}

// A CompressedCoupling from raw arrays in CTC1 payload order: per column j,
// per component k: ranks (r1, r2, r3), core r1 r2 r3 (f1 fastest), then U1,
// U2, U3 column-major (proj/src/io.cpp:104-116).
int ref_cc_from_arrays(int q, std::int64_t m, const std::int64_t* dims, const std::int32_t* ranks,
                       const double* payload, void** out) {
    return guarded([&] {
        auto* cc = new CompressedCoupling;
        cc->q = q;
        cc->m = m;
        cc->grid_dims = {dims[0], dims[1], dims[2]};
        cc->columns.resize(static_cast<size_t>(m));
        const Complex* p = reinterpret_cast<const Complex*>(payload);
        for (std::int64_t j = 0; j < m; ++j)
            for (int k = 0; k < q; ++k) {
                const std::int32_t* r = ranks + 3 * (j * q + k);
                TuckerTensor tt;
                tt.dims = cc->grid_dims;
                tt.core = Tensor3(r[0], r[1], r[2]);
                for (Index i = 0; i < tt.core.size(); ++i) tt.core[i] = *p++;
                for (int g = 0; g < 3; ++g) {
                    Matrix& u = tt.factors[static_cast<size_t>(g)];
                    u.resize(dims[g], r[g]);
                    for (Index c = 0; c < u.cols(); ++c)
                        for (Index rr = 0; rr < u.rows(); ++rr) u(rr, c) = *p++;
                }
                cc->columns[static_cast<size_t>(j)].push_back(std::move(tt));
            }
        *out = cc;
    });
}

void ref_cc_destroy(void* h) { delete static_cast<CompressedCoupling*>(h); }
void ref_aca_destroy(void* h) { delete static_cast<Cta1File*>(h); }

int ref_cc_info(void* h, int* q, std::int64_t* m, std::int64_t* dims) {
    return guarded([&] {
        const auto* cc = static_cast<const CompressedCoupling*>(h);
        *q = cc->q;
        *m = cc->m;
        for (int g = 0; g < 3; ++g) dims[g] = cc->grid_dims[static_cast<size_t>(g)];
    });
}

int ref_aca_info(void* h, int* q, std::int64_t* rc, std::int64_t* m2, std::int64_t* dims) {
    return guarded([&] {
        const AcaFactors& f = static_cast<const Cta1File*>(h)->factors;
        *q = f.q;
        *rc = f.rank();
        *m2 = f.cols();
        for (int g = 0; g < 3; ++g) dims[g] = f.grid_dims[static_cast<size_t>(g)];
    });
}

int ref_save_ctc1(void* h, const char* path) {
    return guarded([&] { save_ctc1(path, *static_cast<const CompressedCoupling*>(h)); });
}

// forward / adjoint (proj/src/matvec.cpp:132-148), OpCounts added to ops[2]
int ref_forward(void* h, const double* x, std::int64_t xrows, std::int64_t p, int workers, double* y,
                std::int64_t* ops) {
    return guarded([&] {
        const auto& cc = *static_cast<const CompressedCoupling*>(h);
        OpCounts oc;
        const MultiVector r = forward(cc, from_buf(x, xrows, p), workers, &oc);
        to_buf(r, y);
        if (ops) {
            ops[0] += oc.decompress_madds;
            ops[1] += oc.accumulate_madds;
        }
    });
}

int ref_adjoint(void* h, const double* phi, std::int64_t phirows, std::int64_t p, int workers, double* z,
                std::int64_t* ops) {
    return guarded([&] {
        const auto& cc = *static_cast<const CompressedCoupling*>(h);
        OpCounts oc;
        const MultiVector r = adjoint(cc, from_buf(phi, phirows, p), workers, &oc);
        to_buf(r, z);
        if (ops) {
            ops[0] += oc.decompress_madds;
            ops[1] += oc.accumulate_madds;
        }
    });
}

// aca_forward / aca_adjoint (proj/src/matvec.cpp:150-175)
int ref_aca_forward(void* h, const double* x, std::int64_t xrows, std::int64_t p, int workers, double* y) {
    return guarded([&] {
        const AcaFactors& f = static_cast<const Cta1File*>(h)->factors;
        to_buf(aca_forward(f, from_buf(x, xrows, p), workers), y);
    });
}

int ref_aca_adjoint(void* h, const double* phi, std::int64_t phirows, std::int64_t p, int workers, double* z) {
    return guarded([&] {
        const AcaFactors& f = static_cast<const Cta1File*>(h)->factors;
        to_buf(aca_adjoint(f, from_buf(phi, phirows, p), workers), z);
    });
}

// element (proj/src/tensor.cpp:183-196) of tensor (column j, component k)
int ref_element(void* h, std::int64_t j, int k, std::int64_t i1, std::int64_t i2, std::int64_t i3, double* out) {
    return guarded([&] {
        const auto& cc = *static_cast<const CompressedCoupling*>(h);
        const Complex v = element(cc.columns.at(static_cast<size_t>(j)).at(static_cast<size_t>(k)), i1, i2, i3);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

// row_of_compressed_u (proj/src/aca.cpp:234-244)
int ref_row_of_compressed_u(void* h, std::int64_t i, double* out) {
    return guarded([&] {
        const AcaFactors& f = static_cast<const Cta1File*>(h)->factors;
        to_buf(MultiVector(row_of_compressed_u(f, i)), out);
    });
}

// ---------------------------------------------------------------- scenes --
// SceneSpec from explicit sources (m x 7 doubles: midpoint xyz, unit
// direction xyz, weight), validated by the reference (validate_scene).
int ref_scene_create(const double* origin, double spacing, const std::int64_t* dims, int op, double k0,
                     const double* src, std::int64_t m, void** out) {
    return guarded([&] {
        auto* s = new SceneSpec;
        s->grid.origin = Vector3(origin[0], origin[1], origin[2]);
        s->grid.spacing = spacing;
        s->grid.dims = {dims[0], dims[1], dims[2]};
        s->kernel = {op == 0 ? KernelOp::EField : KernelOp::HField, k0, 3};
        for (std::int64_t j = 0; j < m; ++j) {
            EdgeSource e;
            e.midpoint = Vector3(src[7 * j], src[7 * j + 1], src[7 * j + 2]);
            e.direction = Vector3(src[7 * j + 3], src[7 * j + 4], src[7 * j + 5]);
            e.weight = src[7 * j + 6];
            s->sources.push_back(e);
        }
        try {
            validate_scene(*s);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

// make_centered_grid + make_loop_scene (proj/src/scene.cpp:17-31,179-205)
int ref_loop_scene(double spacing, const std::int64_t* dims, const double* grid_center, double radius,
                   const double* center, int nseg, int op, double k0, void** out) {
    return guarded([&] {
        const VoxelGrid g = make_centered_grid(Vector3(grid_center[0], grid_center[1], grid_center[2]), spacing,
                                               {dims[0], dims[1], dims[2]});
        const KernelSpec kernel{op == 0 ? KernelOp::EField : KernelOp::HField, k0, 3};
        *out = new SceneSpec(make_loop_scene(radius, Vector3(center[0], center[1], center[2]), nseg, g, kernel));
    });
}

void ref_scene_destroy(void* h) { delete static_cast<SceneSpec*>(h); }

// origin[3], spacing, and the m x 7 source table of a scene
int ref_scene_sources(void* h, double* origin, double* spacing, double* src) {
    return guarded([&] {
        const auto& s = *static_cast<const SceneSpec*>(h);
        for (int a = 0; a < 3; ++a) origin[a] = s.grid.origin[a];
        *spacing = s.grid.spacing;
        for (size_t j = 0; j < s.sources.size(); ++j) {
            const EdgeSource& e = s.sources[j];
            for (int a = 0; a < 3; ++a) {
                src[7 * j + a] = e.midpoint[a];
                src[7 * j + 3 + a] = e.direction[a];
            }
            src[7 * j + 6] = e.weight;
        }
    });
}

// compress_matrix (proj/src/compress.cpp:7-35) -> CompressedCoupling*
int ref_compress(void* scene, double eps, int workers, void** out) {
    return guarded([&] { *out = new CompressedCoupling(compress_matrix(*static_cast<SceneSpec*>(scene), eps, workers)); });
}

// tucker_aca over coupling_oracle (proj/src/aca.cpp:126-232,246-277), saved as
// CTA1 (proj/src/io.cpp:221-237) and returned as a Cta1File*
int ref_tucker_aca(void* scene, double eps, double hosvd_eps, const char* path, void** out) {
    return guarded([&] {
        const SceneSpec& s = *static_cast<SceneSpec*>(scene);
        const AcaFactors f = tucker_aca(coupling_oracle(s), s.grid.dims, s.kernel.q, eps, hosvd_eps);
        save_cta1(path, f, s.kernel.k0, s.kernel.op);
        *out = new Cta1File(load_cta1(path));
    });
}

// assemble_column (proj/src/scene.cpp:127-150): q * n_v complex values
int ref_assemble_column(void* scene, std::int64_t j, double* out) {
    return guarded([&] {
        const SceneSpec& s = *static_cast<SceneSpec*>(scene);
        const std::vector<Tensor3> t = assemble_column(s, j);
        const std::int64_t nv = s.grid.num_voxels();
        for (size_t k = 0; k < t.size(); ++k)
            std::memcpy(out + 2 * nv * static_cast<std::int64_t>(k), static_cast<const void*>(t[k].data()),
                        sizeof(Complex) * static_cast<size_t>(nv));
    });
}

// dense_forward / dense_adjoint (proj/src/matvec.cpp:177-196)
int ref_dense_forward(void* scene, const double* x, std::int64_t p, double* y) {
    return guarded([&] {
        const SceneSpec& s = *static_cast<SceneSpec*>(scene);
        to_buf(dense_forward(s, from_buf(x, s.num_sources(), p)), y);
    });
}

int ref_dense_adjoint(void* scene, const double* phi, std::int64_t p, double* z) {
    return guarded([&] {
        const SceneSpec& s = *static_cast<SceneSpec*>(scene);
        to_buf(dense_adjoint(s, from_buf(phi, s.kernel.q * s.grid.num_voxels(), p)), z);
    });
}

}  // extern "C"
