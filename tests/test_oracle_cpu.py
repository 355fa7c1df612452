"""CPU oracle pinned against the reference's own tests (restated).

The reference (proj/tests/*.cpp) has no stored golden vectors; it pins the
matvec path with properties: loop-oracle mode products, dense-matrix
products, the adjoint identity, linearity, worker invariance, exact OpCounts,
bit-exact persistence.  The oracle must re-pass all of them before it counts
as "the reference".  Plus the committed golden fixtures (tests/golden/).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import rel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_scene(O, n, seg, d):
    g = O.make_centered_grid((0, 0, 0), 0.05, (n, n, n))
    return O.make_loop_scene(0.5, (0, d, 0), seg, g, 0, O.wavenumber_from_mhz(298.06), 3)


test_scene.__test__ = False


# ---------------------------------------------------------------- tensor --
def test_mode_product_identity_and_ones(oracle):
    """proj/tests/test_tensor.cpp:9-23."""
    O = oracle
    t = O.random_tensor((2, 3, 4), 11)
    assert rel(O.mode_product(t, np.eye(2), 1), t) == 0.0
    ones = np.ones((2, 2, 2), complex)
    out = O.mode_product(ones, np.ones((2, 2)), 1)
    assert np.all(out == 2.0)


def test_mode_product_vs_loops(oracle):
    """proj/tests/test_tensor.cpp:25-33 (< 1e-14)."""
    O = oracle
    t = O.random_tensor((4, 5, 6), 22)
    for mode in (1, 2, 3):
        m = O.random_matrix(7, t.shape[mode - 1], 30 + mode)
        assert rel(O.mode_product(t, m, mode), O.mode_product_loops(t, m, mode)) < 1e-14


def test_mode_product_errors_name_the_mode(oracle):
    """proj/tests/test_tensor.cpp:35-43."""
    O = oracle
    t = O.random_tensor((4, 5, 6), 3)
    m = O.random_matrix(7, 5, 4)
    with pytest.raises(O.ContractViolation, match="mode 1"):
        O.mode_product(t, m, 1)
    O.mode_product(t, m, 2)
    for bad in (0, 4):
        with pytest.raises(O.ContractViolation):
            O.mode_product(t, m, bad)


def test_mode_products_commute(oracle):
    """proj/tests/test_tensor.cpp:45-52."""
    O = oracle
    t = O.random_tensor((5, 6, 7), 5)
    a = O.random_matrix(4, 5, 6)
    b = O.random_matrix(3, 6, 7)
    ab = O.mode_product(O.mode_product(t, a, 1), b, 2)
    ba = O.mode_product(O.mode_product(t, b, 2), a, 1)
    assert rel(ab, ba) < 1e-12


def test_hosvd_rank1_and_error_contract(oracle):
    """proj/tests/test_tensor.cpp:54-88: rank-1 is exact; error <= eps; orthonormal factors."""
    O = oracle
    a, b, c = O.randn_c(6, 1), O.randn_c(7, 2), O.randn_c(8, 3)
    t = np.einsum("i,j,k->ijk", a, b, c)
    core, u1, u2, u3 = O.hosvd(t, 1e-8)
    assert core.shape == (1, 1, 1)
    assert rel(O.reconstruct(core, u1, u2, u3), t) < 1e-12
    rng = np.random.default_rng(0)
    for eps in (1e-2, 1e-4, 1e-6):
        t = sum(np.einsum("i,j,k->ijk", *(rng.standard_normal(n) + 1j * rng.standard_normal(n) for n in (9, 8, 7)))
                * 10.0 ** (-k) for k in range(6))
        core, u1, u2, u3 = O.hosvd(t, eps)
        assert rel(O.reconstruct(core, u1, u2, u3), t) <= eps
        for u in (u1, u2, u3):
            assert np.linalg.norm(u.conj().T @ u - np.eye(u.shape[1])) < 1e-12
    core, u1, u2, u3 = O.hosvd(np.zeros((3, 4, 5), complex), 1e-6)
    assert core.shape == (1, 1, 1) and core[0, 0, 0] == 0


# ---------------------------------------------------------------- kernels --
def test_efield_matches_finite_differences(oracle):
    """proj/tests/test_scene.cpp: curl curl (g w p) vs a central-difference Hessian."""
    O = oracle
    k0 = O.wavenumber_from_mhz(298.06)
    src = np.array([0.1, 0.2, -0.3, 0.0, 0.6, 0.8, 0.05])
    obs = np.array([0.4, -0.1, 0.2])

    def g(r):
        R = np.linalg.norm(r - src[:3])
        return np.exp(-1j * k0 * R) / (4 * np.pi * R)

    R = np.linalg.norm(obs - src[:3])
    h = 1e-4 * R
    hess = np.zeros((3, 3), complex)
    for a in range(3):
        ea = np.zeros(3)
        ea[a] = h
        hess[a, a] = (g(obs + ea) - 2 * g(obs) + g(obs - ea)) / h ** 2
        for b in range(a + 1, 3):
            eb = np.zeros(3)
            eb[b] = h
            hess[a, b] = hess[b, a] = (g(obs + ea + eb) - g(obs + ea - eb) - g(obs - ea + eb) + g(obs - ea - eb)) / (
                4 * h * h)
    p = src[3:6]
    fd = src[6] * (hess @ p - np.trace(hess) * p)
    assert rel(O.eval_kernel(0, k0, src, obs), fd) < 1e-5


def test_scene_guards(oracle):
    """Separation guard and q check (src/scene.cpp:43-74)."""
    O = oracle
    g = O.make_centered_grid((0, 0, 0), 0.05, (4, 4, 4))
    with pytest.raises(O.SceneError):
        O.make_loop_scene(0.05, (0, 0, 0), 8, g, 0, 1.0, 3)
    with pytest.raises(O.ContractViolation):
        O.validate_scene(O.Scene(g[0], g[1], g[2], np.array([[0, 1, 0, 1, 0, 0, 1.0]]), 0, 1.0, 5))


# ---------------------------------------------------------------- matvec --
def test_forward_basis_vector_bitwise(oracle):
    """proj/tests/test_matvec.cpp:38-48: forward(e_j) == decompressed column j, bitwise."""
    O = oracle
    cc = O.compress_matrix(test_scene(O, 6, 8, 0.8), 1e-6)
    st = O.OracleStore(cc)
    for j in range(cc.m):
        e = np.zeros((cc.m, 1), complex)
        e[j] = 1.0
        assert np.array_equal(st.forward(e)[:, 0], st.column(j))


def test_forward_adjoint_vs_dense(oracle):
    """proj/tests/test_matvec.cpp:50-58,77-85: within 5 eps of the dense matrix."""
    O = oracle
    eps = 1e-6
    sc = test_scene(O, 8, 10, 0.8)
    cc = O.compress_matrix(sc, eps)
    x = O.random_multivector(cc.m, 8, 31)
    assert rel(O.forward(cc, x), O.dense_forward(sc, x)) <= 5 * eps
    phi = O.random_multivector(cc.rows, 8, 77)
    assert rel(O.adjoint(cc, phi), O.dense_adjoint(sc, phi)) <= 5 * eps


def test_zero_block_adjoint_identity_linearity(oracle):
    """proj/tests/test_matvec.cpp:60-75,117-132."""
    O = oracle
    cc = O.compress_matrix(test_scene(O, 5, 6, 0.9), 1e-6)
    y = O.forward(cc, np.zeros((cc.m, 3), complex))
    assert y.shape == (cc.rows, 3) and np.linalg.norm(y) == 0.0
    cc = O.compress_matrix(test_scene(O, 6, 9, 0.8), 1e-6)
    x = O.random_multivector(cc.m, 4, 7)
    phi = O.random_multivector(cc.rows, 4, 8)
    lhs = np.trace(O.forward(cc, x).conj().T @ phi)
    rhs = np.trace(x.conj().T @ O.adjoint(cc, phi))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    cc = O.compress_matrix(test_scene(O, 6, 7, 0.9), 1e-8)
    x1, x2 = O.random_multivector(cc.m, 2, 1), O.random_multivector(cc.m, 2, 2)
    a, b = 0.7 - 0.3j, -1.1 + 0.2j
    assert rel(O.forward(cc, a * x1 + b * x2), a * O.forward(cc, x1) + b * O.forward(cc, x2)) <= 1e-12


def test_squared_norm_probe(oracle):
    """proj/tests/test_matvec.cpp:87-98."""
    O = oracle
    sc = test_scene(O, 6, 8, 0.8)
    cc = O.compress_matrix(sc, 1e-8)
    col = O.OracleStore(cc).column(3)
    y = O.adjoint(cc, col.reshape(-1, 1))
    sq = float(np.vdot(col, col).real)
    assert abs(y[3, 0] - sq) <= 1e-12 * sq
    assert rel(y, O.dense_adjoint(sc, col.reshape(-1, 1))) <= 5e-8


def test_shape_errors_and_workers(oracle):
    """proj/tests/test_matvec.cpp:134-148."""
    O = oracle
    cc = O.compress_matrix(test_scene(O, 4, 5, 0.9), 1e-6)
    with pytest.raises(O.ContractViolation, match="forward: x has 6 rows, expected m = 5"):
        O.forward(cc, np.zeros((cc.m + 1, 1), complex))
    with pytest.raises(O.ContractViolation):
        O.adjoint(cc, np.zeros((cc.rows - 1, 1), complex))
    cc = O.compress_matrix(test_scene(O, 6, 12, 0.8), 1e-8)
    x = O.random_multivector(cc.m, 3, 5)
    assert rel(O.forward(cc, x, 2), O.forward(cc, x, 1)) <= 1e-13


def test_opcount_formula(oracle):
    """proj/tests/test_matvec.cpp:170-220: madds = m q (n r^3 + n^2 r^2 + n^3 r)."""
    O = oracle
    n = 26
    ops = {}
    cc = O.synthetic_compression(n, 4, 2, 9)
    O.forward(cc, O.random_multivector(cc.m, 2, 3), 1, ops)
    base = 4 * 3 * (n * 8 + n * n * 4 + n * n * n * 2)
    assert ops["decompress_madds"] == base
    assert ops["accumulate_madds"] == 4 * 3 * n ** 3 * 2
    ops2 = {}
    O.forward(O.synthetic_compression(n, 8, 2, 9), O.random_multivector(8, 2, 3), 1, ops2)
    assert ops2["decompress_madds"] == 2 * base
    ops4 = {}
    O.forward(O.synthetic_compression(n, 4, 4, 9), O.random_multivector(4, 2, 3), 1, ops4)
    assert 1.6 < ops4["decompress_madds"] / base < 2.4


def test_rank1_aca_and_tucker_aca(oracle):
    """proj/tests/test_matvec.cpp:150-168 and test_aca.cpp:142-152."""
    O = oracle
    u = O.random_matrix(12, 1, 1)
    v = O.random_matrix(7, 1, 2)
    fac = O.DenseAca(u, v, 1e-3)
    x = O.random_multivector(7, 3, 3)
    assert rel(O.aca_forward(fac, x), u @ (v.conj().T @ x)) <= 1e-14
    phi = O.random_multivector(12, 3, 4)
    assert rel(O.aca_adjoint(fac, phi), v @ (u.conj().T @ phi)) <= 1e-14
    assert np.linalg.norm(O.aca_forward(fac, np.zeros((7, 2)))) == 0.0
    g = O.make_centered_grid((0, 0, 0), 0.04, (10, 10, 10))
    sc = O.make_loop_scene(0.5, (0, 1.2, 0), 16, g, 0, O.wavenumber_from_mhz(123.0), 3)
    row, col, m1, m2 = O.coupling_oracle(sc)
    z = O.assemble_full(sc)
    x = O.random_matrix(m2, 8, 5)
    for eps in (1e-3, 1e-5):
        fac = O.tucker_aca(row, col, m1, m2, sc.dims, 3, eps)
        assert rel(O.aca_forward(fac, x), z @ x) <= 10 * eps


def test_acceptance_criterion_2(oracle):
    """proj/tests/acceptance.cpp:87-112: 12^3, p = 8, <= 5e-8 vs dense, identity <= 1e-12."""
    O = oracle
    g = O.make_centered_grid((0, 0, 0), 0.04, (12, 12, 12))
    sc = O.make_loop_scene(0.5, (0, 0.7, 0), 20, g, 0, O.wavenumber_from_mhz(298.06), 3)
    cc = O.compress_matrix(sc, 1e-8, workers=2)
    x = O.random_multivector(cc.m, 8, 11)
    phi = O.random_multivector(cc.rows, 8, 12)
    y = O.forward(cc, x, 2)
    z = O.adjoint(cc, phi, 2)
    assert rel(y, O.dense_forward(sc, x)) <= 5e-8
    assert rel(z, O.dense_adjoint(sc, phi)) <= 5e-8
    lhs = np.trace(y.conj().T @ phi)
    rhs = np.trace(x.conj().T @ z)
    assert abs(lhs - rhs) / abs(lhs) <= 1e-12


# --------------------------------------------------------------------- io --
def test_ctc1_cta1_round_trip_bit_exact(oracle, tmp_path):
    """proj/tests/test_io.cpp:62-119."""
    O = oracle
    g = O.make_centered_grid((0, 0, 0), 0.05, (6, 5, 4))
    sc = O.make_loop_scene(0.5, (0, 0.8, 0), 5, g, 0, O.wavenumber_from_mhz(298.06), 3)
    cc = O.compress_matrix(sc, 1e-8)
    p = str(tmp_path / "rt.ctc1")
    O.save_ctc1(p, cc)
    back = O.load_ctc1(p)
    assert back.q == cc.q and back.m == cc.m and tuple(back.grid_dims) == tuple(cc.grid_dims)
    assert np.array_equal(back.ranks, cc.ranks) and np.array_equal(back.payload, cc.payload)
    assert back.k0 == cc.k0 and back.eps == cc.eps
    x = O.random_matrix(cc.m, 4, 3)
    assert np.array_equal(O.forward(back, x, 1), O.forward(cc, x, 1))
    row, col, m1, m2 = O.coupling_oracle(sc)
    fac = O.tucker_aca(row, col, m1, m2, sc.dims, 3, 1e-4)
    pa = str(tmp_path / "rt.cta1")
    O.save_cta1(pa, fac, sc.k0, sc.op)
    f2, k0, op = O.load_cta1(pa)
    assert k0 == sc.k0 and op == sc.op and f2.rank == fac.rank
    assert np.array_equal(f2.v, fac.v) and np.array_equal(f2.payload, fac.payload)


def test_malformed_files_raise_parse_errors(oracle, tmp_path):
    """proj/tests/test_io.cpp:121-205."""
    O = oracle
    with pytest.raises(O.ParseError):
        O.load_ctc1(str(tmp_path / "missing.ctc1"))
    bad = tmp_path / "bad.ctc1"
    bad.write_bytes(b"NOPE12345678")
    with pytest.raises(O.ParseError, match="bad magic"):
        O.load_ctc1(str(bad))
    data = open(os.path.join(GOLD, "loop8.ctc1"), "rb").read()
    trunc = tmp_path / "trunc.ctc1"
    trunc.write_bytes(data[:1000])
    with pytest.raises(O.ParseError) as ei:
        O.load_ctc1(str(trunc))
    assert ei.value.byte_offset > 45
    trail = tmp_path / "trail.ctc1"
    trail.write_bytes(data + b"\x00")
    with pytest.raises(O.ParseError, match="trailing"):
        O.load_ctc1(str(trail))


# ----------------------------------------------------------------- golden --
def test_golden_manifest_and_oracle_reproduction(oracle):
    """The committed fixtures are intact and the oracle reproduces them."""
    O = oracle
    man = json.load(open(os.path.join(GOLD, "MANIFEST.json")))
    for f, h in man.items():
        assert hashlib.sha256(open(os.path.join(GOLD, f), "rb").read()).hexdigest() == h, f
    ld = lambda f: np.load(os.path.join(GOLD, f))  # noqa: E731
    cc = O.load_ctc1(os.path.join(GOLD, "loop8.ctc1"))
    st = O.OracleStore(cc)
    assert rel(st.forward(ld("loop8_x.npy"), 1), ld("loop8_y.npy")) <= 1e-14
    assert rel(st.adjoint(ld("loop8_phi.npy"), 1), ld("loop8_z.npy")) <= 1e-14
    assert rel(ld("loop8_y.npy"), ld("loop8_ydense.npy")) <= 5e-6
    assert rel(ld("loop8_z.npy"), ld("loop8_zdense.npy")) <= 5e-6
    fac, _, _ = O.load_cta1(os.path.join(GOLD, "aca8.cta1"))
    assert rel(O.aca_forward(fac, ld("aca8_x.npy")), ld("aca8_y.npy")) <= 1e-14
    assert rel(O.aca_adjoint(fac, ld("aca8_phi.npy")), ld("aca8_z.npy")) <= 1e-14
    pw = O.load_ctc1(os.path.join(GOLD, "pwl.ctc1"))
    s64 = O.OracleStore(pw.rounded_c64())
    assert rel(s64.forward(ld("pwl_x.npy"), 1), ld("pwl_y64.npy")) <= 1e-14
    assert rel(s64.adjoint(ld("pwl_phi.npy"), 1), ld("pwl_z64.npy")) <= 1e-14
