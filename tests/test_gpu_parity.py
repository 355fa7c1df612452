"""GPU parity of the CUDA path against the CPU oracle (reference restatement).

Tolerances (north_star): relative Frobenius error <= 1e-12 for complex128
stores, <= 1e-5 for complex64 stores; the oracle always computes in complex128
on the same (rounded) factors and inputs.  The reference's own matvec tests
(proj/tests/test_matvec.cpp) are restated here against the GPU operator.
"""
import numpy as np
import pytest

from conftest import rel
from helpers import cn01, ragged_store

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}


def _loop_scene(O, n, seg, d, h=0.05):
    g = O.make_centered_grid((0, 0, 0), h, (n, n, n) if np.isscalar(n) else n)
    return O.make_loop_scene(0.5, (0, d, 0), seg, g, 0, O.wavenumber_from_mhz(298.06), 3)


def _pair(O, P, cc, dtype):
    ref = cc.rounded_c64() if dtype == "c64" else cc
    return O.OracleStore(ref), P.DeviceStore.from_compressed(cc, dtype), ref


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("p", [1, 3, 8])
def test_forward_adjoint_physics_scene(oracle, product, dtype, p):
    O, P = oracle, product
    cc = O.compress_matrix(_loop_scene(O, 8, 10, 0.8), 1e-6)
    os_, ds, _ = _pair(O, P, cc, dtype)
    x = cn01(cc.m, p, 31)
    phi = cn01(cc.rows, p, 77)
    if dtype == "c64":
        x = x.astype(np.complex64).astype(np.complex128)
        phi = phi.astype(np.complex64).astype(np.complex128)
    assert rel(ds.forward(x), os_.forward(x)) <= TOL[dtype]
    assert rel(ds.adjoint(phi), os_.adjoint(phi)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("dims,q,m,rmin,rmax", [
    ((7, 5, 9), 3, 13, 1, 5),          # ragged, tiny, non-multiples of every tile
    ((24, 24, 24), 3, 40, 6, 11),      # config-1 shape
    ((33, 17, 130), 2, 9, 2, 12),      # n3 > 128 (two i3 tiles), odd n1/n2
    ((64, 64, 64), 12, 6, 4, 8),       # config-5 shape (q = 12)
    ((1, 1, 1), 3, 4, 1, 1),           # single voxel
    ((12, 40, 3), 1, 17, 1, 20),       # tall ranks clipped to the grid, q = 1
])
def test_ragged_stores(oracle, product, dtype, dims, q, m, rmin, rmax):
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=sum(dims) + m)
    os_, ds, _ = _pair(O, P, cc, dtype)
    for p in (1, 2):
        x = cn01(m, p, 5 + p)
        phi = cn01(cc.rows, p, 9 + p)
        if dtype == "c64":
            x = x.astype(np.complex64).astype(np.complex128)
            phi = phi.astype(np.complex64).astype(np.complex128)
        assert rel(ds.forward(x), os_.forward(x)) <= TOL[dtype]
        assert rel(ds.adjoint(phi), os_.adjoint(phi)) <= TOL[dtype]


def test_basis_vector_extracts_column(oracle, product):
    """forward(e_j) == decompressed column j (test_matvec.cpp:38-48)."""
    O, P = oracle, product
    cc = O.compress_matrix(_loop_scene(O, 6, 8, 0.8), 1e-6)
    os_ = O.OracleStore(cc)
    ds = P.DeviceStore.from_compressed(cc, "c128")
    for j in range(cc.m):
        e = np.zeros((cc.m, 1), complex)
        e[j] = 1.0
        assert rel(ds.forward(e)[:, 0], os_.column(j)) <= 1e-14


def test_zero_block_is_exactly_zero(oracle, product):
    """test_matvec.cpp:60-66."""
    O, P = oracle, product
    cc = O.compress_matrix(_loop_scene(O, 5, 6, 0.9), 1e-6)
    for dtype in ("c128", "c64"):
        ds = P.DeviceStore.from_compressed(cc, dtype)
        y = ds.forward(np.zeros((cc.m, 3), complex))
        assert y.shape == (cc.rows, 3)
        assert np.count_nonzero(y) == 0
        z = ds.adjoint(np.zeros((cc.rows, 2), complex))
        assert np.count_nonzero(z) == 0


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_adjoint_identity(oracle, product, dtype):
    """<F x, phi> = <x, F^H phi> (test_matvec.cpp:68-75); 1e-12 at c128."""
    O, P = oracle, product
    cc = O.compress_matrix(_loop_scene(O, 6, 9, 0.8), 1e-6)
    ds = P.DeviceStore.from_compressed(cc, dtype)
    x = O.random_multivector(cc.m, 4, 7)
    phi = O.random_multivector(cc.rows, 4, 8)
    lhs = np.trace(ds.forward(x).conj().T @ phi)
    rhs = np.trace(x.conj().T @ ds.adjoint(phi))
    assert abs(lhs - rhs) <= (1e-12 if dtype == "c128" else 1e-5) * abs(lhs)


def test_dense_oracle_and_squared_norm(oracle, product):
    """Forward/adjoint vs the dense matrix within 5 eps (test_matvec.cpp:50-58,77-98)."""
    O, P = oracle, product
    eps = 1e-6
    sc = _loop_scene(O, 8, 10, 0.8)
    cc = O.compress_matrix(sc, eps)
    ds = P.DeviceStore.from_compressed(cc, "c128")
    x = O.random_multivector(cc.m, 8, 31)
    assert rel(ds.forward(x), O.dense_forward(sc, x)) <= 5 * eps
    phi = O.random_multivector(cc.rows, 8, 77)
    assert rel(ds.adjoint(phi), O.dense_adjoint(sc, phi)) <= 5 * eps
    cc8 = O.compress_matrix(_loop_scene(O, 6, 8, 0.8), 1e-8)
    ds8 = P.DeviceStore.from_compressed(cc8, "c128")
    col = O.OracleStore(cc8).column(3)
    y = ds8.adjoint(col.reshape(-1, 1))
    sq = float(np.vdot(col, col).real)
    assert abs(y[3, 0] - sq) <= 1e-12 * sq


def test_linearity(oracle, product):
    """test_matvec.cpp:117-132."""
    O, P = oracle, product
    cc = O.compress_matrix(_loop_scene(O, 6, 7, 0.9), 1e-8)
    ds = P.DeviceStore.from_compressed(cc, "c128")
    x1 = O.random_multivector(cc.m, 2, 1)
    x2 = O.random_multivector(cc.m, 2, 2)
    a, b = 0.7 - 0.3j, -1.1 + 0.2j
    lhs = ds.forward(a * x1 + b * x2)
    rhs = a * ds.forward(x1) + b * ds.forward(x2)
    assert rel(lhs, rhs) <= 1e-12


def test_shape_errors(oracle, product):
    """ContractViolation on row-count mismatch (test_matvec.cpp:134-140)."""
    O, P = oracle, product
    cc = O.compress_matrix(_loop_scene(O, 4, 5, 0.9), 1e-6)
    ds = P.DeviceStore.from_compressed(cc, "c128")
    with pytest.raises(P.ContractViolation, match="forward: x has 6 rows, expected m = 5"):
        ds.forward(np.zeros((cc.m + 1, 1), complex))
    with pytest.raises(P.ContractViolation, match="adjoint: phi has"):
        ds.adjoint(np.zeros((cc.rows - 1, 1), complex))


def test_determinism(oracle, product):
    """Fixed column-to-CTA assignment and ordered reductions: bitwise repeatable."""
    O, P = oracle, product
    cc = ragged_store((24, 20, 40), 3, 30, 3, 9, seed=3)
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = cn01(cc.m, 2, 1)
    phi = cn01(cc.rows, 2, 2)
    y1, y2 = ds.forward(x), ds.forward(x)
    z1, z2 = ds.adjoint(phi), ds.adjoint(phi)
    assert np.array_equal(y1, y2) and np.array_equal(z1, z2)


def test_opcounts(oracle, product):
    """Exact OpCounts formula (test_matvec.cpp:170-220)."""
    O, P = oracle, product
    n = 26
    cc = O.synthetic_compression(n, 4, 2, 9)
    ds = P.DeviceStore.from_compressed(cc, "c128")
    ops = P.OpCounts()
    ds.forward(O.random_multivector(cc.m, 2, 3), ops)
    assert ops.decompress_madds == 4 * 3 * (n * 8 + n * n * 4 + n * n * n * 2)
    assert ops.accumulate_madds == 4 * 3 * n * n * n * 2
    assert ds.opcounts(2) == O.OracleStore(cc).opcounts(2)
    ds.forward(O.random_multivector(cc.m, 2, 3), ops)   # counts accumulate (+=)
    assert ops.decompress_madds == 2 * 4 * 3 * (n * 8 + n * n * 4 + n * n * n * 2)


def test_device_tensors_match_host(oracle, product):
    """TM_DEVICE path (torch CUDA tensors on the current stream) == TM_HOST path."""
    import torch
    O, P = oracle, product
    cc = ragged_store((16, 12, 20), 3, 11, 2, 6, seed=11)
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = cn01(cc.m, 3, 4).astype(np.complex64)
    phi = cn01(cc.rows, 3, 5).astype(np.complex64)
    yh = ds.forward(x)
    zh = ds.adjoint(phi)
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    pd = torch.from_numpy(np.ascontiguousarray(phi.T)).cuda().t()
    yd = ds.forward(xd)
    zd = ds.adjoint(pd)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), yh)
    assert np.array_equal(zd.cpu().numpy(), zh)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_aca_products(oracle, product, dtype):
    """aca_forward / aca_adjoint vs the oracle on a Tucker-ACA store (matvec.cpp:150-175)."""
    O, P = oracle, product
    g = O.make_centered_grid((0, 0, 0), 0.04, (8, 8, 8))
    sc = O.make_loop_scene(0.5, (0, 0.9, 0), 12, g, 0, O.wavenumber_from_mhz(123.0), 3)
    row, col, m1, m2 = O.coupling_oracle(sc)
    fac = O.tucker_aca(row, col, m1, m2, sc.dims, 3, 1e-4)
    assert fac.rank >= 2
    ref = fac.rounded_c64() if dtype == "c64" else fac
    ds = P.DeviceStore.from_compressed(fac, dtype)
    x = cn01(m2, 4, 17)
    phi = cn01(m1, 4, 18)
    if dtype == "c64":
        x = x.astype(np.complex64).astype(np.complex128)
        phi = phi.astype(np.complex64).astype(np.complex128)
    assert rel(ds.aca_forward(x), O.aca_forward(ref, x)) <= TOL[dtype]
    assert rel(ds.aca_adjoint(phi), O.aca_adjoint(ref, phi)) <= TOL[dtype]
    # and the operator stays within a decade of the ACA tolerance (test_aca.cpp:134-139)
    z = O.assemble_full(sc)
    assert rel(ds.aca_forward(x), z @ x) <= 10 * 1e-4


@pytest.mark.parametrize("dims,q,m,rmin,rmax,p", [
    ((16, 16, 16), 3, 9, 2, 6, 1),       # smallest tensor-core shape
    ((24, 40, 40), 2, 21, 3, 16, 2),     # ranks up to the tensor-core limit, partial row tiles
    ((64, 64, 64), 12, 7, 4, 9, 1),      # config-5 grid
    ((20, 18, 300), 1, 5, 2, 8, 1),      # n3 > 256: three i3 blocks, partial N
    ((192, 224, 256), 1, 3, 5, 12, 1),   # config-4 grid, a few columns
    ((9, 70, 20), 2, 40, 1, 13, 3),      # many short chains, ragged ranks from 1
])
def test_tensor_core_forward(oracle, product, monkeypatch, dims, q, m, rmin, rmax, p):
    """tcgen05 fp16-split forward and adjoint (c64, the default c64 path) vs the
    oracle and vs the CUDA-core kernels (TMB_DISABLE_TC=1)."""
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=7 * m + q)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = cn01(m, p, 3).astype(np.complex64).astype(np.complex128)
    phi = cn01(cc.rows, p, 4).astype(np.complex64).astype(np.complex128)
    y_tc, z_tc = ds.forward(x), ds.adjoint(phi)
    monkeypatch.setenv("TMB_DISABLE_TC", "1")
    y_cc, z_cc = ds.forward(x), ds.adjoint(phi)
    monkeypatch.delenv("TMB_DISABLE_TC")
    y_ref, z_ref = ref.forward(x), ref.adjoint(phi)
    assert rel(y_tc, y_ref) <= 1e-5
    assert rel(y_cc, y_ref) <= 1e-5
    assert rel(z_tc, z_ref) <= 1e-5
    assert rel(z_cc, z_ref) <= 1e-5


@pytest.mark.parametrize("dims,q,m,rmin,rmax,p", [
    ((24, 18, 300), 2, 11, 2, 12, 1),    # forward pairs over a partial second i3 tile, nrt = 6
    ((16, 40, 200), 1, 17, 1, 16, 2),    # nt1 = 4 (two i1 pairs), partial i2 tiles, two RHS
    ((8, 64, 130), 3, 6, 3, 9, 1),       # nt1 = 2: one pair; adjoint nrt = 4
])
def test_cta_pair_kernels(oracle, product, monkeypatch, dims, q, m, rmin, rmax, p):
    """The CTA-pair (cta_group::2) forward and adjoint against the oracle and
    against the single-CTA kernels (TMB_DISABLE_PAIR=1) on shapes that take
    the pair path (even i1-block / row-tile counts, 256-voxel i3 tiles)."""
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=11 * m + q)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = cn01(m, p, 5).astype(np.complex64).astype(np.complex128)
    phi = cn01(cc.rows, p, 6).astype(np.complex64).astype(np.complex128)
    y2, z2 = ds.forward(x), ds.adjoint(phi)
    monkeypatch.setenv("TMB_DISABLE_PAIR", "1")
    y1, z1 = ds.forward(x), ds.adjoint(phi)
    monkeypatch.delenv("TMB_DISABLE_PAIR")
    y_ref, z_ref = ref.forward(x), ref.adjoint(phi)
    for got in (y1, y2):
        assert rel(got, y_ref) <= 1e-5
    for got in (z1, z2):
        assert rel(got, z_ref) <= 1e-5
    assert rel(y2, y1) <= 1e-6 and rel(z2, z1) <= 1e-6


def test_forward_rhs_passes(oracle, product, monkeypatch):
    """The x-in-B forward over several right-hand-side passes (a B-operand
    budget smaller than one pass of all p), host and device I/O, against
    the oracle and against the single-pass result."""
    O, P = oracle, product
    cc = ragged_store((20, 36, 140), 2, 13, 2, 11, seed=29)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = cn01(cc.m, 7, 31).astype(np.complex64).astype(np.complex128)
    y1 = ds.forward(x)
    monkeypatch.setenv("TMB_XB_CAP_MB", "1")  # ~1 MB: one right-hand side per pass here
    y2 = ds.forward(x)
    monkeypatch.delenv("TMB_XB_CAP_MB")
    y_ref = ref.forward(x)
    assert rel(y1, y_ref) <= 1e-5
    assert rel(y2, y_ref) <= 1e-5
    assert rel(y2, y1) <= 1e-6


@pytest.mark.parametrize("dims,q,m,rmin,rmax,p", [
    ((24, 40, 40), 2, 21, 3, 16, 5),      # a quad + an odd one (pairs: two + odd)
    ((64, 64, 64), 12, 6, 4, 9, 8),       # config-5 grid, two quads
    ((9, 70, 20), 1, 70, 1, 13, 2),       # many columns: 64-slot chunks with many short columns
    ((16, 12, 48), 3, 17, 20, 32, 7),     # r3 up to 32 = a full 32-slot chunk; quad + pair + odd
    ((8, 8, 64), 2, 9, 33, 40, 6),        # r3 > 32: no quads, three pairs
])
def test_adjoint_rhs_pairs(oracle, product, monkeypatch, dims, q, m, rmin, rmax, p):
    """The multi-right-hand-side adjoint (adj_tc2_kernel<NR>: W once per
    column for a quad / pair, 32- / 64-slot chunks) against the oracle and against the single-RHS kernel."""
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=13 * m + p)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    phi = cn01(cc.rows, p, 41).astype(np.complex64).astype(np.complex128)
    z4 = ds.adjoint(phi)
    monkeypatch.setenv("TMB_ADJ_NR", "2")
    z2 = ds.adjoint(phi)
    monkeypatch.setenv("TMB_ADJ_NR", "1")
    z1 = ds.adjoint(phi)
    monkeypatch.delenv("TMB_ADJ_NR")
    z_ref = ref.adjoint(phi)
    assert rel(z4, z_ref) <= 1e-5
    assert rel(z2, z_ref) <= 1e-5
    assert rel(z1, z_ref) <= 1e-5
    for z in (z4, z2):
        assert rel(z, z1) <= 1e-6


@pytest.mark.parametrize("chain", ["", "1", "3", "48"])
def test_tensor_core_long_k(product, monkeypatch, chain):
    """Accumulation over a long K stream (2 500 columns, K ~ 21 000 per
    component): the chained TMEM accumulation must stay within 1e-5 of the
    complex128 GPU forward on the same rounded factors (the c128 kernels are
    pinned to the oracle at 1e-12 above).  An unchained accumulator drifts
    to ~3e-4 here."""
    import torch
    from paper_2103_06393_b200.workloads import Config, rank_table, synthetic_payload
    P = product
    cfg = Config("longk", (32, 32, 128), 2, 2500, "c64", 1, (3.0, 50.0))
    ranks = rank_table(cfg, 5)
    pay, _ = synthetic_payload(cfg.grid, ranks, np.ones(cfg.m), 9, device="cuda")
    p64 = pay.to(torch.complex64).to(torch.complex128)
    s64 = P.DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, "c64", 0)
    s128 = P.DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, p64, "c128", 0)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    x = torch.randn((1, cfg.m), dtype=torch.complex64, device="cuda", generator=g).t()
    if chain:
        monkeypatch.setenv("TMB_TC_CHAIN", chain)
    y64 = s64.forward(x).to(torch.complex128)
    y128 = s128.forward(x.to(torch.complex128))
    err = float(torch.linalg.vector_norm(y64 - y128) / torch.linalg.vector_norm(y128))
    assert err <= 1e-5, err
    phi = torch.randn((1, y128.shape[0]), dtype=torch.complex64, device="cuda", generator=g).t()
    z64 = s64.adjoint(phi).to(torch.complex128)
    z128 = s128.adjoint(phi.to(torch.complex128))
    err = float(torch.linalg.vector_norm(z64 - z128) / torch.linalg.vector_norm(z128))
    assert err <= 1e-5, err


@pytest.mark.parametrize("dims,q,m,rmin,rmax,p", [
    ((16, 16, 16), 3, 9, 2, 6, 3),        # smallest batched shape, partial i2/i3 tiles
    ((21, 40, 37), 2, 19, 1, 13, 8),      # ragged ranks from 1, n2 and n3 not multiples of the tile
    ((64, 64, 64), 12, 6, 4, 9, 32),      # config-5 grid, a full 32-RHS block
    ((9, 20, 70), 1, 11, 3, 16, 40),      # rank-16 factors, two RHS blocks (32 + 8)
])
def test_batched_forward(oracle, product, monkeypatch, dims, q, m, rmin, rmax, p):
    """Batched multi-RHS forward (one pass: W shared by all p right-hand
    sides in the N space) vs the oracle and vs one-RHS passes (the B-operand
    budget TMB_XB_CAP_MB=1 forces a pass per right-hand side)."""
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=11 * m + p)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = cn01(m, p, 21).astype(np.complex64).astype(np.complex128)
    y_b = ds.forward(x)
    monkeypatch.setenv("TMB_XB_CAP_MB", "1")
    y_s = ds.forward(x)
    monkeypatch.delenv("TMB_XB_CAP_MB")
    y_ref = ref.forward(x)
    assert rel(y_b, y_ref) <= 1e-5
    assert rel(y_s, y_ref) <= 1e-5
    # linearity across the RHS block: column c of the batched product is the
    # single-RHS product of column c
    y1 = ds.forward(x[:, p - 1:p])
    assert rel(y_b[:, p - 1:p], y1) <= 1e-5


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_rows_and_element(oracle, product, dtype):
    """Batched element() / row_of_compressed_u: rows of the
    stored operator vs the oracle's element() and vs columns of the forward."""
    O, P = oracle, product
    cc = ragged_store((13, 11, 20), 3, 9, 1, 7, seed=5)
    ref = O.OracleStore(cc.rounded_c64() if dtype == "c64" else cc)
    ds = P.DeviceStore.from_compressed(cc, dtype)
    n1, n2, n3 = cc.grid_dims
    nv = n1 * n2 * n3
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 3 * nv, size=17)
    got = ds.row_block(rows)
    want = np.zeros_like(got, dtype=np.complex128)
    for r, g in enumerate(rows):
        k, v = divmod(int(g), nv)
        i1, i2, i3 = v % n1, (v // n1) % n2, v // (n1 * n2)
        for j in range(cc.m):
            want[r, j] = ref.element(j, k, i1, i2, i3)
    tol = TOL[dtype]
    assert rel(got, want) <= tol
    # the same rows of Z from the product with basis vectors (test_matvec.cpp:38-48)
    y = ds.forward(np.eye(cc.m))
    assert rel(got, y[rows, :]) <= tol
    assert abs(ds.element(4, 2, 1, 2, 3) - ref.element(4, 2, 1, 2, 3)) <= 10 * tol * np.abs(want).max()
    with pytest.raises(P.ContractViolation, match="index out of range"):
        ds.row_block([3 * nv])
    with pytest.raises(P.ContractViolation, match="index out of range"):
        ds.element(0, 0, n1, 0, 0)


def test_row_of_compressed_u_aca(oracle, product):
    """row_of_compressed_u on an ACA store (src/aca.cpp:234-244)."""
    O, P = oracle, product
    import os
    GOLD = os.path.join(os.path.dirname(__file__), "golden")
    ds = P.DeviceStore.load_cta1(os.path.join(GOLD, "aca8.cta1"), "c128")
    fac = O.load_cta1(os.path.join(GOLD, "aca8.cta1"))[0]
    i = 5 + ds.num_voxels  # component 1
    got = ds.row_block([i])[0]
    st = O.OracleStore(fac)
    n1, n2, _ = ds.dims
    v = i - ds.num_voxels
    want = np.array([st.element(l, 1, v % n1, (v // n1) % n2, v // (n1 * n2)) for l in range(ds.ncols)])
    assert rel(got, want) <= 1e-12


@pytest.mark.parametrize("q,eps", [(3, 1e-6), (12, 1e-4), (3, 1e-8), (12, 1e-9)])
def test_gpu_compressor(oracle, product, tmp_path, q, eps):
    """GPU column assembly + HOSVD vs the restated reference
    compressor: identical per-tensor ranks, columns identical to the oracle's
    assemble_column, and the operator within the reference's 5*eps of the
    dense matrix (proj/tests/test_matvec.cpp:50-58); CTC1 round trip."""
    import torch
    O, P = oracle, product
    from paper_2103_06393_b200 import compress as C
    g = O.make_centered_grid((0, 0, 0), 0.05, (8, 9, 10))
    sc = O.make_loop_scene(0.5, (0, 0.8, 0), 10, g, 0, O.wavenumber_from_mhz(298.06), q)
    # assembly vs the oracle, column by column
    cols = C.assemble_columns(sc, range(sc.num_sources)).cpu().numpy().reshape(sc.num_sources, -1)
    for j in (0, 3, 9):
        assert rel(cols[j], O.assemble_column(sc, j)) <= 1e-13
    ranks, payload = C.compress_scene(sc, eps)
    cc = O.compress_matrix(sc, eps)
    assert np.array_equal(ranks, np.asarray(cc.ranks).reshape(ranks.shape))
    ds = P.DeviceStore.from_arrays(sc.dims, q, ranks, payload, "c128", 0)
    z = O.assemble_full(sc)
    x = cn01(sc.num_sources, 4, 31)
    phi = cn01(sc.rows, 4, 77)
    assert rel(ds.forward(x), z @ x) <= 5 * eps
    assert rel(ds.adjoint(phi), z.conj().T @ phi) <= 5 * eps
    # the same operator as the oracle's compressed store (the compressions
    # differ only by singular-vector phases and rounding)
    assert rel(ds.forward(x), O.OracleStore(cc).forward(x)) <= 5 * eps
    path = tmp_path / "gpu.ctc1"
    C.write_ctc1(path, sc.dims, q, ranks, payload, sc.k0, eps, sc.op)
    back = O.load_ctc1(str(path))
    assert np.array_equal(np.asarray(back.ranks).reshape(ranks.shape), ranks)
    assert rel(back.payload, payload.cpu().numpy()) == 0.0
    ld = P.DeviceStore.load_ctc1(str(path), "c128")
    assert rel(ld.forward(x), ds.forward(x)) == 0.0


@pytest.mark.parametrize("q", [3, 12])
def test_gpu_tucker_aca(oracle, product, q):
    """GPU Tucker-ACA (Algorithm 3) vs the restated reference
    tucker_aca (src/aca.cpp:126-232): same rank, pivots and convergence, the
    product within 10*eps of the dense matrix (test_aca.cpp:142-152) and
    within eps of the oracle's factors."""
    import torch
    O, P = oracle, product
    from paper_2103_06393_b200 import aca as A
    g = O.make_centered_grid((0, 0, 0), 0.04, (8, 8, 8))
    sc = O.make_loop_scene(0.5, (0, 0.9, 0), 12, g, 0, O.wavenumber_from_mhz(123.0), q)
    eps = 1e-4
    row, col, m1, m2 = O.coupling_oracle(sc)
    ref = O.tucker_aca(row, col, m1, m2, sc.dims, q, eps)
    fac = A.tucker_aca(sc, eps)
    assert fac.rank == ref.rank and fac.converged == ref.converged
    assert np.array_equal(fac.ranks, np.asarray(ref.ranks).reshape(fac.ranks.shape))
    assert rel(fac.v.cpu().numpy(), ref.v) <= 1e-6  # greedy ACA amplifies 1e-13 residual differences in late rows
    ds = fac.store("c128")
    x = cn01(m2, 3, 17)
    z = O.assemble_full(sc)
    y = ds.aca_forward(x)
    assert rel(y, z @ x) <= 10 * eps
    assert rel(y, O.aca_forward(ref, x)) <= eps
    phi = cn01(m1, 2, 18)
    assert rel(ds.aca_adjoint(phi), z.conj().T @ phi) <= 10 * eps


def test_device_inputs_with_lazy_conjugation(oracle, product):
    """torch conj() / neg() views (lazy bits over unconjugated memory) must
    be materialised before the device pointer reaches the C ABI."""
    import torch
    O, P = oracle, product
    cc = ragged_store((6, 7, 8), 2, 5, 1, 4, seed=3)
    ds = P.DeviceStore.from_compressed(cc, "c128")
    x = torch.from_numpy(cn01(cc.m, 2, 1)).cuda()
    xc = x.conj()
    assert xc.is_conj()
    h = lambda t: t.cpu().numpy()
    want = h(ds.forward(x.conj().resolve_conj()))
    assert rel(h(ds.forward(xc)), want) <= 1e-15
    assert rel(h(ds.forward(-x)), -h(ds.forward(x))) <= 1e-15
    phi = torch.from_numpy(cn01(cc.rows, 1, 2)).cuda()
    assert rel(h(ds.adjoint(phi.conj())), h(ds.adjoint(phi.conj().resolve_conj()))) <= 1e-15


@pytest.mark.parametrize("dims,q,m,hi,p", [
    ((48, 40, 96), 3, 12, (20, 20, 20), 1),     # one rank-20 tensor among ranks <= 12
    ((40, 36, 140), 2, 9, (24, 18, 24), 3),     # r2 != r3, two i3 halves
    ((36, 33, 64), 3, 7, (8, 12, 32), 2),        # r3 = 32: a column spans three 16-K stages
    ((64, 64, 64), 12, 6, (16, 17, 17), 5),     # just past the old rank-16 bound, quads + single adjoint
])
@pytest.mark.parametrize("warena", ["on", "off"])
def test_ranks_above_16_stay_on_tensor_cores(oracle, product, dims, q, m, hi, p, warena, monkeypatch):
    """Ranks up to 32 run on tcgen05 (the reference accepts any 1 <= r <= n,
    src/io.cpp:131-139): one or more high-rank tensors in a ragged store."""
    O, P = oracle, product
    base = ragged_store(dims, q, m, 2, 12, seed=sum(dims) + p)
    rng = np.random.default_rng(7)
    tens = [base.tensor(j, k) for j in range(m) for k in range(q)]
    for t in (1, (m * q) // 2, m * q - 1):  # replace three tensors by high-rank ones
        rk = [min(hi[g], dims[g]) for g in range(3)]
        core = rng.standard_normal(rk) + 1j * rng.standard_normal(rk)
        us = [np.linalg.qr(rng.standard_normal((dims[g], rk[g])) + 1j * rng.standard_normal((dims[g], rk[g])))[0]
              for g in range(3)]
        tens[t] = (np.asfortranarray(core), *[np.asfortranarray(u) for u in us])
    ranks, payload = O.pack_tensors(tens)
    cc = O.Compressed(dims, q, m, ranks.reshape(m, q, 3), payload)
    ds = P.DeviceStore.from_compressed(cc, "c64")
    kp = ds.kernel_paths()
    assert kp["forward"] == "tcgen05+warena" and kp["adjoint"] in ("tcgen05", "tcgen05+gemm")
    if warena == "off":  # the producer-warp forward (the BIG instantiation for r3 > 16)
        monkeypatch.setenv("TMB_WARENA", "0")
        assert ds.kernel_paths() == {"forward": "tcgen05", "adjoint": "tcgen05"}
    ref = O.OracleStore(cc.rounded_c64())
    x = cn01(m, p, 3).astype(np.complex64).astype(np.complex128)
    phi = cn01(cc.rows, p, 4).astype(np.complex64).astype(np.complex128)
    assert rel(ds.forward(x), ref.forward(x)) <= 1e-5
    assert rel(ds.adjoint(phi), ref.adjoint(phi)) <= 1e-5
