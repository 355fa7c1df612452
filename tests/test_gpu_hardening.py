"""C-ABI hardening on the GPU: device-side ordering of products on one store,
non-orthonormal factors on the fp16 tensor-core path, the dense-U ACA store,
and argument validation of the device entry points."""
import numpy as np
import pytest

from conftest import rel
from helpers import cn01, ragged_store

pytestmark = pytest.mark.gpu


def _c64(a):
    return a.astype(np.complex64).astype(np.complex128)


def test_products_on_two_streams_and_host_are_ordered(oracle, product):
    """TM_DEVICE on stream A, then TM_DEVICE on stream B, then TM_HOST, with
    no synchronisation in between: the three products share the store's
    work buffers and must still each match the oracle (the per-store
    completion event orders them on the device)."""
    import torch
    O, P = oracle, product
    cc = ragged_store((48, 40, 256), 12, 40, 6, 12, seed=99)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    xs = [_c64(cn01(cc.m, 2, 100 + i)) for i in range(3)]
    phis = [_c64(cn01(cc.rows, 2, 200 + i)) for i in range(3)]
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    xd = [torch.from_numpy(np.ascontiguousarray(x.T)).to(torch.complex64).cuda().t() for x in xs[:2]]
    pd = [torch.from_numpy(np.ascontiguousarray(p.T)).to(torch.complex64).cuda().t() for p in phis[:2]]
    torch.cuda.synchronize()
    ya = torch.empty((2, cc.rows), dtype=torch.complex64, device="cuda").t()
    yb = torch.empty((2, cc.rows), dtype=torch.complex64, device="cuda").t()
    za = torch.empty((2, cc.m), dtype=torch.complex64, device="cuda").t()
    zb = torch.empty((2, cc.m), dtype=torch.complex64, device="cuda").t()
    for _ in range(2):
        ds.forward_into(xd[0], ya, stream=sa.cuda_stream)
        ds.forward_into(xd[1], yb, stream=sb.cuda_stream)
        yh = ds.forward(xs[2])
        ds.adjoint_into(pd[0], za, stream=sa.cuda_stream)
        ds.adjoint_into(pd[1], zb, stream=sb.cuda_stream)
        zh = ds.adjoint(phis[2])
        torch.cuda.synchronize()
        for y, x in ((ya, xs[0]), (yb, xs[1])):
            assert rel(y.cpu().numpy(), ref.forward(x)) <= 1e-5
        assert rel(yh, ref.forward(xs[2])) <= 1e-5
        for z, p in ((za, phis[0]), (zb, phis[1])):
            assert rel(z.cpu().numpy(), ref.adjoint(p)) <= 1e-5
        assert rel(zh, ref.adjoint(phis[2])) <= 1e-5


def _rescaled(O, cc, s1, s2, s3):
    """The same operator with factors scaled by s_g and the core by 1/(s1 s2 s3)
    — valid for the reference (it checks ranks only, src/io.cpp:131-139) but
    not orthonormal."""
    tens = []
    for j in range(cc.m):
        for k in range(cc.q):
            core, u1, u2, u3 = cc.tensor(j, k)
            tens.append((core / (s1 * s2 * s3), u1 * s1, u2 * s2, u3 * s3))
    ranks, payload = O.pack_tensors(tens)
    return O.Compressed(cc.grid_dims, cc.q, cc.m, ranks.reshape(cc.m, cc.q, 3), payload)


@pytest.mark.parametrize("s1,s2,s3", [(1.0, 1.0, 1e3), (1.0, 1e-2, 1.0), (1e2, 1e-3, 1e-4), (7.0, 3e2, 0.05)])
def test_non_orthonormal_factors_on_tensor_cores(oracle, product, s1, s2, s3):
    O, P = oracle, product
    base = ragged_store((40, 36, 64), 3, 30, 2, 12, seed=5)
    cc = _rescaled(O, base, s1, s2, s3)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    for p in (1, 4):
        x = _c64(cn01(cc.m, p, 7))
        phi = _c64(cn01(cc.rows, p, 8))
        y, z = ds.forward(x), ds.adjoint(phi)
        assert np.all(np.isfinite(y)) and np.all(np.isfinite(z))
        assert rel(y, ref.forward(x)) <= 1e-5
        assert rel(z, ref.adjoint(phi)) <= 1e-5


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-12), ("c64", 1e-5)])
def test_dense_u_aca_store(product, dtype, tol):
    """aca_forward / aca_adjoint with a dense U (src/matvec.cpp:158,173) on the device."""
    P = product
    rng = np.random.default_rng(3)
    m1, m2, r = 3000, 211, 17
    u = rng.standard_normal((m1, r)) + 1j * rng.standard_normal((m1, r))
    v = rng.standard_normal((m2, r)) + 1j * rng.standard_normal((m2, r))
    if dtype == "c64":
        u, v = _c64(u), _c64(v)
    ds = P.DeviceStore.dense_aca(u, v, dtype)
    x = _c64(cn01(m2, 3, 1)) if dtype == "c64" else cn01(m2, 3, 1)
    phi = _c64(cn01(m1, 3, 2)) if dtype == "c64" else cn01(m1, 3, 2)
    assert rel(ds.aca_forward(x), u @ (v.conj().T @ x)) <= tol
    assert rel(ds.aca_adjoint(phi), v @ (u.conj().T @ phi)) <= tol
    with pytest.raises(P.ContractViolation, match="dense ACA U"):
        ds.forward(np.zeros((r, 1)))
    with pytest.raises(P.ContractViolation, match="aca_forward: x has"):
        ds.aca_forward(np.zeros((m2 + 1, 1)))


def test_device_out_validation(product):
    import torch
    P = product
    cc = ragged_store((8, 8, 16), 3, 5, 1, 4, seed=1)
    ds = P.DeviceStore.from_compressed(cc, "c64")
    x = torch.zeros((cc.m, 2), dtype=torch.complex64, device="cuda")
    good = torch.empty((2, cc.rows), dtype=torch.complex64, device="cuda").t()
    ds.forward_into(x, good)
    for bad in (torch.empty((cc.rows - 1, 2), dtype=torch.complex64, device="cuda"),
                torch.empty((2, cc.rows), dtype=torch.complex64, device="cuda"),       # row-major (stride(0) != 1)
                torch.empty((2, cc.rows), dtype=torch.complex128, device="cuda").t(),  # wrong dtype
                torch.empty((cc.rows, 2), dtype=torch.complex64)):                     # host tensor
        with pytest.raises(P.ContractViolation):
            ds.forward_into(x, bad)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_empty_store_and_empty_blocks(oracle, product, dtype):
    """A store with no columns (the reference's stacked_forward with
    ncols = 0 returns zeros, src/matvec.cpp:28-38), and p = 0 blocks."""
    O, P = oracle, product
    cc = O.Compressed((6, 5, 17), 3, 0, np.zeros((0, 3, 3), np.int32), np.zeros(0, np.complex128))
    ds = P.DeviceStore.from_compressed(cc, dtype)
    y = ds.forward(np.zeros((0, 2)))
    assert y.shape == (ds.rows, 2) and not np.any(y)
    z = ds.adjoint(np.ones((ds.rows, 2)))
    assert z.shape == (0, 2)
    full = ragged_store((6, 5, 17), 3, 4, 1, 4, seed=2)
    d2 = P.DeviceStore.from_compressed(full, dtype)
    assert d2.forward(np.zeros((4, 0))).shape == (d2.rows, 0)
    assert d2.adjoint(np.zeros((d2.rows, 0))).shape == (4, 0)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_many_columns(oracle, product, dtype):
    """70 000 columns (more than a 16-bit grid dimension, long K streams and
    many adjoint chunks) on a small grid: forward / adjoint vs the oracle."""
    O, P = oracle, product
    rng = np.random.default_rng(0)
    m, q, dims = 70000, 1, (4, 4, 16)
    ranks = rng.integers(1, 3, size=(m, q, 3)).astype(np.int32)
    from paper_2103_06393_b200.workloads import synthetic_payload
    pay, _ = synthetic_payload(dims, ranks, np.exp(-rng.random(m) * 3), 5, device="cpu")
    cc = O.Compressed(dims, q, m, ranks, pay.numpy())
    ds = P.DeviceStore.from_compressed(cc, dtype)
    ref = O.OracleStore(cc.rounded_c64() if dtype == "c64" else cc)
    x = cn01(m, 2, 1)
    phi = cn01(cc.rows, 2, 2)
    if dtype == "c64":
        x, phi = _c64(x), _c64(phi)
    tol = 1e-5 if dtype == "c64" else 1e-12
    assert rel(ds.forward(x), ref.forward(x, 8)) <= tol
    assert rel(ds.adjoint(phi), ref.adjoint(phi, 8)) <= tol
