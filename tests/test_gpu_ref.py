"""GPU path against the REFERENCE ITSELF (oracle/_ref: /root/reference/proj/src
compiled unchanged, see oracle/Makefile and tests/test_ref_pin_cpu.py).

Same inputs, same (c64-rounded) compressed factors on both sides; the
reference computes in complex128.  Tolerances (north_star): relative
Frobenius error <= 1e-12 for complex128 stores, <= 1e-5 for complex64.
Covers the reference's own loaders (CTC1 / CTA1 files written by the
reference's save_ctc1 / save_cta1), stores compressed by the reference's
compress_matrix and tucker_aca, ragged random stores, and OpCounts.
"""
import os

import numpy as np
import pytest

from conftest import ROOT, rel
from helpers import cn01, ragged_store

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")
TOL = {"c128": 1e-12, "c64": 1e-5}


@pytest.fixture(scope="module")
def R():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (build() compiles it where /root/reference exists)")
    ref.lib()
    return ref


def _r64(a, dtype):
    return a.astype(np.complex64).astype(np.complex128) if dtype == "c64" else a


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_reference_compressed_loop_scene(R, oracle, product, dtype, tmp_path):
    """compress_matrix of the reference (test_matvec.cpp:11-16 scene, and the
    acceptance criterion-2 scene of acceptance.cpp:87-112 at eps 1e-8),
    saved by the reference's save_ctc1, loaded by the native CTC1 ingest."""
    P, O = product, oracle
    k0 = O.wavenumber_from_mhz(298.06)
    for spacing, n, radius, center, seg, eps, p in [(0.05, 8, 0.5, (0, 0.8, 0), 10, 1e-6, 8),
                                                   (0.04, 12, 0.5, (0, 0.7, 0), 20, 1e-8, 8)]:
        sc = R.RefScene.loop(spacing, (n, n, n), radius, center, seg, 0, k0)
        cc = sc.compress(eps, workers=4)
        path = str(tmp_path / f"ref{n}.ctc1")
        cc.save_ctc1(path)
        ref = cc if dtype == "c128" else R.RefCC.from_compressed(O.load_ctc1(path).rounded_c64())
        ds = P.DeviceStore.load_ctc1(path, dtype)
        x = _r64(cn01(cc.m, p, 11), dtype)
        phi = _r64(cn01(cc.rows, p, 12), dtype)
        y, z = ds.forward(x), ds.adjoint(phi)
        assert rel(y, ref.forward(x, 4)) <= TOL[dtype]
        assert rel(z, ref.adjoint(phi, 4)) <= TOL[dtype]
        # adjoint identity on the GPU operator (test_matvec.cpp:68-75); a c64
        # inner product carries ~1e-6 |y| |phi| of absolute error
        lhs = np.vdot(y, phi)
        rhs = np.vdot(x, z)
        if dtype == "c128":
            assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
        else:
            assert abs(lhs - rhs) <= 1e-5 * np.linalg.norm(y) * np.linalg.norm(phi)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_reference_tucker_aca_store(R, oracle, product, dtype, tmp_path):
    """tucker_aca of the reference (test_aca.cpp:21-26 distant loop scene),
    saved by its save_cta1; GPU aca_forward / aca_adjoint vs the
    reference's (src/matvec.cpp:150-175)."""
    P, O = product, oracle
    sc = R.RefScene.loop(0.04, (10, 10, 10), 0.5, (0, 0.9, 0), 16, 0, O.wavenumber_from_mhz(123.0))
    path = str(tmp_path / "ref.cta1")
    fac = sc.tucker_aca(1e-5, 0.0, path)
    if dtype == "c64":
        f, k0, op = O.load_cta1(path)
        p64 = str(tmp_path / "ref64.cta1")
        O.save_cta1(p64, f.rounded_c64(), k0, op)
        fac = R.RefAca.load_cta1(p64)
    ds = P.DeviceStore.load_cta1(path, dtype)
    assert ds.ncols == fac.rank and ds.m2 == fac.cols
    x = _r64(cn01(fac.cols, 3, 5), dtype)
    phi = _r64(cn01(fac.rows, 3, 6), dtype)
    assert rel(ds.aca_forward(x), fac.aca_forward(x)) <= TOL[dtype]
    assert rel(ds.aca_adjoint(phi), fac.aca_adjoint(phi)) <= TOL[dtype]
    # batched row extraction vs the reference's row_of_compressed_u (src/aca.cpp:234-244)
    rows = [0, 7, fac.rows // 2, fac.rows - 1]
    got = ds.row_block(rows)
    for i, r in enumerate(rows):
        assert rel(got[i], fac.row_of_compressed_u(r)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("dims,q,m,rmin,rmax,p", [
    ((7, 5, 9), 3, 13, 1, 5, 2),
    ((33, 17, 130), 2, 9, 2, 12, 3),
    ((64, 64, 64), 12, 6, 4, 8, 1),
    ((1, 1, 1), 3, 4, 1, 1, 2),
    ((40, 36, 300), 12, 5, 3, 16, 4),
])
def test_ragged_stores_vs_reference(R, product, dtype, dims, q, m, rmin, rmax, p):
    P = product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=3 * sum(dims) + m)
    ref = R.RefCC.from_compressed(cc.rounded_c64() if dtype == "c64" else cc)
    ds = P.DeviceStore.from_compressed(cc, dtype)
    x = _r64(cn01(m, p, 21), dtype)
    phi = _r64(cn01(cc.rows, p, 22), dtype)
    ops_ref = [0, 0]
    assert rel(ds.forward(x), ref.forward(x, 4, ops_ref)) <= TOL[dtype]
    assert rel(ds.adjoint(phi), ref.adjoint(phi, 4)) <= TOL[dtype]
    # OpCounts (src/matvec.cpp:10-15,50-51): identical to the reference's
    ops = {}
    ds.forward(x, ops)
    assert [ops["decompress_madds"], ops["accumulate_madds"]] == ops_ref


def test_golden_files_through_reference_loader(R, product):
    """The committed fixtures read by the reference's own load_ctc1 /
    load_cta1 and by the native streaming ingest give the same operator."""
    P = product
    cc = R.RefCC.load_ctc1(os.path.join(GOLD, "pwl.ctc1"))
    x = np.load(os.path.join(GOLD, "pwl_x.npy"))
    phi = np.load(os.path.join(GOLD, "pwl_phi.npy"))
    ds = P.DeviceStore.load_ctc1(os.path.join(GOLD, "pwl.ctc1"), "c128")
    assert rel(ds.forward(x), cc.forward(x)) <= 1e-12
    assert rel(ds.adjoint(phi), cc.adjoint(phi)) <= 1e-12
    aca = R.RefAca.load_cta1(os.path.join(GOLD, "aca8.cta1"))
    da = P.DeviceStore.load_cta1(os.path.join(GOLD, "aca8.cta1"), "c128")
    xa = np.load(os.path.join(GOLD, "aca8_x.npy"))
    pa = np.load(os.path.join(GOLD, "aca8_phi.npy"))
    assert rel(da.aca_forward(xa), aca.aca_forward(xa)) <= 1e-12
    assert rel(da.aca_adjoint(pa), aca.aca_adjoint(pa)) <= 1e-12
