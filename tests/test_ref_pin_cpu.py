"""Pins the CPU oracle to the REFERENCE ITSELF (oracle/_ref, test infrastructure).

oracle/_ref/libtuckmat_ref.so is /root/reference/proj/src/*.cpp compiled
unchanged (Eigen replaced by oracle/eigen_shim, doctest by
oracle/doctest_shim; oracle/Makefile target `ref`).  These tests check:

* the reference's own unit suites (proj/tests/test_{tensor,matvec,io,aca,
  compress,scene}.cpp, unchanged) pass on that build — which pins the shim;
* the reference's load_ctc1 / load_cta1 read the committed golden fixtures,
  and its forward / adjoint / aca_forward / aca_adjoint reproduce the golden
  outputs and the CPU restatement (oracle/) on them and on ragged stores;
* the reference's compress_matrix and tucker_aca choose the same ranks,
  pivots and cross rank as the restated producers in oracle/oracle.py.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import rel  # noqa: E402
from oracle import ref as R  # noqa: E402

if not R.available():
    R.build()
pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")

SUITES = ["test_tensor", "test_matvec", "test_io", "test_aca", "test_compress", "test_scene"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_passes_on_ref_build(suite, tmp_path):
    exe = os.path.join(ROOT, "oracle", "_ref", suite)
    if not os.path.exists(exe):
        pytest.skip(f"{suite} not built")
    r = subprocess.run([exe], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def _gold(name):
    return np.load(os.path.join(GOLD, name))


def test_ref_loads_goldens_and_reproduces_oracle_outputs(oracle):
    cc = R.RefCC.load_ctc1(os.path.join(GOLD, "loop8.ctc1"))
    x, phi = _gold("loop8_x.npy"), _gold("loop8_phi.npy")
    ops = [0, 0]
    y = cc.forward(x, 1, ops)
    z = cc.adjoint(phi, 1)
    assert rel(y, _gold("loop8_y.npy")) <= 1e-14
    assert rel(z, _gold("loop8_z.npy")) <= 1e-14
    # the reference's dense oracle products at eps 1e-6 (test_matvec.cpp:50-85)
    assert rel(y, _gold("loop8_ydense.npy")) <= 5e-6
    assert rel(z, _gold("loop8_zdense.npy")) <= 5e-6
    # OpCounts: reference == restated
    st = oracle.OracleStore(oracle.load_ctc1(os.path.join(GOLD, "loop8.ctc1")))
    ops2 = {}
    st.forward(x, 1, ops2)
    assert ops == [ops2["decompress_madds"], ops2["accumulate_madds"]]

    pw = R.RefCC.load_ctc1(os.path.join(GOLD, "pwl.ctc1"))
    assert pw.q == 12
    assert rel(pw.forward(_gold("pwl_x.npy")), _gold("pwl_y128.npy")) <= 1e-14
    assert rel(pw.adjoint(_gold("pwl_phi.npy")), _gold("pwl_z128.npy")) <= 1e-14
    # c64-rounded factors (the c64 stores' CPU side)
    pw64 = R.RefCC.from_compressed(oracle.load_ctc1(os.path.join(GOLD, "pwl.ctc1")).rounded_c64())
    assert rel(pw64.forward(_gold("pwl_x.npy")), _gold("pwl_y64.npy")) <= 1e-14
    assert rel(pw64.adjoint(_gold("pwl_phi.npy")), _gold("pwl_z64.npy")) <= 1e-14

    aca = R.RefAca.load_cta1(os.path.join(GOLD, "aca8.cta1"))
    assert rel(aca.aca_forward(_gold("aca8_x.npy")), _gold("aca8_y.npy")) <= 1e-14
    assert rel(aca.aca_adjoint(_gold("aca8_phi.npy")), _gold("aca8_z.npy")) <= 1e-14


@pytest.mark.parametrize("q,dims,m,rmax,seed", [(3, (7, 5, 9), 6, 5, 1), (12, (12, 9, 20), 4, 7, 2),
                                                (1, (1, 1, 1), 3, 1, 3), (2, (16, 3, 33), 5, 3, 4)])
def test_ref_vs_oracle_ragged_stores(oracle, q, dims, m, rmax, seed):
    from helpers import ragged_store
    cc = ragged_store(dims, q, m, 1, rmax, seed)
    ref = R.RefCC.from_compressed(cc)
    st = oracle.OracleStore(cc)
    x = oracle.random_multivector(cc.m, 3, seed + 10)
    phi = oracle.random_multivector(cc.rows, 3, seed + 11)
    for w in (1, 3):
        assert rel(ref.forward(x, w), st.forward(x, w)) <= 1e-14
        assert rel(ref.adjoint(phi, w), st.adjoint(phi, w)) <= 1e-14
    # element (src/tensor.cpp:183-196)
    t = cc.tensor(m - 1, q - 1)
    dense = oracle.reconstruct(*t)
    i = tuple(d - 1 for d in dims)
    assert abs(ref.element(m - 1, q - 1, *i) - dense[i]) <= 1e-13 * max(1.0, abs(dense[i]))


def test_ref_compress_matches_restated_compressor(oracle):
    """compress_matrix (src/compress.cpp:7-35) with the reference's own
    make_loop_scene: same per-tensor ranks as the restated hosvd
    (oracle.py), same operator to rounding."""
    g = oracle.make_centered_grid((0, 0, 0), 0.05, (8, 8, 8))
    k0 = oracle.wavenumber_from_mhz(298.06)
    sc = oracle.make_loop_scene(0.5, (0, 0.8, 0), 10, g, 0, k0, 3)
    rs = R.RefScene.loop(0.05, (8, 8, 8), 0.5, (0, 0.8, 0), 10, 0, k0)
    origin, sp, src = rs.sources()
    assert np.allclose(src, sc.sources, rtol=0, atol=1e-15) and np.allclose(origin, sc.origin, atol=1e-15)
    for eps in (1e-4, 1e-6, 1e-8):
        ref_cc = rs.compress(eps, workers=2)
        mine = oracle.compress_matrix(sc, eps, workers=2)
        got = ref_cc.to_compressed()
        assert np.array_equal(np.asarray(got.ranks).reshape(-1, 3), np.asarray(mine.ranks).reshape(-1, 3)), eps
        x = oracle.random_multivector(mine.m, 2, 5)
        phi = oracle.random_multivector(mine.rows, 2, 6)
        assert rel(oracle.OracleStore(mine).forward(x), ref_cc.forward(x)) <= 1e-12
        assert rel(oracle.OracleStore(mine).adjoint(phi), ref_cc.adjoint(phi)) <= 1e-12
        # both within the compression contract of the dense operator
        yd = rs.dense_forward(x, mine.rows)
        assert rel(ref_cc.forward(x), yd) <= 5 * eps


def test_ref_tucker_aca_matches_restated(oracle, tmp_path):
    """tucker_aca (src/aca.cpp:126-232) on the golden ACA scene: the
    reference and the restatement accept the same cross rank, and the
    products agree within the nested tolerance."""
    g = oracle.make_centered_grid((0, 0, 0), 0.04, (8, 8, 8))
    k0 = oracle.wavenumber_from_mhz(123.0)
    sc = oracle.make_loop_scene(0.5, (0, 0.9, 0), 12, g, 0, k0, 3)
    rs = R.RefScene.from_scene(sc)
    ra = rs.tucker_aca(1e-4, 0.0, str(tmp_path / "ref.cta1"))
    mine = oracle.load_cta1(os.path.join(GOLD, "aca8.cta1"))[0]
    assert ra.rank == mine.rank
    assert np.array_equal(np.asarray(oracle.load_cta1(str(tmp_path / "ref.cta1"))[0].ranks).reshape(-1, 3),
                          np.asarray(mine.ranks).reshape(-1, 3))
    x = _gold("aca8_x.npy")
    assert rel(ra.aca_forward(x), _gold("aca8_y.npy")) <= 1e-9
    # row_of_compressed_u (src/aca.cpp:234-244) vs the restated element path
    i = 5
    ri = ra.row_of_compressed_u(i)
    st = oracle.OracleStore(mine.store())
    want = np.array([st.element(l, 0, i % 8, (i // 8) % 8, i // 64) for l in range(mine.rank)])
    assert rel(ri, want) <= 1e-9


def test_ref_shapes_raise_contract_violations(oracle):
    cc = R.RefCC.load_ctc1(os.path.join(GOLD, "loop8.ctc1"))
    with pytest.raises(R.RefError) as e:
        cc.forward(np.zeros((cc.m + 1, 1)))
    assert e.value.code == 2 and "forward: x has" in str(e.value)
    with pytest.raises(R.RefError) as e:
        cc.adjoint(np.zeros((cc.rows - 1, 1)))
    assert e.value.code == 2 and "adjoint: phi has" in str(e.value)
    with pytest.raises(R.RefError) as e:
        R.RefCC.load_ctc1(os.path.join(GOLD, "aca8.cta1"))
    assert e.value.code == 5 and "bad magic" in str(e.value)
