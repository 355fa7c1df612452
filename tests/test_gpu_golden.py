"""GPU path against the committed golden fixtures (tests/golden/), through the
native CTC1 / CTA1 ingest of the C ABI, the C++ drop-in, and the sm_100a
UMMA building-block probe."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


def ld(f):
    return np.load(os.path.join(GOLD, f))


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-12), ("c64", 1e-5)])
def test_golden_loop_scene(product, dtype, tol):
    P = product
    s = P.load_ctc1(os.path.join(GOLD, "loop8.ctc1"), dtype)
    assert (s.q, s.ncols, s.dims) == (3, 10, (8, 8, 8))
    x, phi = ld("loop8_x.npy"), ld("loop8_phi.npy")
    if dtype == "c64":  # the c64 store's golden values are the c128 ones within the c64 tolerance
        x = x.astype(np.complex64)
        phi = phi.astype(np.complex64)
    assert rel(s.forward(x), ld("loop8_y.npy")) <= (tol if dtype == "c128" else 1e-5)
    assert rel(s.adjoint(phi), ld("loop8_z.npy")) <= (tol if dtype == "c128" else 1e-5)
    # and within 5 eps of the dense matrix (test_matvec.cpp:50-58)
    assert rel(s.forward(x), ld("loop8_ydense.npy")) <= 5e-6


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-12), ("c64", 1e-5)])
def test_golden_aca(product, dtype, tol):
    P = product
    s = P.load_cta1(os.path.join(GOLD, "aca8.cta1"), dtype)
    assert s.m2 == 12 and s.ncols == 12
    x, phi = ld("aca8_x.npy"), ld("aca8_phi.npy")
    assert rel(s.aca_forward(x), ld("aca8_y.npy")) <= tol
    assert rel(s.aca_adjoint(phi), ld("aca8_z.npy")) <= tol


def test_golden_pwl(product):
    P = product
    s64 = P.load_ctc1(os.path.join(GOLD, "pwl.ctc1"), "c64")
    s128 = P.load_ctc1(os.path.join(GOLD, "pwl.ctc1"), "c128")
    x, phi = ld("pwl_x.npy"), ld("pwl_phi.npy")
    assert rel(s64.forward(x), ld("pwl_y64.npy")) <= 1e-5
    assert rel(s64.adjoint(phi), ld("pwl_z64.npy")) <= 1e-5
    assert rel(s128.forward(x), ld("pwl_y128.npy")) <= 1e-12
    assert rel(s128.adjoint(phi), ld("pwl_z128.npy")) <= 1e-12


def test_cpp_dropin_on_gpu(product, tmp_path):
    """The C++ drop-in (reference signatures) against the golden products."""
    from test_capi_cpu import build_dropin_test
    exe = build_dropin_test(tmp_path)
    r = subprocess.run([str(exe), os.path.join(GOLD, "loop8.ctc1")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu forward ok rows=1536" in r.stdout and "gpu adjoint ok" in r.stdout
    assert "contract: element: index out of range" in r.stdout
    # element(tensor (j=3, k=1), 2, 5, 7) vs the oracle's element()
    from oracle import oracle as O
    cc = O.load_ctc1(os.path.join(GOLD, "loop8.ctc1"))
    want = O.OracleStore(cc).element(3, 1, 2, 5, 7)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("element ")][0].split()
    got = complex(float(line[1]), float(line[2]))
    assert abs(got - want) <= 1e-12 * max(abs(want), 1e-30)


def test_umma_probe():
    """tcgen05 / TMA / TMEM building blocks on sm_100a (tests/cuda/umma_probe.cu)."""
    exe = os.path.join(ROOT, "tests", "cuda", "bin", "umma_probe")
    if not os.path.exists(exe):
        pytest.skip("probe not built (run __graft_entry__.build())")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "PROBE OK" in r.stdout, r.stdout
