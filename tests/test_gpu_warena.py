"""The W arena (fwd_tc_kernel<..., WA>): for stores whose W = U1 x1 G x2 U2
fits the memory budget, the forward's A operand is precomputed once
(build_warena_kernel) and streamed by TMA — no producer warps — and the
adjoint runs as one GEMM, G = conj(W)^T Phi on the transposed arena
(fwd_tc_kernel<..., WA, ADJ>), then z = sum conj(U3) G (adjg_contract_kernel).  Checked
against the oracle and against the producer-warp forward of the same store
(TMB_WARENA=0 switches a store back at run time), over ragged ranks, grids
whose n2 is not a multiple of 32, one and many right-hand sides, split final
waves (cut at K-stage boundaries) and CTA pairs; and the budget switch."""
import numpy as np
import pytest

from conftest import rel
from helpers import cn01, ragged_store

pytestmark = pytest.mark.gpu


def _c64(a):
    return a.astype(np.complex64).astype(np.complex128)


@pytest.mark.parametrize("dims,q,m,rlo,rhi,p", [
    ((16, 12, 40), 3, 17, 2, 9, 1),       # single-CTA tiles, n2 < 32
    ((64, 64, 64), 12, 10, 2, 9, 3),      # q = 12, three right-hand sides
    ((48, 40, 256), 3, 23, 4, 12, 1),     # CTA pairs (256-voxel i3 span), n2 = 40
    ((40, 36, 140), 2, 9, 10, 16, 2),     # two i3 halves
    ((24, 32, 64), 3, 300, 1, 6, 40),     # many columns and right-hand sides
    ((8, 8, 16), 1, 2, 1, 3, 1),          # tiny
])
def test_warena_products_match_oracle_and_producer_path(oracle, product, dims, q, m, rlo, rhi, p, monkeypatch):
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rlo, rhi, seed=m + q + p)
    ds = P.DeviceStore.from_compressed(cc, "c64")
    assert ds.kernel_paths() == {"forward": "tcgen05+warena", "adjoint": "tcgen05+gemm"}
    ref = O.OracleStore(cc.rounded_c64())
    x = _c64(cn01(m, p, 11))
    phi = _c64(cn01(cc.rows, p, 12))
    yo, zo = ref.forward(x), ref.adjoint(phi)
    yw, zw = ds.forward(x), ds.adjoint(phi)
    assert rel(yw, yo) <= 1e-5 and rel(zw, zo) <= 1e-5
    monkeypatch.setenv("TMB_WARENA", "0")
    assert ds.kernel_paths() == {"forward": "tcgen05", "adjoint": "tcgen05"}
    yp, zp = ds.forward(x), ds.adjoint(phi)
    assert rel(yp, yo) <= 1e-5 and rel(zp, zo) <= 1e-5
    # the same W bits: the forwards differ only where final-wave splits differ
    print(f"forward {rel(yw, yo):.2e} / {rel(yp, yo):.2e}, adjoint gemm {rel(zw, zo):.2e} / consumers {rel(zp, zo):.2e}")
    assert rel(yw, yp) <= 1e-6 and rel(zw, zp) <= 1e-5
    monkeypatch.delenv("TMB_WARENA")
    assert rel(ds.forward(x), yw) == 0.0 and rel(ds.adjoint(phi), zw) == 0.0  # deterministic
    # the adjoint GEMM's final partial wave split into row (K-stage) parts vs unsplit
    monkeypatch.setenv("TMB_ADJ_NOSPLIT", "1")
    zn = ds.adjoint(phi)
    monkeypatch.delenv("TMB_ADJ_NOSPLIT")
    assert rel(zn, zo) <= 1e-5 and rel(zn, zw) <= 1e-6
    # TMB_ADJ_GEMM=0: the consumer-warp adjoint (forming W) on an arena store
    monkeypatch.setenv("TMB_ADJ_GEMM", "0")
    assert ds.kernel_paths() == {"forward": "tcgen05+warena", "adjoint": "tcgen05"}
    za = ds.adjoint(phi)
    assert rel(za, zo) <= 1e-5 and rel(za, zp) == 0.0


def test_warena_budget(oracle, product, monkeypatch):
    """A store whose W arena exceeds $TMB_WARENA_GB keeps the producer path;
    TMB_WARENA=0 at build time builds none."""
    P = product
    cc = ragged_store((32, 32, 64), 3, 8, 2, 6, seed=5)
    monkeypatch.setenv("TMB_WARENA_GB", "0.000001")
    assert P.DeviceStore.from_compressed(cc, "c64").kernel_paths()["forward"] == "tcgen05"
    monkeypatch.delenv("TMB_WARENA_GB")
    monkeypatch.setenv("TMB_WARENA", "0")
    ds = P.DeviceStore.from_compressed(cc, "c64")
    monkeypatch.delenv("TMB_WARENA")
    assert ds.kernel_paths()["forward"] == "tcgen05"
    assert P.DeviceStore.from_compressed(cc, "c64").kernel_paths()["forward"] == "tcgen05+warena"
