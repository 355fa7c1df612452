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
    # (p >= 16 runs K3W, T = W U3^T rounded to fp16 splits before Y += T X)
    print(f"forward {rel(yw, yo):.2e} / {rel(yp, yo):.2e}, adjoint gemm {rel(zw, zo):.2e} / consumers {rel(zp, zo):.2e}")
    assert rel(yw, yp) <= (1e-5 if p >= 16 else 1e-6) and rel(zw, zp) <= 1e-5
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


@pytest.mark.parametrize("dims,q,m,rmin,rmax,p", [
    ((64, 64, 64), 12, 40, 4, 9, 32),     # config-5 shape, one 32-right-hand-side pass
    ((21, 40, 37), 3, 19, 1, 13, 16),     # ragged: n1 / n2 / n3 not multiples of the tile, m not of 16
    ((9, 33, 70), 2, 35, 3, 16, 40),      # rank-16 factors, two passes (32 + 8)
    ((16, 32, 20), 1, 100, 2, 5, 20),     # many columns: several accumulation chains per tile
    ((20, 36, 24), 2, 1, 16, 16, 17),     # one column, r3 = 16 (whole stages of one column)
])
def test_k3w_forward(oracle, product, monkeypatch, dims, q, m, rmin, rmax, p):
    """K3W, the batched forward of a W-arena store at the algorithmic cost (T
    decompressed once per tile from the arena, Y += T X on tcgen05; the
    default for p >= 16) vs the oracle and vs the x-in-B arena forward
    (TMB_K3=0), with short accumulation chains and the default."""
    O, P = oracle, product
    cc = ragged_store(dims, q, m, rmin, rmax, seed=7 * m + p)
    ref = O.OracleStore(cc.rounded_c64())
    ds = P.DeviceStore.from_compressed(cc, "c64")
    assert ds.kernel_paths()["forward"] == "tcgen05+warena"
    x = _c64(cn01(m, p, 17))
    yo = ref.forward(x)
    monkeypatch.setenv("TMB_TC_CHAIN", "3")  # short chains: exercise the fold
    y3 = ds.forward(x)
    monkeypatch.delenv("TMB_TC_CHAIN")
    y3b = ds.forward(x)
    monkeypatch.setenv("TMB_K3", "0")
    yb = ds.forward(x)
    monkeypatch.delenv("TMB_K3")
    print(f"K3W {rel(y3b, yo):.2e} (chains of 3: {rel(y3, yo):.2e}), x-in-B {rel(yb, yo):.2e}")
    assert rel(y3, yo) <= 1e-5 and rel(y3b, yo) <= 1e-5 and rel(yb, yo) <= 1e-5
    assert rel(ds.forward(x), y3b) == 0.0  # deterministic
    assert rel(ds.forward(x[:, :1]), yo[:, :1]) <= 1e-5  # p = 1 stays on the x-in-B forward
