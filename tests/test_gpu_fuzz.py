"""Seeded random-shape sweep of the GPU products against the CPU oracle.

Each case draws a grid (1..80 per mode, n3 up to 300), q in {1, 2, 3, 12},
column counts and ragged ranks (up to the tensor-core bound 16, clipped to
the grid), a dtype and a right-hand-side count, so the launch-shape logic
(tile splits of partial waves and small stores, CTA-pair eligibility,
right-hand-side groups of the adjoint, CUDA-core column splits) meets shapes
the hand-picked parity cases do not.  Tolerances as tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

from conftest import rel
from helpers import cn01, ragged_store

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    dims = tuple(int(v) for v in rng.integers(1, 81, 2)) + (int(rng.integers(1, 301)),)
    q = int(rng.choice([1, 2, 3, 12]))
    m = int(rng.integers(1, 60))
    rmin = int(rng.integers(1, 6))
    rmax = int(rng.integers(rmin, 17))
    dtype = "c64" if rng.random() < 0.75 else "c128"
    p = int(rng.choice([1, 1, 2, 3, 4, 5, 7, 9]))
    # keep the oracle (pure numpy over q * m tensors of n1 n2 n3 voxels) fast
    while q * m * dims[0] * dims[1] * dims[2] > 6e7 and m > 1:
        m //= 2
    return dims, q, m, rmin, rmax, dtype, p


@pytest.mark.parametrize("seed", range(48))
def test_random_shapes(oracle, product, seed):
    O, P = oracle, product
    dims, q, m, rmin, rmax, dtype, p = _case(seed)
    cc = ragged_store(dims, q, m, rmin, rmax, seed=seed)
    ref = O.OracleStore(cc.rounded_c64() if dtype == "c64" else cc)
    ds = P.DeviceStore.from_compressed(cc, dtype)
    x = cn01(m, p, 3 + seed)
    phi = cn01(cc.rows, p, 5 + seed)
    if dtype == "c64":
        x = x.astype(np.complex64).astype(np.complex128)
        phi = phi.astype(np.complex64).astype(np.complex128)
    case = f"dims={dims} q={q} m={m} ranks=[{rmin},{rmax}] {dtype} p={p}"
    assert rel(ds.forward(x), ref.forward(x)) <= TOL[dtype], case
    assert rel(ds.adjoint(phi), ref.adjoint(phi)) <= TOL[dtype], case
