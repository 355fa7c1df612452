#!/usr/bin/env python
"""Seeded random shapes with tensor ranks above 16 (up to 32) through the
tcgen05 path vs the CPU oracle (development sweep; the committed cases are in
tests/test_gpu_parity.py::test_ranks_above_16_stay_on_tensor_cores)."""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from helpers import ragged_store, cn01  # noqa: E402
import paper_2103_06393_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(5000 + seed)
    dims = (int(rng.integers(1, 70)), int(rng.integers(1, 70)), int(rng.integers(16, 260)))
    q = int(rng.choice([1, 2, 3, 12]))
    m = int(rng.integers(1, 30))
    rmax = int(rng.integers(17, 33))
    p = int(rng.choice([1, 2, 3, 4, 5, 9]))
    while q * m * dims[0] * dims[1] * dims[2] > 4e7 and m > 1:
        m //= 2
    cc = ragged_store(dims, q, m, 1, rmax, seed=seed)
    ds = P.DeviceStore.from_compressed(cc, "c64")
    ref = O.OracleStore(cc.rounded_c64())
    x = cn01(m, p, seed).astype(np.complex64).astype(np.complex128)
    phi = cn01(cc.rows, p, seed + 1).astype(np.complex64).astype(np.complex128)
    yo, zo = ref.forward(x), ref.adjoint(phi)
    y = ds.forward(x)
    ef = np.linalg.norm(y - yo) / np.linalg.norm(yo)
    z = ds.adjoint(phi)
    ea = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    print(seed, dims, q, m, rmax, p, ds.kernel_paths(), f"{ef:.2e} {ea:.2e}", "OK" if max(ef, ea) < 1e-5 else "BAD",
          flush=True)
