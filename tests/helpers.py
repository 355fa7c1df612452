"""Seeded test stores (test infrastructure)."""
import numpy as np


def ragged_store(dims, q, m, rmin, rmax, seed, scale_decay=0.0):
    """Random Tucker store with per-tensor ragged ranks in [rmin, rmax]
    (clipped to the grid), random cores and QR-orthonormal factors — the
    pattern of the reference's synthetic_compression (tests/test_compress.cpp:21-45)
    with ranks that differ per tensor and per mode."""
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    tensors = []
    for j in range(m):
        for k in range(q):
            rk = [int(min(d, rng.integers(rmin, rmax + 1))) for d in dims]
            core = (rng.standard_normal(rk) + 1j * rng.standard_normal(rk)) * np.exp(-scale_decay * j)
            us = []
            for g in range(3):
                a = rng.standard_normal((dims[g], rk[g])) + 1j * rng.standard_normal((dims[g], rk[g]))
                us.append(np.asfortranarray(np.linalg.qr(a)[0]))
            tensors.append((np.asfortranarray(core), us[0], us[1], us[2]))
    ranks, payload = O.pack_tensors(tensors)
    return O.Compressed(tuple(dims), q, m, ranks.reshape(m, q, 3), payload, 0, 1.0, 1e-6)


def cn01(rows, cols, seed):
    """Seeded CN(0,1) block: the reference generator (src/experiments.cpp:26-33) scaled by 1/sqrt(2)."""
    from oracle import oracle as O
    return O.random_multivector(rows, cols, seed) / np.sqrt(2.0)
