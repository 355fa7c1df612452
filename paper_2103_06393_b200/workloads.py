"""Benchmark workloads (BASELINE.json configs) and seeded synthetic stores.

The paper's MRI models and coil meshes are not available (SURVEY.md §0 gap 4)
and compressing the 1 mm-class config at real scale is the "next" row of
SURVEY.md §8f, so the benchmark stores are seeded synthetic Tucker stores
with the configs' shapes, component counts, column counts and rank
distributions: random complex-normal cores and QR-orthonormal factors, the
pattern of the reference's synthetic_compression
(proj/tests/test_compress.cpp:21-45), with per-tensor ranks drawn from the
survey's rank-vs-distance probes and per-column
magnitudes that decay with the coil-edge distance the way a dipole field does.
Physics-compressed stores (loop scenes, compress_matrix) are used by the
parity tests at the sizes the CPU oracle can produce.

Config 4 uses the MEASURED rank table of its physics store instead: every
one of the 4 992 columns of the close-fitting array (scenes.close_fitting_array,
192x224x256 at 1 mm, q = 12) was compressed on a B200 with the GPU compressor
at eps 1e-4 (tools/c4_rank_table.py, data/c4_physics_ranks.npz: per-tensor
ranks and Frobenius norms).  The benched store has exactly those ranks and
those per-tensor magnitudes, with seeded random cores and orthonormal factors
in place of the physics values (the 4 GB payload itself is not shipped).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    grid: tuple
    q: int
    m: int
    dtype: str
    p: int
    # rank model: gap range (mm) -> ranks per the survey's probe table
    gap_mm: tuple
    aca_m2: int = 0  # ACA configs: length of V's column space (coil edges)
    rank_source: str = ""  # "" = survey rank model; else a measured table in data/<rank_source>.npz


# Survey probes (SURVEY.md Appendix A, config-4 grid, eps 1e-4): gap -> (r1, r2, r3).
_GAP_TABLE = [(3.0, (11, 11, 12)), (6.0, (10, 11, 11)), (12.0, (9, 9, 10)), (25.0, (7, 8, 8)), (50.0, (5, 6, 7))]

CONFIGS = {
    "c1": Config("c1: 24^3 5mm PWC loop, 128 edges, c128", (24, 24, 24), 3, 128, "c128", 1, (40.0, 60.0)),
    "c2": Config("c2: 64^3 2mm PWC birdcage-like, 1024 edges, c64", (64, 64, 64), 3, 1024, "c64", 1, (12.0, 50.0)),
    "c3": Config("c3: 96^3 2mm PWL ACA, r_c 150 of 2048 edges, c64", (96, 96, 96), 12, 150, "c64", 1, (25.0, 50.0),
                 aca_m2=2048),
    "c4": Config("c4: 192x224x256 1mm PWL close-fitting array, 4992 edges (physics rank table), c64",
                 (192, 224, 256), 12, 4992, "c64", 1, (3.0, 50.0), rank_source="c4_physics_ranks"),
    "c5": Config("c5: 64^3 2mm PWL, 1024 edges, p=32, c64", (64, 64, 64), 12, 1024, "c64", 32, (12.0, 50.0)),
}


def _interp_ranks(gap):
    g = min(max(gap, _GAP_TABLE[0][0]), _GAP_TABLE[-1][0])
    for (g0, r0), (g1, r1) in zip(_GAP_TABLE, _GAP_TABLE[1:]):
        if g <= g1:
            t = (math.log(g) - math.log(g0)) / (math.log(g1) - math.log(g0))
            return [r0[i] + t * (r1[i] - r0[i]) for i in range(3)]
    return list(_GAP_TABLE[-1][1])


def column_gaps(cfg: Config, seed: int):
    """Edge-to-grid distance per column (mm); more edges close to the body."""
    rng = np.random.default_rng(seed)
    lo, hi = cfg.gap_mm
    u = rng.random(cfg.m)
    return lo + (hi - lo) * u ** 1.5


DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


def _measured(cfg: Config):
    d = np.load(os.path.join(DATA, cfg.rank_source + ".npz"))
    ranks, norms = d["ranks"].astype(np.int32), d["norms"].astype(np.float64)
    if ranks.shape != (cfg.m, cfg.q, 3) or tuple(int(v) for v in d["grid"]) != tuple(cfg.grid):
        raise ValueError(f"{cfg.rank_source}: table shape {ranks.shape} does not match {cfg.name}")
    return ranks, norms


def rank_table(cfg: Config, seed: int = 1234):
    """(m, q, 3) int32 ranks: the measured table of the config's physics
    store when there is one, else the survey table at each column's gap with
    +-1 jitter per tensor."""
    if cfg.rank_source:
        return _measured(cfg)[0]
    rng = np.random.default_rng(seed + 7)
    gaps = column_gaps(cfg, seed)
    out = np.zeros((cfg.m, cfg.q, 3), np.int32)
    for j, gp in enumerate(gaps):
        base = _interp_ranks(gp)
        jit = rng.integers(-1, 2, size=(cfg.q, 3))
        out[j] = np.clip(np.rint(np.asarray(base)[None, :] + jit), 1, np.asarray(cfg.grid)[None, :])
    return out


def column_scales(cfg: Config, seed: int = 1234):
    """Relative column magnitude ~ (3 mm / gap)^2 (near-field dipole decay)."""
    return (3.0 / column_gaps(cfg, seed)) ** 2


def tensor_scales(cfg: Config, seed: int = 1234):
    """(m, q) core scales of the synthetic store: with a measured table, the
    physics tensors' Frobenius norms (a random CN(0,1) core of r1 r2 r3
    entries has norm ~ sqrt(r1 r2 r3)), relative to the largest; else the
    column decay model, the same for the q components."""
    if cfg.rank_source:
        ranks, norms = _measured(cfg)
        s = norms / np.sqrt(ranks.prod(axis=2))
        return s / s.max()
    return np.repeat(column_scales(cfg, seed)[:, None], cfg.q, axis=1)


def tensor_offsets(dims, ranks):
    r = np.asarray(ranks, np.int64).reshape(-1, 3)
    n = np.asarray(dims, np.int64)
    sizes = r[:, 0] * r[:, 1] * r[:, 2] + r @ n
    off = np.zeros(len(sizes) + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    return off


def synthetic_payload(dims, ranks, scales, seed, device="cuda"):
    """CTC1-layout payload (complex128 torch tensor on `device`) for the
    tensors of `ranks` ((ncols, q, 3), [col][comp] order): cores ~ CN(0,1) x
    scale (per column (ncols,) or per tensor (ncols, q)), factors = Q of a complex-normal matrix (orthonormal
    columns), generated in rank-grouped batches with a seeded generator."""
    import torch

    dims = tuple(int(d) for d in dims)
    if np.asarray(ranks).ndim != 3:
        raise ValueError("ranks must be (ncols, q, 3)")
    q = np.asarray(ranks).shape[1]
    r = np.asarray(ranks, np.int64).reshape(-1, 3)
    off = tensor_offsets(dims, r)
    total = int(off[-1])
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    pay = torch.empty(total, dtype=torch.complex128, device=device)
    off_t = torch.from_numpy(off[:-1]).to(device)
    # cores
    csz = torch.from_numpy(r[:, 0] * r[:, 1] * r[:, 2]).to(device)
    ncore = int(csz.sum())
    start = torch.repeat_interleave(off_t, csz)
    within = torch.arange(ncore, device=device) - torch.repeat_interleave(torch.cumsum(csz, 0) - csz, csz)
    scales = np.asarray(scales, np.float64)
    sc = torch.from_numpy(np.repeat(scales, q) if scales.ndim == 1 else scales.reshape(-1)).to(device)
    vals = torch.randn(ncore, dtype=torch.complex128, device=device, generator=gen)
    pay[start + within] = vals * torch.repeat_interleave(sc, csz)
    # factors, grouped by (mode, rank)
    base = r[:, 0] * r[:, 1] * r[:, 2]
    seg = [base, base + dims[0] * r[:, 0], base + dims[0] * r[:, 0] + dims[1] * r[:, 1]]
    for g in range(3):
        n = dims[g]
        for rk in np.unique(r[:, g]):
            ids = np.flatnonzero(r[:, g] == rk)
            for c0 in range(0, len(ids), 4096):
                sel = ids[c0:c0 + 4096]
                a = torch.randn((len(sel), n, int(rk)), dtype=torch.complex128, device=device, generator=gen)
                qm = torch.linalg.qr(a)[0]  # (b, n, rk) orthonormal columns
                o = torch.from_numpy(off[sel] + seg[g][sel]).to(device)
                i = torch.arange(n, device=device)
                aa = torch.arange(int(rk), device=device)
                idx = o[:, None, None] + i[None, :, None] + n * aa[None, None, :]
                pay[idx.reshape(-1)] = qm.reshape(-1)
    return pay, off


def synthetic_v(cfg: Config, seed: int = 1234):
    """ACA V factor (m2 x r_c, complex128, column-major) for the ACA configs:
    column l stands for conj(r_l / r_l(j_l)), the pivot-normalised residual
    row of Algorithm 3 (proj/src/aca.cpp:184-186) — unit pivot entry and
    entries of magnitude below one."""
    if not cfg.aca_m2:
        raise ValueError(f"{cfg.name} is not an ACA config")
    rng = np.random.default_rng(seed + 17)
    v = (rng.standard_normal((cfg.aca_m2, cfg.m)) + 1j * rng.standard_normal((cfg.aca_m2, cfg.m))) / 3.0
    piv = rng.choice(cfg.aca_m2, size=cfg.m, replace=False)
    v[piv, np.arange(cfg.m)] = 1.0
    return np.asfortranarray(v)


def bench_store_arrays(cfg: Config, seed: int = 1234, c0: int = 0, c1: int | None = None, device="cuda"):
    """The bench's store for columns [c0, c1): (ranks, complex128 payload
    tensor on `device`) — exactly what bench.py builds, so the full-size
    parity tests check the benched operator."""
    c1 = cfg.m if c1 is None else c1
    ranks = rank_table(cfg, seed)
    scales = tensor_scales(cfg, seed)
    pay, _ = synthetic_payload(cfg.grid, ranks[c0:c1], scales[c0:c1], seed + 1000 + c0, device=device)
    return ranks[c0:c1], pay
