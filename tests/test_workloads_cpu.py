"""Benchmark workload definitions (BASELINE.json configs) on CPU."""
import numpy as np

from conftest import ROOT
from paper_2103_06393_b200.sharded import column_costs
from paper_2103_06393_b200.workloads import CONFIGS, rank_table, synthetic_payload, tensor_offsets


def test_configs_match_baseline():
    c4 = CONFIGS["c4"]
    assert c4.grid == (192, 224, 256) and c4.q == 12 and abs(c4.m - 5000) < 100 and c4.dtype == "c64"
    assert CONFIGS["c1"].grid == (24, 24, 24) and CONFIGS["c1"].dtype == "c128" and CONFIGS["c1"].m == 128
    assert CONFIGS["c5"].p == 32 and CONFIGS["c5"].q == 12
    assert CONFIGS["c3"].aca_m2 == 2048


def test_config4_uses_the_measured_physics_rank_table():
    """data/c4_physics_ranks.npz (tools/c4_rank_table.py on a B200: all 4 992
    columns of the close-fitting array, eps 1e-4): ranks 9-12, mean ~10.5,
    ~8 200 scalars per tensor, ~4 GB compressed store (c64)."""
    from paper_2103_06393_b200.workloads import tensor_scales
    cfg = CONFIGS["c4"]
    r = rank_table(cfg)
    assert r.shape == (cfg.m, cfg.q, 3)
    assert r.min() >= 9 and r.max() <= 12
    assert 10.0 <= r.mean() <= 11.0
    n = np.array(cfg.grid)
    scalars = (r[..., 0] * r[..., 1] * r[..., 2] + r @ n).sum()
    assert 3.6e9 < 8 * scalars < 4.4e9
    s = tensor_scales(cfg)
    assert s.shape == (cfg.m, cfg.q) and s.max() == 1.0 and s.min() > 0


def test_rank_model_matches_survey_probes():
    """ranks 4-12 at the survey's gaps (configs without a measured table)."""
    r = rank_table(CONFIGS["c2"])
    assert r.min() >= 4 and r.max() <= 13
    assert 6.0 <= r.mean() <= 9.5


def test_column_costs_are_opcounts(oracle):
    cc = oracle.synthetic_compression(6, 3, 2, 1)
    st = oracle.OracleStore(cc)
    dec, acc = st.opcounts(4)
    assert column_costs(cc.grid_dims, cc.ranks, 4).sum() == dec + acc


def test_synthetic_payload_layout_cpu(oracle):
    """The device generator's CTC1 layout on CPU: orthonormal factors, seeded."""
    import torch
    cfg = CONFIGS["c1"]
    ranks = rank_table(cfg)[:3]
    pay, off = synthetic_payload(cfg.grid, ranks, np.ones(3), 5, device="cpu")
    pay2, _ = synthetic_payload(cfg.grid, ranks, np.ones(3), 5, device="cpu")
    assert torch.equal(pay, pay2)
    assert off[-1] == tensor_offsets(cfg.grid, ranks)[-1] == pay.numel()
    p = pay.numpy()
    for i in range(ranks.shape[0] * ranks.shape[1]):
        core, u1, u2, u3 = oracle.split_tensor(cfg.grid, ranks.reshape(-1, 3)[i], p[off[i]:off[i + 1]])
        for u in (u1, u2, u3):
            assert np.linalg.norm(u.conj().T @ u - np.eye(u.shape[1])) < 1e-12


def test_cpu_sample_columns_are_balanced_and_cover_the_payload():
    """The CPU legs' column sample (bench.sample_columns): n distinct columns
    in order, per-column madds within a narrow band around the median; and
    bench.column_payload returns exactly those columns' tensors."""
    import sys
    sys.path.insert(0, ROOT)
    import bench as B
    from paper_2103_06393_b200.sharded import column_costs
    from paper_2103_06393_b200.workloads import CONFIGS, rank_table, tensor_offsets
    cfg = CONFIGS["c4"]
    ranks = rank_table(cfg, 1234)
    costs = column_costs(cfg.grid, ranks, cfg.p)
    sel = B.sample_columns(cfg, ranks, 32)
    assert len(set(sel.tolist())) == 32 and np.all(np.diff(sel) > 0)
    med = np.median(costs)
    assert np.abs(costs[sel] - med).max() <= np.abs(costs - med).max() * 0.1
    small = CONFIGS["c1"]
    r1 = rank_table(small, 1234)
    off = tensor_offsets(small.grid, r1)
    pay = np.arange(off[-1]).astype(np.complex128)
    sel1 = B.sample_columns(small, r1, 5)
    got = B.column_payload(small, r1, pay, sel1)
    want = np.concatenate([pay[off[j * small.q]:off[(j + 1) * small.q]] for j in sel1])
    assert np.array_equal(got, want)
