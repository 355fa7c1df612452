#!/usr/bin/env python
"""Batched element() / row extraction (tm_rows) on the full
config-4 bench store: time R random rows (each = element() of all 5 000
columns, O(r1 r2 r3) per entry) on the GPU, and the restated reference's
element() (oracle, CPU) on a sample of the same entries; check the sample.

  python tools/rows_bench.py [--rows 256] [--cpu-entries 2000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--cpu-entries", type=int, default=2000)
    args = ap.parse_args()
    import torch
    from oracle import oracle as O
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.workloads import CONFIGS, column_scales, rank_table, synthetic_payload
    cfg = CONFIGS["c4"]
    ranks = rank_table(cfg, 1234)
    pay, _ = synthetic_payload(cfg.grid, ranks, column_scales(cfg, 1234), 2234, device="cuda")
    s = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, "c128", 0)
    rng = np.random.default_rng(5)
    rows = rng.integers(0, s.rows, args.rows)
    s.row_block(rows[:8])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = s.row_block(rows)
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    # CPU oracle element() on a sample of the entries (columns 0.. of the first rows)
    pay_np = pay.cpu().numpy()
    del pay
    n1, n2, n3 = cfg.grid
    nv = n1 * n2 * n3
    ncheck = min(args.cpu_entries, args.rows * cfg.m)
    pick = rng.integers(0, args.rows * cfg.m, ncheck)
    # oracle store over the needed columns only
    cols = sorted(set(int(p % cfg.m) for p in pick))
    sizes = []
    for j in range(cfg.m):
        for k in range(cfg.q):
            r1, r2, r3 = ranks[j, k]
            sizes.append(r1 * r2 * r3 + n1 * r1 + n2 * r2 + n3 * r3)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    sub_ranks = ranks[cols]
    sub_pay = np.concatenate([pay_np[offs[j * cfg.q]:offs[(j + 1) * cfg.q]] for j in cols])
    cc = O.Compressed(cfg.grid, cfg.q, len(cols), sub_ranks, sub_pay)
    ref = O.OracleStore(cc)
    where = {j: i for i, j in enumerate(cols)}
    err = 0.0
    t0 = time.perf_counter()
    vals = []
    for p in pick:
        r, j = int(p // cfg.m), int(p % cfg.m)
        k, v = divmod(int(rows[r]), nv)
        i1, rest = v % n1, v // n1
        vals.append(ref.element(where[j], k, i1, rest % n2, rest // n2))
    tc = time.perf_counter() - t0
    got = np.array([out[int(p // cfg.m), int(p % cfg.m)] for p in pick])
    err = float(np.linalg.norm(got - np.array(vals)) / max(np.linalg.norm(vals), 1e-300))
    entries = args.rows * cfg.m
    print(json.dumps({"store": cfg.name, "dtype": "c128", "rows": args.rows, "entries": entries,
                      "gpu_seconds": round(tg, 4), "gpu_entries_per_s": round(entries / tg, 1),
                      "cpu_oracle_entries": ncheck, "cpu_seconds": round(tc, 3),
                      "cpu_entries_per_s": round(ncheck / tc, 1), "rel_err_sample_vs_oracle": err,
                      "note": "GPU time includes the D2H copy of the rows (TM_HOST)"}))


if __name__ == "__main__":
    main()
