#!/usr/bin/env python
"""Compress every column of the config-4 physics scene on the GPU (the
close-fitting array of scenes.close_fitting_array, 192x224x256 at 1 mm,
q = 12, eps 1e-4; BASELINE.json configs[3]) and save its per-tensor Tucker
ranks and Frobenius norms:

  python tools/c4_rank_table.py --out gpurun_out/c4_ranks.npz

The payload itself (~8 GB complex128) is discarded batch by batch; the rank
table (m x q x 3) and norms (m x q) are what bench.py's config-4 store reuses
(workloads.rank_table) so the benched operator has the compressed physics
store's ranks and column magnitudes.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/c4_ranks.npz")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--cols", type=int, default=0, help="first N columns only (0 = all)")
    args = ap.parse_args()
    import torch
    from paper_2103_06393_b200 import compress as C
    from paper_2103_06393_b200 import scenes as S

    g = S.centered_grid(0.001, (192, 224, 256))
    sc = S.close_fitting_array(g, 0.006, channels=8, loops_per_channel=4, segs_per_loop=156, q=12)
    m = sc.num_sources if not args.cols else min(args.cols, sc.num_sources)
    n1, n2, n3 = sc.dims
    ranks = np.zeros((m, sc.q, 3), np.int32)
    norms = np.zeros((m, sc.q), np.float64)
    t0 = time.time()
    for j0 in range(0, m, args.batch):
        cols = list(range(j0, min(m, j0 + args.batch)))
        f = C.assemble_columns(sc, cols)
        t = f.reshape(len(cols) * sc.q, n3, n2, n1)
        nr = torch.linalg.vector_norm(t.reshape(t.shape[0], -1), dim=1).cpu().numpy()
        res = C.hosvd_batch(t, 1e-4)
        for i, (core, u1, u2, u3) in enumerate(res):
            ranks[cols[i // sc.q], i % sc.q] = (u1.shape[1], u2.shape[1], u3.shape[1])
            norms[cols[i // sc.q], i % sc.q] = nr[i]
        del f, t, res
        if j0 % 512 == 0:
            print(f"{j0}/{m} columns, {time.time() - t0:.0f} s", flush=True)
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    np.savez_compressed(args.out, ranks=ranks, norms=norms, grid=np.array(sc.dims), q=sc.q, eps=1e-4,
                        gap=0.006)
    r = ranks.reshape(-1, 3)
    print(f"{m} columns in {time.time() - t0:.0f} s; mean ranks {r.mean(0)}, max {r.max(0)}, "
          f"tensors with a rank > 16: {(r.max(1) > 16).sum()}, scalars/tensor "
          f"{(r.prod(1) + r @ np.array(sc.dims)).mean():.0f}", flush=True)


if __name__ == "__main__":
    main()
