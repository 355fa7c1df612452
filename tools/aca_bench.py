#!/usr/bin/env python
"""Time the GPU Tucker-ACA (paper_2103_06393_b200/aca.py) and
the restated reference tucker_aca (oracle, CPU) on a small scene, then the
GPU Tucker-ACA alone on the config-3 geometry (96^3 at 2 mm, q = 12, 2 048
edges on a 16-rung cylinder of radius 0.30 m, eps 1e-4), with the ACA
products of the resulting store.  One JSON line per case.

  python tools/aca_bench.py [--skip-c3]
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
    ap.add_argument("--skip-c3", action="store_true")
    args = ap.parse_args()
    import torch
    from oracle import oracle as O
    from paper_2103_06393_b200 import aca as A
    from paper_2103_06393_b200 import scenes as S

    # small case: both arms
    g = O.make_centered_grid((0, 0, 0), 0.01, (16, 16, 16))
    sc = O.make_loop_scene(0.12, (0, 0.2, 0), 48, g, 0, O.wavenumber_from_mhz(298.0), 3)
    eps = 1e-4
    A.tucker_aca(sc, eps)  # warm-up (kernels, cuSOLVER handles)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fac = A.tucker_aca(sc, eps)
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    row, col, m1, m2 = O.coupling_oracle(sc)
    t0 = time.perf_counter()
    ref = O.tucker_aca(row, col, m1, m2, sc.dims, 3, eps)
    tc = time.perf_counter() - t0
    print(json.dumps({"case": "16^3 loop, 48 edges, q=3, eps 1e-4", "rank": fac.rank, "rank_oracle": ref.rank,
                      "gpu_seconds": round(tg, 3), "cpu_oracle_seconds": round(tc, 3),
                      "cpu_note": "restated reference, 1 worker (the reference's tucker_aca runs workers = 1)"}),
          flush=True)
    if args.skip_c3:
        return
    grid = S.centered_grid(0.002, (96, 96, 96))
    sc3 = S.birdcage(grid, 0.30, 0.40, rungs=16, segs_per_rung=128, ring_segs=0, q=12)
    trace = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fac3 = A.tucker_aca(sc3, 1e-4, trace=trace)
    torch.cuda.synchronize()
    t3 = time.perf_counter() - t0
    ds = fac3.store("c64")
    m2 = sc3.num_sources
    x = torch.randn((1, m2), dtype=torch.complex64, device="cuda").t().contiguous()
    phi = torch.randn((1, ds.rows), dtype=torch.complex64, device="cuda").t().contiguous()
    for _ in range(2):
        ds.aca_forward(x)
        ds.aca_adjoint(phi)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    ds.aca_forward(x)
    e[1].record()
    ds.aca_adjoint(phi)
    e[2].record()
    e[2].synchronize()
    print(json.dumps({"case": "config 3: 96^3 2 mm, q=12, 2048 edges (16-rung cylinder R 0.30 m), eps 1e-4",
                      "rank": fac3.rank, "converged": bool(fac3.converged), "gpu_aca_seconds": round(t3, 2),
                      "mean_tucker_ranks": [round(float(v), 2) for v in fac3.ranks.reshape(-1, 3).mean(0)],
                      "aca_forward_ms": round(e[0].elapsed_time(e[1]), 3),
                      "aca_adjoint_ms": round(e[1].elapsed_time(e[2]), 3)}), flush=True)


if __name__ == "__main__":
    main()
