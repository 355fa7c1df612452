#!/usr/bin/env python
"""Time the GPU compressor (paper_2103_06393_b200/compress.py)
on the configs' geometries, and the restated reference compressor (oracle,
CPU) on samples of the same scenes.  One JSON line per case.

  python tools/compress_bench.py [--cases c1,c2,c4] [--c4-cols 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def scene_for(name):
    from paper_2103_06393_b200 import scenes as S
    if name == "c1":
        # 24^3, 5 mm, loop r = 10 cm 4 cm off the +y face, 128 edges (BASELINE configs[0])
        g = S.centered_grid(0.005, (24, 24, 24))
        import math
        m, r = 128, 0.10
        src = []
        for s in range(m):
            th = 2 * math.pi * (s + 0.5) / m
            src.append([r * math.cos(th), 0.10, r * math.sin(th), -math.sin(th), 0.0, math.cos(th),
                        2 * r * math.sin(math.pi / m)])
        return S.Scene(g[0], g[1], g[2], np.array(src), 0, S.wavenumber_from_mhz(298.0), 3), 1e-6
    if name == "c2":
        g = S.centered_grid(0.002, (64, 64, 64))
        return S.birdcage(g, 0.11, 0.16, rungs=8, segs_per_rung=48, ring_segs=128, shield_radius=0.13,
                          shield_rows=4, shield_segs=128, q=3), 1e-4
    if name == "c4":
        g = S.centered_grid(0.001, (192, 224, 256))
        return S.close_fitting_array(g, 0.006, channels=8, loops_per_channel=4, segs_per_loop=156, q=12), 1e-4
    raise ValueError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1,c2,c4")
    ap.add_argument("--c4-cols", type=int, default=8)
    ap.add_argument("--cpu-cols", type=int, default=4)
    args = ap.parse_args()
    import torch
    from paper_2103_06393_b200 import compress as C
    for name in args.cases.split(","):
        sc, eps = scene_for(name)
        m = sc.num_sources
        cols = m if name != "c4" else min(m, args.c4_cols)
        sub = type(sc)(sc.origin, sc.spacing, sc.dims, sc.sources[:cols], sc.op, sc.k0, sc.q)
        C.compress_scene(type(sc)(sc.origin, sc.spacing, sc.dims, sc.sources[:1], sc.op, sc.k0, sc.q), eps)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ranks, payload = C.compress_scene(sub, eps)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        line = {"case": name, "grid": list(sc.dims), "q": sc.q, "edges": m, "eps": eps, "gpu_cols": cols,
                "gpu_seconds": round(dt, 3), "gpu_ms_per_column": round(1e3 * dt / cols, 2),
                "gpu_seconds_all_columns": round(dt * m / cols, 1),
                "mean_ranks": [round(float(v), 2) for v in ranks.reshape(-1, 3).mean(0)],
                "scalars_per_tensor": round(float(payload.numel()) / (cols * sc.q), 1)}
        if name != "c4":
            from oracle import oracle as O
            oc = type(O.Scene(sc.origin, sc.spacing, sc.dims, sc.sources))(
                sc.origin, sc.spacing, sc.dims, sc.sources[:args.cpu_cols], sc.op, sc.k0, sc.q)
            t0 = time.perf_counter()
            cc = O.compress_matrix(oc, eps, workers=os.cpu_count())
            dc = time.perf_counter() - t0
            line.update({"cpu_oracle_cols": args.cpu_cols, "cpu_seconds": round(dc, 3),
                         "cpu_cores": os.cpu_count(), "cpu_seconds_all_columns": round(dc * m / args.cpu_cols, 1),
                         "ranks_match_on_sample": bool(np.array_equal(np.asarray(cc.ranks).reshape(-1, 3),
                                                                      ranks[:args.cpu_cols].reshape(-1, 3)))})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
