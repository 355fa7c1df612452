#!/usr/bin/env python
"""Per-shard timing of the config-4 store at N = 1, 2, 4, 8 on ONE GPU: for
each N, every cost-balanced column shard of bench.py's store
(sharded.balanced_shards) is built and its forward + adjoint timed with CUDA
events — exactly the compute one GPU of an N-GPU run performs.  The step time
of an N-GPU run is then max over shards + the exposed part of the
collectives, modelled at NVLink 5 bandwidth (900 GB/s per direction; the
forward's partial-y reduce runs per component group while the next group
computes, so only the last group's reduce is exposed; the adjoint's z
gather is a few KB).  A projection from measured shard times, NOT a multi-GPU
measurement (this pool has one GPU per box).

--mode rows times the voxel-slab alternative (sharded.row_pieces):
each GPU holds the (component, i1-slab) pieces of its row range as stores on
the sub-grid (all m columns, U1 rows sliced), runs every piece's forward and
adjoint; no forward reduction (each GPU owns its rows of y; gathering them to
one GPU is modelled as the last piece's copy at 900 GB/s), the adjoint
all-reduces the m x p partial z (a few KB).

  python tools/shard_scaling.py --config c4 --out gpurun_out/shard_scaling.jsonl
  python tools/shard_scaling.py --config c4 --mode rows --out gpurun_out/shard_rows.jsonl
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/shard_scaling.jsonl")
    ap.add_argument("--mode", default="columns", choices=["columns", "rows"])
    args = ap.parse_args()
    if args.mode == "rows":
        return rows_mode(args)
    import torch
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.sharded import balanced_shards, column_costs
    from paper_2103_06393_b200.workloads import CONFIGS, bench_store_arrays, rank_table

    cfg = CONFIGS[args.config]
    ranks_all = rank_table(cfg, 1234)
    costs = column_costs(cfg.grid, ranks_all, cfg.p)
    rows = cfg.q * int(np.prod(cfg.grid))
    g = torch.Generator(device="cuda")
    g.manual_seed(1235)
    phi = torch.randn((cfg.p, rows), dtype=torch.complex64, device="cuda", generator=g).t()
    x = torch.randn((cfg.p, cfg.m), dtype=torch.complex64, device="cuda").t()
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    base = None
    for n in [int(v) for v in args.ns.split(",")]:
        shards = balanced_shards(costs, n)
        per = []
        for c0, c1 in shards:
            ranks, pay = bench_store_arrays(cfg, 1234, c0, c1)
            st = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, cfg.dtype, 0)
            del pay
            xs = x[c0:c1]
            st.forward(xs)
            st.adjoint(phi)
            torch.cuda.synchronize()
            tf, ta = [], []
            for _ in range(args.steps):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record()
                st.forward(xs)
                e[1].record()
                st.adjoint(phi)
                e[2].record()
                torch.cuda.synchronize()
                tf.append(e[0].elapsed_time(e[1]))
                ta.append(e[1].elapsed_time(e[2]))
            per.append((statistics.median(tf), statistics.median(ta)))
            del st
            torch.cuda.empty_cache()
        fwd = max(p[0] for p in per)
        adj = max(p[1] for p in per)
        ybytes = rows * cfg.p * 8
        coll = 0.0 if n == 1 else (ybytes / 4) / 900e9 * 1e3 + 0.02  # last of 4 component groups + z gather
        step = fwd + adj + coll
        if base is None:
            base = step
        line = {"config": cfg.name, "n_gpus": n, "shards": shards, "forward_ms_per_shard": [round(p[0], 2) for p in per],
                "adjoint_ms_per_shard": [round(p[1], 2) for p in per], "max_forward_ms": round(fwd, 2),
                "max_adjoint_ms": round(adj, 2), "collective_exposed_ms_model": round(coll, 3),
                "projected_step_ms": round(step, 2), "projected_strong_efficiency": round(base / (n * step), 3),
                "note": "shard compute measured on one B200 (one shard at a time); collectives modelled at 900 GB/s"}
        print(json.dumps(line), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(line) + "\n")


def rows_mode(args):
    import torch
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.sharded import component_costs, row_pieces
    from paper_2103_06393_b200.workloads import CONFIGS, rank_table, synthetic_payload, tensor_scales

    cfg = CONFIGS[args.config]
    n1, n2, n3 = cfg.grid
    ranks = rank_table(cfg, 1234)
    scales = tensor_scales(cfg, 1234)
    cc = component_costs(cfg.grid, ranks, cfg.p)
    r1max = int(ranks[..., 0].max())
    minr = 8 * ((r1max + 7) // 8)
    x = torch.randn((cfg.p, cfg.m), dtype=torch.complex64, device="cuda").t()
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    cache = {}
    base = None
    for n in [int(v) for v in args.ns.split(",")]:
        shards = row_pieces(cc, n1, n, align=8, min_rows=minr)
        per = []
        for pcs in shards:
            tf = ta = 0.0
            for k, a, b in pcs:
                key = (k, b - a)  # piece time depends on the component and the slab height only
                if key not in cache:
                    rk = ranks[:, k:k + 1, :].copy()
                    pay, _ = synthetic_payload((b - a, n2, n3), rk, scales[:, k:k + 1], 77 + k)
                    st = DeviceStore.from_arrays((b - a, n2, n3), 1, rk, pay, cfg.dtype, 0)
                    del pay
                    phi = torch.randn((cfg.p, st.rows), dtype=torch.complex64, device="cuda").t()
                    st.forward(x)
                    st.adjoint(phi)
                    torch.cuda.synchronize()
                    f, g = [], []
                    for _ in range(args.steps):
                        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                        e[0].record()
                        st.forward(x)
                        e[1].record()
                        st.adjoint(phi)
                        e[2].record()
                        torch.cuda.synchronize()
                        f.append(e[0].elapsed_time(e[1]))
                        g.append(e[1].elapsed_time(e[2]))
                    cache[key] = (statistics.median(f), statistics.median(g))
                    del st, phi
                    torch.cuda.empty_cache()
                tf += cache[key][0]
                ta += cache[key][1]
            per.append((tf, ta))
        fwd = max(p[0] for p in per)
        adj = max(p[1] for p in per)
        # gather of the last piece's y rows to the root, z all-reduce ~20 us
        last = max((pcs[-1][2] - pcs[-1][1]) for pcs in shards)
        coll = 0.0 if n == 1 else last * n2 * n3 * cfg.p * 8 / 900e9 * 1e3 + 0.02
        step = fwd + adj + coll
        if base is None:
            base = step
        line = {"config": cfg.name, "mode": "rows", "n_gpus": n, "pieces": shards,
                "forward_ms_per_shard": [round(p[0], 2) for p in per],
                "adjoint_ms_per_shard": [round(p[1], 2) for p in per], "max_forward_ms": round(fwd, 2),
                "max_adjoint_ms": round(adj, 2), "collective_exposed_ms_model": round(coll, 3),
                "projected_step_ms": round(step, 2), "projected_strong_efficiency": round(base / (n * step), 3),
                "note": "piece compute measured on one B200 (one piece at a time); collectives modelled at 900 GB/s"}
        print(json.dumps(line), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
