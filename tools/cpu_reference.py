#!/usr/bin/env python
"""Measure the REFERENCE's own CPU matvec (oracle/_ref: /root/reference/proj/src
compiled unchanged) on the benched stores, at full size, on this host's cores
— the run_matvec_bench protocol (proj/src/experiments.cpp:504-595: wall clock
around forward and adjoint, timing at :530-535) — and, beside it, the bounded
sample model bench.py's reference arm extrapolates from, so the model's error
is measured, not assumed.

  python tools/cpu_reference.py --configs c1,c2,c3,c5,c4 --out gpurun_out/cpu_full.jsonl

One JSON line per config: full forward / adjoint seconds (median of
--repeats, config 4 once), workers, host, and the sample model's prediction.
The store is exactly bench.py's (workloads.bench_store_arrays, c64-rounded
factors, the reference computes in complex128).
"""
import argparse
import json
import os
import platform
import statistics
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SEED = 1234


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def build_reference(cfg, host, ranks, v, tmpdir):
    from oracle import oracle as O
    from oracle import ref as R
    if v is None:
        return R.RefCC.from_compressed(O.Compressed(cfg.grid, cfg.q, cfg.m, ranks, host))
    path = os.path.join(tmpdir, "store.cta1")
    O.save_cta1(path, O.Aca(cfg.grid, cfg.q, ranks, host, v), 1.0, 0)
    return R.RefAca.load_cta1(path)  # the reference's own CTA1 loader


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c5,c4")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/cpu_full.jsonl")
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--sample-only", default="",
                    help="skip the full run: compare the sample model with the full measurement in this jsonl file")
    args = ap.parse_args()
    import torch
    import bench as B
    from helpers import cn01
    from oracle import ref as R
    from paper_2103_06393_b200.workloads import CONFIGS, bench_store_arrays, synthetic_v

    if not R.available():
        raise SystemExit("oracle/_ref is not built")
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        t0 = time.time()
        ranks, pay = bench_store_arrays(cfg, SEED, device=dev)
        host = (pay.to(torch.complex64).to(torch.complex128) if cfg.dtype == "c64" else pay).cpu().numpy()
        del pay
        v = synthetic_v(cfg, SEED) if cfg.aca_m2 else None
        if v is not None and cfg.dtype == "c64":
            v = v.astype(np.complex64).astype(np.complex128)
        W = args.workers or B.cpu_workers(cfg, 64)
        with tempfile.TemporaryDirectory() as td:
            ref = build_reference(cfg, host, ranks, v, td)
            t_build = time.time() - t0
            rows = cfg.q * int(np.prod(cfg.grid))
            r64 = (lambda a: a.astype(np.complex64).astype(np.complex128)) if cfg.dtype == "c64" else (lambda a: a)
            x = r64(cn01(cfg.aca_m2 or cfg.m, cfg.p, SEED))
            phi = r64(cn01(rows, cfg.p, SEED + 1))
            reps = 1 if name == "c4" else args.repeats
            tf, ta = [], []
            if args.sample_only:
                prev = [json.loads(ln) for ln in open(args.sample_only) if json.loads(ln)["config"] == cfg.name]
                tf, ta, reps = [prev[-1]["forward_s"]], [prev[-1]["adjoint_s"]], 0
            for _ in range(reps):
                s = time.perf_counter()
                y = ref.aca_forward(x, W) if v is not None else ref.forward(x, W)
                tf.append(time.perf_counter() - s)
                del y
                s = time.perf_counter()
                z = ref.aca_adjoint(phi, W) if v is not None else ref.adjoint(phi, W)
                ta.append(time.perf_counter() - s)
                del z
            del ref
        line = {"config": cfg.name, "kind": "reference", "impl": "oracle/_ref (proj/src compiled unchanged)",
                "forward_s": round(statistics.median(tf), 3), "adjoint_s": round(statistics.median(ta), 3),
                "pair_s": round(statistics.median(tf) + statistics.median(ta), 3), "repeats": reps,
                "full_from": args.sample_only or "this run",
                "forward_runs_s": [round(t, 3) for t in tf], "adjoint_runs_s": [round(t, 3) for t in ta],
                "workers": W, "nproc": os.cpu_count(), "cpu": cpu_model(), "store_build_s": round(t_build, 1)}
        # the sample model of bench.py's CPU legs (W and 2W median-cost columns, two-point fits)
        if v is None:
            ncs = min(2 * W, cfg.m)
            samp = B.cpu_sample(cfg, ranks, lambda sel: B.column_payload(cfg, ranks, host, sel), x,
                                np.asfortranarray(phi), ncs, W, kind="reference")
            pred = samp["fwd_s"] + samp["adj_s"]
            line["sample_model"] = {"columns": ncs, "forward_s": round(samp["fwd_s"], 3),
                                    "fwd_fixed_s": round(float(samp["fwd_fixed_s"]), 3),
                                    "adj_fixed_s": round(float(samp.get("adj_fixed_s", 0.0)), 3),
                                    "adjoint_s": round(samp["adj_s"], 3), "pair_s": round(pred, 3),
                                    "rel_error_vs_full": round(pred / line["pair_s"] - 1.0, 4)}
        print(json.dumps(line), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
