#!/usr/bin/env python
"""Time the tensor-core forward / adjoint on a column slice of a config
store under diagnostic switches (TMB_TC_DEBUG, TMB_TC_CHAIN): which pipeline
stage bounds the kernel.  Prints one JSON line per setting."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--cols", type=int, default=400)
    ap.add_argument("--settings", default="0,1,2,3")
    ap.add_argument("--reps", type=int, default=11)
    args = ap.parse_args()
    import torch
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.workloads import CONFIGS, column_scales, rank_table, synthetic_payload
    cfg = CONFIGS[args.config]
    m = args.cols
    ranks = rank_table(cfg, 1234)[:m]
    pay, _ = synthetic_payload(cfg.grid, ranks, column_scales(cfg, 1234)[:m], 2234, device="cuda")
    s = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, cfg.dtype, 0)
    del pay
    rows = cfg.q * int(np.prod(cfg.grid))
    x = torch.randn((1, m), dtype=torch.complex64, device="cuda").t()
    phi = torch.randn((1, rows), dtype=torch.complex64, device="cuda").t()
    dec, acc = s.opcounts(1)
    flops = 8.0 * (dec + acc)
    for st in args.settings.split(","):
        os.environ["TMB_TC_DEBUG"] = st
        for name, fn in (("forward", lambda: s.forward(x)), ("adjoint", lambda: s.adjoint(phi))):
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[len(ts) // 2]
            print(json.dumps({"debug": st, "op": name, "cols": m, "ms": round(ms, 3), "ms_min": round(ts[0], 3),
                              "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
                              "tflops_best": round(flops / (ts[0] * 1e-3) / 1e12, 1)}), flush=True)
    os.environ.pop("TMB_TC_DEBUG")


if __name__ == "__main__":
    main()
