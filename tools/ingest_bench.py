#!/usr/bin/env python
"""Time the streaming CTC1 ingest (tm_store_load_ctc1) on a
synthetic file with the config-4 grid, and check the loaded store against
one built from the same arrays in memory (bitwise-equal forward products).

  python tools/ingest_bench.py [--cols 400] [--dir /tmp]
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
    ap.add_argument("--cols", type=int, default=400)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--dtype", default="c64")
    args = ap.parse_args()
    import torch
    import paper_2103_06393_b200 as P
    from paper_2103_06393_b200.compress import write_ctc1
    from paper_2103_06393_b200.workloads import CONFIGS, column_scales, rank_table, synthetic_payload
    cfg = CONFIGS["c4"]
    m = args.cols
    ranks = rank_table(cfg, 77)[:m]
    pay, _ = synthetic_payload(cfg.grid, ranks, column_scales(cfg, 77)[:m], 78, device="cuda")
    path = os.path.join(args.dir, "ingest_c4_%d.ctc1" % m)
    write_ctc1(path, cfg.grid, cfg.q, ranks, pay)
    size = os.path.getsize(path)
    ref = P.DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, args.dtype, 0)
    del pay
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        s = P.DeviceStore.load_ctc1(path, args.dtype)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    x = torch.randn((1, m), dtype=torch.complex64 if args.dtype == "c64" else torch.complex128, device="cuda").t()
    same = bool(torch.equal(s.forward(x), ref.forward(x)))
    best = min(times)
    print(json.dumps({"file_bytes": size, "columns": m, "grid": list(cfg.grid), "q": cfg.q, "dtype": args.dtype,
                      "load_s": [round(t, 3) for t in times], "gb_per_s": round(size / best / 1e9, 2),
                      "products_bitwise_equal": same,
                      "note": "file in the page cache after the first load; includes the tensor-core operand build"}))
    os.remove(path)


if __name__ == "__main__":
    main()
