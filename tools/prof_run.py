#!/usr/bin/env python
"""Profiling driver: build a bench store unprofiled, then run exactly one
forward and one adjoint between cudaProfilerStart / Stop, so that
`ncu --profile-from-start off` sees only the product kernels."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--cols", type=int, default=0, help="use only the first N columns (0 = all)")
    ap.add_argument("--cc", action="store_true", help="force the CUDA-core forward (TMB_DISABLE_TC=1)")
    args = ap.parse_args()
    import torch
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.workloads import CONFIGS, bench_store_arrays
    if args.cc:
        os.environ["TMB_DISABLE_TC"] = "1"
    cfg = CONFIGS[args.config]
    m = args.cols or cfg.m
    ranks, pay = bench_store_arrays(cfg, 1234, 0, m)  # bench.py's store (its first m columns)
    s = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, cfg.dtype, 0)
    del pay
    rows = cfg.q * int(np.prod(cfg.grid))
    cdt = torch.complex64 if cfg.dtype == "c64" else torch.complex128
    x = torch.randn((cfg.p, m), dtype=cdt, device="cuda").t()
    phi = torch.randn((cfg.p, rows), dtype=cdt, device="cuda").t()
    s.forward(x)
    s.adjoint(phi)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    s.forward(x)
    s.adjoint(phi)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("prof_run done", cfg.name, "cols", m)


if __name__ == "__main__":
    main()
