#!/usr/bin/env python
"""How does the c64 tensor-core forward's error grow with the column count?
(Diagnostic: linear growth = biased accumulation in the MMA adder.)"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.workloads import Config, column_scales, rank_table, synthetic_payload
    res = []
    for m in (50, 200, 800, 3200):
        for scaled in (False, True):
            cfg = Config("probe", (32, 32, 256), 1, m, "c64", 1, (3.0, 50.0))
            ranks = rank_table(cfg, 5)
            sc = column_scales(cfg, 5) if scaled else np.ones(m)
            pay, _ = synthetic_payload(cfg.grid, ranks, sc, 9, device="cuda")
            p64 = pay.to(torch.complex64).to(torch.complex128)
            s64 = DeviceStore.from_arrays(cfg.grid, 1, ranks, pay, "c64", 0)
            s128 = DeviceStore.from_arrays(cfg.grid, 1, ranks, p64, "c128", 0)
            g = torch.Generator(device="cuda")
            g.manual_seed(3)
            x = torch.randn((1, m), dtype=torch.complex64, device="cuda", generator=g).t()
            yr = s128.forward(x.to(torch.complex128))
            yt = s64.forward(x)
            os.environ["TMB_DISABLE_TC"] = "1"
            yc = s64.forward(x)
            os.environ.pop("TMB_DISABLE_TC")
            n = torch.linalg.vector_norm(yr)
            res.append({"m": m, "scaled": scaled,
                        "tc": float(torch.linalg.vector_norm(yt.to(torch.complex128) - yr) / n),
                        "cc": float(torch.linalg.vector_norm(yc.to(torch.complex128) - yr) / n),
                        "tc_mean_ratio": float((yt.to(torch.complex128).abs().sum() / yr.abs().sum()).real)})
            print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
