#!/usr/bin/env python
"""Full-size parity evidence for a bench config (default c4) on one GPU.

1. The same seeded synthetic store is built as complex128 and as complex64
   (c64 = the c128 factors rounded once).  The c128 store runs the FP64
   CUDA-core kernels, which are pinned to the CPU oracle at 1e-12 by
   tests/test_gpu_parity.py; it serves as the full-size high-precision
   reference for every c64 kernel variant (relative L2 error, north_star
   tolerance 1e-5).
2. A column-sample check against the CPU oracle itself at full grid size:
   x supported on the first S columns (forward) and z restricted to those
   columns (adjoint), compared with the oracle on an S-column store.
Prints one JSON line.
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
    ap.add_argument("--config", default="c4")
    ap.add_argument("--sample-cols", type=int, default=4)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--chains", default="", help="comma list of TMB_TC_CHAIN values to also check")
    args = ap.parse_args()
    import torch
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200.workloads import CONFIGS, bench_store_arrays, tensor_offsets

    cfg = CONFIGS[args.config]
    ranks, pay = bench_store_arrays(cfg, 1234)  # exactly bench.py's store
    pay64 = pay.to(torch.complex64).to(torch.complex128)  # the c64 store's values, exactly
    s64 = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay, "c64", 0)
    s128 = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks, pay64, "c128", 0)
    S = args.sample_cols
    off = tensor_offsets(cfg.grid, ranks[:S])
    host_sample = pay64[: int(off[-1])].cpu().numpy()
    del pay, pay64
    rows = cfg.q * int(np.prod(cfg.grid))
    rng = np.random.default_rng(7)
    x = ((rng.standard_normal((cfg.m, cfg.p)) + 1j * rng.standard_normal((cfg.m, cfg.p))) / np.sqrt(2)).astype(
        np.complex64)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    phi = torch.randn((cfg.p, rows), dtype=torch.complex64, device="cuda", generator=g).t()
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    out = {"config": cfg.name}

    def rel(a, b):
        return float(torch.linalg.vector_norm((a - b).reshape(-1)) / torch.linalg.vector_norm(b.reshape(-1)))

    t0 = time.time()
    y_ref = s128.forward(xd.to(torch.complex128))
    z_ref = s128.adjoint(phi.to(torch.complex128))
    torch.cuda.synchronize()
    out["c128_seconds"] = round(time.time() - t0, 2)
    os.environ.pop("TMB_DISABLE_TC", None)
    y_tc = s64.forward(xd)   # default path
    z_tc = s64.adjoint(phi)
    os.environ["TMB_DISABLE_TC"] = "1"
    y_cc = s64.forward(xd)
    z_cc = s64.adjoint(phi)
    os.environ.pop("TMB_DISABLE_TC", None)
    torch.cuda.synchronize()
    out["forward_rel_l2_default_vs_c128"] = rel(y_tc.to(torch.complex128), y_ref)
    out["adjoint_rel_l2_default_vs_c128"] = rel(z_tc.to(torch.complex128), z_ref)
    out["forward_rel_l2_cudacore_vs_c128"] = rel(y_cc.to(torch.complex128), y_ref)
    for ch in [c for c in args.chains.split(",") if c]:
        os.environ["TMB_TC_CHAIN"] = ch
        out[f"forward_rel_l2_chain{ch}_vs_c128"] = rel(s64.forward(xd).to(torch.complex128), y_ref)
        os.environ.pop("TMB_TC_CHAIN")
    out["adjoint_rel_l2_cudacore_vs_c128"] = rel(z_cc.to(torch.complex128), z_ref)

    if not args.no_oracle:
        from oracle import oracle as O
        cc = O.Compressed(cfg.grid, cfg.q, S, ranks[:S], host_sample)
        st = O.OracleStore(cc)
        xs = np.zeros((cfg.m, cfg.p), np.complex64)
        xs[:S] = x[:S]
        ys = s64.forward(torch.from_numpy(np.ascontiguousarray(xs.T)).cuda().t()).cpu().numpy()
        yo = st.forward(x[:S].astype(np.complex128), workers=min(S, os.cpu_count() or 1))
        zo = st.adjoint(phi.cpu().numpy().astype(np.complex128), workers=min(S, os.cpu_count() or 1))
        out["oracle_sample_cols"] = S
        out["forward_rel_l2_vs_oracle_sample"] = float(np.linalg.norm(ys - yo) / np.linalg.norm(yo))
        zd = z_tc.cpu().numpy()[:S]
        out["adjoint_rel_l2_vs_oracle_sample"] = float(np.linalg.norm(zd - zo) / np.linalg.norm(zo))
    out["tolerance"] = 1e-5
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
