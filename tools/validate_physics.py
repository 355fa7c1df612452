#!/usr/bin/env python
"""Parity on physics-compressed stores at config-4 grid size: the first N
columns of the close-fitting-array scene (192x224x256, 1 mm, PWL q = 12) are
compressed on the GPU (compress.py), loaded as complex64 (tensor-core path)
and complex128 (FP64 path, pinned to the oracle at 1e-12 by the tests), and
the products compared (relative L2, tolerance 1e-5).  A few whole columns
of the operator are also checked against direct kernel evaluation
(assemble_columns): the compression error, at the eps level.  Prints one JSON line."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cols", type=int, default=96)
    ap.add_argument("--case", default="c4")
    args = ap.parse_args()
    import torch
    from compress_bench import scene_for
    from paper_2103_06393_b200 import DeviceStore
    from paper_2103_06393_b200 import compress as C
    sc, eps = scene_for(args.case)
    sub = type(sc)(sc.origin, sc.spacing, sc.dims, sc.sources[:args.cols], sc.op, sc.k0, sc.q)
    ranks, payload = C.compress_scene(sub, eps)
    p64 = payload.to(torch.complex64).to(torch.complex128)
    s64 = DeviceStore.from_arrays(sc.dims, sc.q, ranks, payload, "c64", 0)
    s128 = DeviceStore.from_arrays(sc.dims, sc.q, ranks, p64, "c128", 0)
    rel = lambda a, b: float(torch.linalg.vector_norm((a - b).reshape(-1)) / torch.linalg.vector_norm(b.reshape(-1)))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn((1, args.cols), dtype=torch.complex64, device="cuda", generator=g).t()
    phi = torch.randn((1, sub.rows), dtype=torch.complex64, device="cuda", generator=g).t()
    y64, y128 = s64.forward(x), s128.forward(x.to(torch.complex128))
    z64, z128 = s64.adjoint(phi), s128.adjoint(phi.to(torch.complex128))
    # whole columns vs the uncompressed kernel: the compression error itself
    # (HOSVD guarantees |T - T~|_F <= eps |T|_F per tensor)
    colerr = []
    for j in (0, args.cols // 2, args.cols - 1):
        e = torch.zeros((args.cols, 1), dtype=torch.complex128, device="cuda")
        e[j] = 1.0
        colerr.append(rel(s128.forward(e).reshape(-1), C.assemble_columns(sub, [j]).reshape(-1)))
    out = {"case": args.case, "grid": list(sc.dims), "q": sc.q, "cols": args.cols, "eps": eps,
           "mean_ranks": [round(float(v), 2) for v in ranks.reshape(-1, 3).mean(0)],
           "forward_rel_l2_c64_tensorcore_vs_c128": rel(y64.to(torch.complex128), y128),
           "adjoint_rel_l2_c64_tensorcore_vs_c128": rel(z64.to(torch.complex128), z128),
           "columns_rel_l2_compressed_vs_kernel": colerr, "tolerance": 1e-5}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
