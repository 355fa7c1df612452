"""Per-phase timing of the GPU compressor (compress.py) on config-4 columns:
field assembly vs Gram matrices vs eigensolves vs core projection.
  python tools/compress_prof.py [--cols 8]"""
import argparse, collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cols", type=int, default=8)
    args = ap.parse_args()
    import torch
    from paper_2103_06393_b200 import compress as C, scenes as S
    acc = collections.defaultdict(float)

    def wrap(mod, name, label):
        f = getattr(mod, name)

        def g(*a, **k):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = f(*a, **k)
            torch.cuda.synchronize()
            acc[label] += time.perf_counter() - t
            return r
        setattr(mod, name, g)
    wrap(C, "assemble_columns", "assemble_columns")
    wrap(torch.linalg, "eigh", "eigh")
    wrap(torch, "einsum", "core einsum")
    g = S.centered_grid(0.001, (192, 224, 256))
    sc = S.close_fitting_array(g, 0.006, channels=8, loops_per_channel=4, segs_per_loop=156, q=12)
    sub = type(sc)(sc.origin, sc.spacing, sc.dims, sc.sources[:args.cols], sc.op, sc.k0, sc.q)
    C.compress_scene(type(sc)(sc.origin, sc.spacing, sc.dims, sc.sources[:1], sc.op, sc.k0, sc.q), 1e-4)
    acc.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    C.compress_scene(sub, 1e-4)
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
    print("total %.3f s for %d columns (%.1f ms/column)" % (tt, args.cols, 1e3 * tt / args.cols))
    for k, v in sorted(acc.items(), key=lambda x: -x[1]):
        print("  %-18s %.3f s" % (k, v))


if __name__ == "__main__":
    main()
