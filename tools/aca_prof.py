"""Per-phase timing of the GPU Tucker-ACA on the config-3 geometry (which
step dominates: HOSVD eigensolves, store rebuilds, products).  python tools/aca_prof.py"""
import sys, time, collections, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2103_06393_b200 import aca as A, compress as C, scenes as S, matvec as M
acc = collections.defaultdict(float); cnt = collections.Counter()
def wrap(obj, name, label):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); acc[label] += time.perf_counter() - t; cnt[label] += 1
        return r
    setattr(obj, name, g)
wrap(A, "device_rows", "device_rows")
wrap(C, "assemble_columns", "assemble_columns(all)")
wrap(C, "hosvd_batch", "hosvd_batch")
wrap(M.DeviceStore, "from_arrays", "store_build")
for n in ("forward", "adjoint", "row_block"):
    f = getattr(M.DeviceStore, n)
    def mk(f, n):
        def g(self, *a, **k):
            torch.cuda.synchronize(); t = time.perf_counter()
            r = f(self, *a, **k)
            torch.cuda.synchronize(); acc[n] += time.perf_counter() - t; cnt[n] += 1
            return r
        return g
    setattr(M.DeviceStore, n, mk(f, n))
grid = S.centered_grid(0.002, (96, 96, 96))
sc3 = S.birdcage(grid, 0.30, 0.40, rungs=16, segs_per_rung=128, ring_segs=0, q=12)
t0 = time.perf_counter()
fac = A.tucker_aca(sc3, 1e-4)
tt = time.perf_counter() - t0
print("total", round(tt, 2), "rank", fac.rank)
for k, v in sorted(acc.items(), key=lambda x: -x[1]): print(f"{k:25s} {v:8.2f} s  calls {cnt[k]}")
