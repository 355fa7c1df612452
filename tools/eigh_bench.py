"""Batched Hermitian eigensolver timing for the compressor's Gram matrices
(cuSOLVER vs MAGMA vs host LAPACK through torch).  python tools/eigh_bench.py"""
import torch, time
a = torch.randn(12, 96, 9216, dtype=torch.complex128, device="cuda")
g = a @ a.conj().transpose(1, 2)
def t(f, n=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("gram ms", t(lambda: a @ a.conj().transpose(1, 2)))
for lib in ("cusolver", "magma"):
    torch.backends.cuda.preferred_linalg_library(lib)
    print(lib, "eigh (12,96,96) ms", t(lambda: torch.linalg.eigh(g)))
torch.backends.cuda.preferred_linalg_library("cusolver")
gc = g.cpu()
print("cpu eigh ms", t(lambda: torch.linalg.eigh(gc)))
g3 = torch.randn(36, 96, 96, dtype=torch.complex128, device="cuda"); g3 = g3 @ g3.conj().transpose(1,2)
print("cusolver eigh (36,96,96) ms", t(lambda: torch.linalg.eigh(g3)))
print("cpu eigh (36) ms", t(lambda: torch.linalg.eigh(g3.cpu())))
