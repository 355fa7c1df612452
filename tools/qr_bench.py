import torch, time
def t(f, n=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
for n in (96, 256):
    y = torch.randn(96, n, 32, dtype=torch.complex128, device="cuda")
    g = torch.randn(96, n, n, dtype=torch.complex128, device="cuda"); g = g @ g.conj().transpose(1, 2)
    print(n, "qr (96,n,32) ms", t(lambda: torch.linalg.qr(y)))
    print(n, "householder_product path ms", t(lambda: torch.geqrf(y)))
    print(n, "eigh (96,n,n) ms", t(lambda: torch.linalg.eigh(g), 2))
    print(n, "gemm g@y ms", t(lambda: g @ y))
