"""GPU Tucker-ACA (Algorithm 3).

Restates tucker_aca (src/aca.cpp:126-232) with every heavy step on the
device: the accepted U columns are HOSVD-compressed on the GPU (compress.py),
residual rows come from batched element() on the growing compressed store
(tm_rows, src/tensor.cpp:183-196), and the residual column update and the
Frobenius-norm estimate run through the store's own forward / adjoint
products at p = 1 (src/aca.cpp:197-208) — the hot-path kernels of this
library, on a complex128 store (the reference's arithmetic).  Row and
column providers evaluate the scene's field kernels on the device
(coupling_oracle, src/aca.cpp:246-273).

Control flow (pivoting, zero-pivot skips, the noise floor, convergence test
|x||y| <= eps sqrt(s)) follows the reference step for step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import compress as C

_ZERO_PIVOT = 1e-300
_NOISE_FLOOR = 1e-14


@dataclass
class TuckerAca:
    """AcaFactors with Tucker-compressed U (include/tuckmat/aca.hpp:24-41):
    ranks (r_c, q, 3), payload (device, CTC1 tensor layout [l][comp]),
    v (m2 x r_c, device)."""
    grid_dims: tuple
    q: int
    ranks: np.ndarray
    payload: object
    v: object
    eps: float
    hosvd_eps: float
    converged: bool
    final_stat: float

    @property
    def rank(self):
        return int(self.ranks.shape[0])

    def store(self, dtype="c64", device=0):
        from .matvec import DeviceStore
        return DeviceStore.from_arrays(self.grid_dims, self.q, self.ranks, self.payload, dtype, device, v=self.v)


def device_rows(scene, rows, device="cuda"):
    """Rows of the coupling matrix (all sources) at global row indices:
    (len(rows), m) complex128 — the row provider of coupling_oracle."""
    import torch
    nv = scene.num_voxels
    n1, n2, _ = scene.dims
    out = []
    for i in rows:
        comp, v = divmod(int(i), nv)
        i1, i2, i3 = v % n1, (v // n1) % n2, v // (n1 * n2)
        sub = type(scene)(scene.origin + scene.spacing * np.array([i1, i2, i3], float), scene.spacing, (1, 1, 1),
                          scene.sources, scene.op, scene.k0, scene.q)
        out.append(C.assemble_columns(sub, range(scene.num_sources), device)[:, comp, 0])
    return torch.stack(out)


def tucker_aca(scene, eps=1e-3, hosvd_eps=0.0, device=0, trace=None):
    """tucker_aca (src/aca.cpp:126-232) on the device for a scene.  `trace`,
    if a list, receives (k, pivot row i, pivot column j, |x|, |y|, s) per step."""
    import torch
    from .matvec import DeviceStore
    if not 0.0 < eps < 1.0:
        raise ValueError("aca: eps must lie in (0,1)")
    if hosvd_eps <= 0.0:
        hosvd_eps = min(3.0 * eps, 0.99)  # src/aca.cpp:129
    dev = f"cuda:{device}"
    q, dims = scene.q, tuple(int(d) for d in scene.dims)
    nv = int(np.prod(dims))
    m1, m2 = q * nv, scene.num_sources
    kmax = min(m1, m2)
    n1, n2, n3 = dims
    ranks, parts, vs = [], [], []
    used = torch.zeros(m1, dtype=torch.bool, device=dev)
    i, s, row_scale = 0, 0.0, 0.0
    converged, final_stat = False, 0.0
    store = None
    for k in range(kmax):
        exhausted = False
        while True:
            r = device_rows(scene, [i], dev)[0]
            row_scale = max(row_scale, float(r.abs().max()))
            if k > 0:
                t = torch.from_numpy(store.row_block([i])[0]).to(dev)  # element() of every stored U column
                r = r - t @ torch.stack(vs).conj()
            j = int(torch.argmax(r.abs()))
            if float(r[j].abs()) > max(_ZERO_PIVOT, _NOISE_FLOOR * row_scale):
                break
            if k > 0:
                exhausted = True
                break
            used[i] = True
            free = torch.nonzero(~used)
            if free.numel() == 0:
                exhausted = True
                break
            i = int(free[0])
        if exhausted:
            converged, final_stat = True, 0.0
            break
        y = (r / r[j]).conj()
        x = C.assemble_columns(scene, [j], dev).reshape(-1)
        if k > 0:
            V = torch.stack(vs, dim=1)  # m2 x k
            x = x - store.forward(V[j, :].conj().reshape(-1, 1).contiguous())[:, 0]
        nx, ny = float(torch.linalg.vector_norm(x)), float(torch.linalg.vector_norm(y))
        s += (nx * ny) ** 2
        if k > 0:
            s += 2.0 * float((store.adjoint(x.reshape(-1, 1).contiguous())[:, 0] * (V.conj().T @ y)).real.sum())
        if trace is not None:
            trace.append((k, i, j, nx, ny, s))
        res = C.hosvd_batch(x.reshape(q, n3, n2, n1), hosvd_eps)
        for core, u1, u2, u3 in res:
            ranks.append((u1.shape[1], u2.shape[1], u3.shape[1]))
            parts += [core.reshape(-1), u1.t().reshape(-1), u2.t().reshape(-1), u3.t().reshape(-1)]
        vs.append(y)
        store = DeviceStore.from_arrays(dims, q, np.array(ranks, np.int32), torch.cat(parts), "c128", device)
        scale = math.sqrt(max(s, 0.0))
        final_stat = nx * ny / scale if scale > 0 else 0.0
        if nx * ny <= eps * scale:
            converged = True
            break
        used[i] = True
        ax = x.abs()
        ax[used] = 0.0
        i = int(torch.argmax(ax))
    rc = len(vs)
    v = torch.stack(vs, dim=1) if rc else torch.zeros((m2, 0), dtype=torch.complex128, device=dev)
    payload = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.complex128, device=dev)
    return TuckerAca(dims, q, np.array(ranks, np.int32).reshape(rc, q, 3), payload, v, eps, hosvd_eps, converged,
                     final_stat)
