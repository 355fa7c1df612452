"""Column sharding of a Tucker store across GPUs (one process per GPU).

The reference parallelises products over columns with host threads
(stacked_forward's per-worker partials, src/matvec.cpp:28-59; stacked_adjoint's
per-column rows, :78-96).  Here each rank of a torch.distributed process group
owns a contiguous, cost-balanced range of columns (all q components of each)
as its own DeviceStore, and the products exchange data only where the
algorithm has a real exchange step:

  forward  y = sum_ranks Zbc[:, shard] x[shard]    -> NCCL reduce (or all-reduce)
                                                      of the q*n_v x p partial
  adjoint  z[shard] = Zbc[:, shard]^H phi          -> NCCL all-gather of the
                                                      r-row blocks (m x p total)

An ACA store (Zbc ~ U V^H, aca_forward / aca_adjoint, src/matvec.cpp:150-175)
shards the r_c U columns with the matching columns of V:

  aca_forward  y = sum_ranks U[:, l] (V[:, l]^H x)  -> reduce, as the forward
  aca_adjoint  z = sum_ranks V[:, l] (U[:, l]^H phi) -> all-reduce of m2 x p

The class is agnostic of the store type (anything with forward / adjoint /
rows / ncols), which lets the CPU tests drive the same host logic with gloo.
"""
from __future__ import annotations

import numpy as np


def balanced_shards(costs, world, align=1):
    """Contiguous [begin, end) column ranges with near-equal total cost.

    costs: per-column cost (e.g. reconstruct_madds + accumulate madds);
    boundaries are multiples of `align` (except the last)."""
    costs = np.asarray(costs, np.float64)
    m = len(costs)
    pref = np.concatenate([[0.0], np.cumsum(costs)])
    bounds = [0]
    for r in range(1, world):
        target = pref[-1] * r / world
        b = int(np.searchsorted(pref, target))
        b = int(round(b / align) * align) if align > 1 else b
        b = min(max(b, bounds[-1]), m)
        bounds.append(b)
    bounds.append(m)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def row_pieces(comp_costs, n1, world, align=8, min_rows=8):
    """Row (voxel-slab) sharding, the alternative of SURVEY §8e: the q * n1
    (component, i1) slabs of the output are cut into `world` contiguous
    ranges of near-equal cost (a slab of component k costs comp_costs[k] / n1:
    every stage of the product is linear in the i1 rows).  Cuts inside a
    component fall on multiples of `align` rows and leave at least
    `min_rows` rows on both sides (a piece is a Tucker store on the sub-grid
    i1 in [a, b), so it needs b - a >= r1 of its tensors); otherwise they
    move to the nearer component boundary.  Returns, per shard, a list of
    pieces (k, a, b) — component k, i1 rows [a, b)."""
    cc = np.asarray(comp_costs, np.float64)
    q = len(cc)
    n1 = int(n1)
    step = max(int(align), 1)
    lo = max(int(min_rows), step)
    pref = np.concatenate([[0.0], np.cumsum(cc)])
    cuts = [0]
    for s in range(1, world):
        target = pref[-1] * s / world
        k = int(np.clip(np.searchsorted(pref, target, side="right") - 1, 0, q - 1))
        frac = (target - pref[k]) / cc[k] if cc[k] > 0 else 0.0
        loc = int(round(frac * n1 / step)) * step
        if loc < lo or n1 - loc < lo:
            loc = 0 if frac < 0.5 else n1
        cuts.append(max(cuts[-1], min(k * n1 + loc, q * n1)))
    cuts.append(q * n1)
    out = []
    for s in range(world):
        r0, r1 = cuts[s], cuts[s + 1]
        pcs = []
        while r0 < r1:
            k = r0 // n1
            e = min(r1, (k + 1) * n1)
            pcs.append((k, r0 - k * n1, e - k * n1))
            r0 = e
        out.append(pcs)
    return out


def component_costs(dims, ranks, p=1):
    """Per-component madds of one product: sum_j reconstruct_madds + m n_v p."""
    r = np.asarray(ranks, np.int64)
    n1, n2, n3 = (int(d) for d in dims)
    dec = n1 * r[..., 0] * r[..., 1] * r[..., 2] + n1 * n2 * r[..., 1] * r[..., 2] + n1 * n2 * n3 * r[..., 2]
    return dec.sum(axis=0) + r.shape[0] * n1 * n2 * n3 * p


def column_costs(dims, ranks, p=1):
    """Per-column madds of one product: sum_k reconstruct_madds + q n_v p."""
    r = np.asarray(ranks, np.int64)
    n1, n2, n3 = (int(d) for d in dims)
    dec = n1 * r[..., 0] * r[..., 1] * r[..., 2] + n1 * n2 * r[..., 1] * r[..., 2] + n1 * n2 * n3 * r[..., 2]
    return dec.sum(axis=1) + r.shape[1] * n1 * n2 * n3 * p


class ShardedStore:
    """One rank's column shard plus the collectives that assemble products."""

    def __init__(self, store, col_begin, col_end, ncols_total, group=None, shards=None):
        import torch.distributed as dist

        self.store = store
        self.c0, self.c1 = int(col_begin), int(col_end)
        self.ncols = int(ncols_total)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if shards is None:
            shards = [None] * self.world
            if self.world > 1:
                dist.all_gather_object(shards, (self.c0, self.c1), group=group)
            else:
                shards = [(self.c0, self.c1)]
        self.shards = [tuple(s) for s in shards]
        self.max_cols = max(b - a for a, b in self.shards)

    @property
    def rows(self):
        return self.store.rows

    def forward(self, x, dst=0, allreduce=False, groups=4):
        """y = Zbc x.  x: (ncols x p) on this rank's device (the full block or
        just this shard's rows).  Returns the full y on `dst` (or every rank
        with allreduce=True); other ranks get their partial.

        With N > 1 and a device store the forward runs in `groups` component
        groups (tm_forward_components) and each group's rows of the partial y
        are reduced asynchronously as soon as the group is done, so the
        reduce of group g overlaps the computation of group g + 1 (only the
        last group's reduce is exposed)."""
        xs = x[self.c0:self.c1] if x.shape[0] == self.ncols else x
        if self.world == 1 or not hasattr(self.store, "forward_components") or groups <= 1:
            return self._sum(self.store.forward(xs), dst, allreduce)
        import torch
        import torch.distributed as dist

        squeeze = xs.dim() == 1
        x2 = xs.reshape(-1, 1) if squeeze else xs
        q, nv, p = self.store.q, self.store.num_voxels, x2.shape[1]
        dt = torch.complex64 if self.store.np_dtype == np.complex64 else torch.complex128
        y = torch.empty((p, q * nv), dtype=dt, device=x2.device).t()
        bounds = [round(q * g / groups) for g in range(groups + 1)]
        handles = []
        for k0, k1 in zip(bounds, bounds[1:]):
            if k1 <= k0:
                continue
            self.store.forward_components(x2, k0, k1, y)
            for c in range(p):  # rows [k0 nv, k1 nv) of column c: contiguous
                seg = y.t()[c, k0 * nv:k1 * nv]
                handles.append(dist.all_reduce(seg, group=self.group, async_op=True) if allreduce else
                               dist.reduce(seg, dst=dst, group=self.group, async_op=True))
        for h in handles:
            h.wait()
        return y[:, 0] if squeeze else y

    def _sum(self, y, dst=0, allreduce=False):
        import torch.distributed as dist

        if self.world > 1:
            # column-major (rows x p) blocks are contiguous as their transpose
            buf = y if y.is_contiguous() else y.t()
            if allreduce:
                dist.all_reduce(buf, group=self.group)
            else:
                dist.reduce(buf, dst=dst, group=self.group)
        return y

    def aca_forward(self, x, dst=0, allreduce=False):
        """y = U (V^H x) of an ACA store sharded by U columns (this rank's
        store holds its U columns and the matching columns of V).  x: (m2 x
        p), replicated.  The full y on `dst` (every rank with allreduce)."""
        return self._sum(self.store.aca_forward(x), dst, allreduce)

    def aca_adjoint(self, phi):
        """z = V (U^H phi) on every rank: the shards' V[:, l] (U[:, l]^H phi)
        partials (m2 x p each) summed by an all-reduce."""
        return self._sum(self.store.aca_adjoint(phi), allreduce=True)

    def adjoint(self, phi):
        """z = Zbc^H phi on every rank.  phi: (q n_v x p), replicated."""
        import torch
        import torch.distributed as dist

        z = self.store.adjoint(phi)
        if self.world == 1:
            return z
        squeeze = z.dim() == 1
        zz = z.reshape(z.shape[0], -1)
        p = zz.shape[1]
        pad = torch.zeros((self.max_cols, p), dtype=zz.dtype, device=zz.device)
        pad[: zz.shape[0]] = zz
        full = torch.empty((self.world * self.max_cols, p), dtype=zz.dtype, device=zz.device)
        dist.all_gather_into_tensor(full, pad.contiguous(), group=self.group)
        parts = [full[r * self.max_cols: r * self.max_cols + (b - a)] for r, (a, b) in enumerate(self.shards)]
        out = torch.cat(parts, 0)
        return out[:, 0] if squeeze else out
