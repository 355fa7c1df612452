"""Column and row sharding of a Tucker store across GPUs (one process per GPU).

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

Row (voxel-slab) sharding, the alternative of SURVEY §8e (RowShardedStore,
row_pieces, slice_payload_rows): each rank owns cost-balanced (component,
i1-slab) pieces of the output rows, each a store on its sub-grid with every
column; the forward needs no reduction (the pieces' rows of y are sent to the
destination rank), the adjoint reads only the rank's rows of Phi and
all-reduces the m x p partial z.

The classes are agnostic of the store type (anything with forward / adjoint /
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


def slice_payload_rows(dims, ranks, payload, a, b):
    """The payload of one-component tensors (`ranks`: (ncols, 1, 3), CTC1 layout
    `payload`, numpy or torch) restricted to the i1 rows [a, b): core and
    U2 / U3 unchanged, U1 (n1 x r1, column-major) -> (b - a) x r1.  The
    tensors then describe the same operator on the sub-grid (b - a, n2, n3)."""
    r = np.asarray(ranks, np.int64).reshape(-1, 3)
    n1, n2, n3 = (int(d) for d in dims)
    h = int(b) - int(a)
    if np.any(r[:, 0] > h):
        raise ValueError(f"a slab of {h} i1 rows is below a tensor's rank r1 = {int(r[:, 0].max())}")
    core = r[:, 0] * r[:, 1] * r[:, 2]
    size = core + n1 * r[:, 0] + n2 * r[:, 1] + n3 * r[:, 2]
    off = np.concatenate([[0], np.cumsum(size)])[:-1]
    # source segments per tensor: core, r1 column pieces of U1, then U2 + U3
    nseg = 2 + r[:, 0]
    t_of = np.repeat(np.arange(len(r)), nseg)
    pos = np.arange(int(nseg.sum())) - np.repeat(np.cumsum(nseg) - nseg, nseg)  # segment index inside its tensor
    o, c0, r1 = off[t_of], core[t_of], r[t_of, 0]
    is_core, is_tail = pos == 0, pos == nseg[t_of] - 1
    start = np.where(is_core, o, np.where(is_tail, o + c0 + n1 * r1, o + c0 + (pos - 1) * n1 + int(a)))
    length = np.where(is_core, c0, np.where(is_tail, n2 * r[t_of, 1] + n3 * r[t_of, 2], h))
    total = int(length.sum())
    idx = np.repeat(start - (np.cumsum(length) - length), length) + np.arange(total)
    if isinstance(payload, np.ndarray):
        return payload[idx]
    import torch  # a torch tensor (the bench slices its device payload)
    return payload[torch.from_numpy(idx).to(payload.device)]


class RowShardedStore:
    """One rank's row-slab pieces (the alternative of SURVEY §8e; the C-ABI
    counterpart is TM_SHARD_ROWS) plus the collectives that assemble the
    products.  `pieces`: this rank's [(k, a, b, store)], each store a
    one-component store on the sub-grid (b - a, n2, n3) with every column
    (slice_payload_rows); `layout`: every rank's [(k, a, b)] lists
    (row_pieces).  The forward has no reduction: each rank sends its pieces'
    rows of y to `dst` (or every rank, allreduce=True); the adjoint reads only
    this rank's rows of Phi and all-reduces the m x p partial z."""

    def __init__(self, pieces, dims, q, ncols, layout, group=None, m2=0):
        import torch.distributed as dist

        self.pieces = [(int(k), int(a), int(b), st) for k, a, b, st in pieces]
        self.dims = tuple(int(d) for d in dims)
        self.q, self.ncols, self.m2 = int(q), int(ncols), int(m2)
        self.layout = [[tuple(int(v) for v in pc) for pc in lst] for lst in layout]
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nv = int(np.prod(self.dims))

    @property
    def rows(self):
        return self.q * self.nv

    def _slab(self, t, k, a, b):
        """(p, n2 n3, b - a) view of rows [k n_v, (k + 1) n_v), i1 in [a, b) of a
        column-major (rows x p) tensor."""
        n1, n2, n3 = self.dims
        tt = t.t()[:, k * self.nv:(k + 1) * self.nv]
        return tt.reshape(tt.shape[0], n2 * n3, n1)[:, :, a:b]

    def _assemble(self, outs, p, dtype, device, dst, allreduce):
        import torch
        import torch.distributed as dist

        y = torch.zeros((p, self.rows), dtype=dtype, device=device).t()
        for (k, a, b, _), yk in zip(self.pieces, outs):
            self._slab(y, k, a, b).copy_(yk.t().reshape(p, -1, b - a))
        if self.world == 1:
            return y
        if allreduce:  # rows are disjoint: the sum is the assembly
            dist.all_reduce(y.t(), group=self.group)
            return y
        nccl = dist.get_backend(self.group) == "nccl"
        stage = (lambda t: t) if nccl else (lambda t: t.cpu())  # gloo point-to-point: host tensors
        ops, recv = [], []
        if self.rank == dst:
            for r, lst in enumerate(self.layout):
                if r == dst:
                    continue
                for k, a, b in lst:
                    buf = stage(torch.empty((p, (b - a) * self.nv // self.dims[0]), dtype=dtype, device=device))
                    ops.append(dist.P2POp(dist.irecv, buf, r, self.group))
                    recv.append((k, a, b, buf))
        else:
            for (k, a, b, _), yk in zip(self.pieces, outs):
                ops.append(dist.P2POp(dist.isend, stage(yk.t().contiguous()), dst, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for k, a, b, buf in recv:
            self._slab(y, k, a, b).copy_(buf.to(device).reshape(p, -1, b - a))
        return y

    def _forward(self, x, dst, allreduce, aca):
        import torch

        squeeze = x.dim() == 1
        x2 = x.reshape(-1, 1) if squeeze else x
        outs = [(st.aca_forward(x2) if aca else st.forward(x2)) for *_, st in self.pieces]
        outs = [o.reshape(-1, 1) if o.dim() == 1 else o for o in outs]
        dtype = outs[0].dtype if outs else (x2.dtype if x2.is_complex() else torch.complex128)
        y = self._assemble(outs, x2.shape[1], dtype, x2.device, dst, allreduce)
        return y[:, 0] if squeeze else y

    def forward(self, x, dst=0, allreduce=False):
        """y = Zbc x (x: m x p, replicated): the full y on `dst` (every rank
        with allreduce=True); other ranks get their own rows only."""
        return self._forward(x, dst, allreduce, False)

    def aca_forward(self, x, dst=0, allreduce=False):
        """y = U (V^H x) (x: m2 x p, replicated; every piece store holds V)."""
        return self._forward(x, dst, allreduce, True)

    def _adjoint(self, phi, aca):
        import torch
        import torch.distributed as dist

        squeeze = phi.dim() == 1
        ph = phi.reshape(-1, 1) if squeeze else phi
        p = ph.shape[1]
        z = None
        for k, a, b, st in self.pieces:
            pk = self._slab(ph, k, a, b).reshape(p, -1).t()  # contiguous copy of this piece's rows
            zk = st.aca_adjoint(pk) if aca else st.adjoint(pk)
            zk = zk.reshape(-1, 1) if zk.dim() == 1 else zk
            z = zk.clone() if z is None else z + zk
        if z is None:
            n = self.m2 if aca else self.ncols
            z = torch.zeros((n, p), dtype=ph.dtype, device=ph.device)
        if self.world > 1:
            zt = z.t().contiguous()
            dist.all_reduce(zt, group=self.group)
            z = zt.t()
        return z[:, 0] if squeeze else z

    def adjoint(self, phi):
        """z = Zbc^H phi on every rank (phi: q n_v x p, replicated; each rank
        reads only its rows)."""
        return self._adjoint(phi, False)

    def aca_adjoint(self, phi):
        """z = V (U^H phi) on every rank."""
        return self._adjoint(phi, True)
