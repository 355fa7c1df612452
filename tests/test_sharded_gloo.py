"""Multi-GPU column sharding (Tucker and ACA stores), host logic on CPU with gloo (world_size 2 and 3).

Each rank wraps an oracle-backed store over its cost-balanced column shard;
ShardedStore must reproduce the single-process products: the forward by a
sum-reduce of the partial y blocks, the adjoint by an all-gather of the shard
rows of z.  (On the GPU box the same class runs DeviceStore shards over NCCL.)
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


class OracleShard:
    """Store-like wrapper (rows / forward / adjoint on torch CPU tensors)."""

    def __init__(self, cc, v=None):
        from oracle import oracle as O
        self.st = O.OracleStore(cc)
        self.rows = self.st.rows
        self.v = v  # ACA: this shard's columns of V (m2 x r)

    def forward(self, x):
        import torch
        y = self.st.forward(x.numpy())
        return torch.from_numpy(np.ascontiguousarray(y))

    def adjoint(self, phi):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self.st.adjoint(phi.numpy())))

    def aca_forward(self, x):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self.st.aca_forward(self.v, x.numpy())))

    def aca_adjoint(self, phi):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self.st.aca_adjoint(self.v, phi.numpy())))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from helpers import ragged_store
    from oracle import oracle as O
    from paper_2103_06393_b200.sharded import ShardedStore, balanced_shards, column_costs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cc = ragged_store((9, 7, 11), 3, 13, 1, 5, seed=42)
        shards = balanced_shards(column_costs(cc.grid_dims, cc.ranks, 2), world)
        c0, c1 = shards[rank]
        off = O.tensor_offsets(cc.grid_dims, cc.ranks)
        sub = O.Compressed(cc.grid_dims, cc.q, c1 - c0, cc.ranks[c0:c1],
                           cc.payload[off[c0 * cc.q]:off[c1 * cc.q]])
        sh = ShardedStore(OracleShard(sub), c0, c1, cc.m)
        assert sh.shards == [tuple(s) for s in shards]
        rng = np.random.default_rng(3)
        x = rng.standard_normal((cc.m, 2)) + 1j * rng.standard_normal((cc.m, 2))
        phi = rng.standard_normal((cc.rows, 2)) + 1j * rng.standard_normal((cc.rows, 2))
        y = sh.forward(torch.from_numpy(x), dst=0)
        ya = sh.forward(torch.from_numpy(x), allreduce=True)
        z = sh.adjoint(torch.from_numpy(phi))
        full = O.OracleStore(cc)
        res = {"rank": rank,
               "ya": float(np.linalg.norm(ya.numpy() - full.forward(x)) / np.linalg.norm(full.forward(x))),
               "z": float(np.linalg.norm(z.numpy() - full.adjoint(phi)) / np.linalg.norm(full.adjoint(phi)))}
        if rank == 0:
            res["y"] = float(np.linalg.norm(y.numpy() - full.forward(x)) / np.linalg.norm(full.forward(x)))
        # ACA store sharded by U columns with the matching columns of V
        m2 = 11
        v = rng.standard_normal((m2, cc.m)) + 1j * rng.standard_normal((m2, cc.m))
        sha = ShardedStore(OracleShard(sub, np.asfortranarray(v[:, c0:c1])), c0, c1, cc.m, shards=shards)
        xa = rng.standard_normal((m2, 2)) + 1j * rng.standard_normal((m2, 2))
        ya = sha.aca_forward(torch.from_numpy(xa), allreduce=True).numpy()
        za = sha.aca_adjoint(torch.from_numpy(phi)).numpy()
        ya_ref = full.aca_forward(v, xa)
        za_ref = full.aca_adjoint(v, phi)
        res["aca_y"] = float(np.linalg.norm(ya - ya_ref) / np.linalg.norm(ya_ref))
        res["aca_z"] = float(np.linalg.norm(za - za_ref) / np.linalg.norm(za_ref))
        out_q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_products_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(world)]
    for r in res:
        assert r["ya"] < 1e-13 and r["z"] < 1e-13
        assert r["aca_y"] < 1e-13 and r["aca_z"] < 1e-13
        if r["rank"] == 0:
            assert r["y"] < 1e-13


def test_balanced_shards():
    from paper_2103_06393_b200.sharded import balanced_shards
    costs = np.array([5, 1, 1, 1, 1, 1, 5, 5, 1, 1], float)
    for world in (1, 2, 3, 4, 8):
        sh = balanced_shards(costs, world)
        assert sh[0][0] == 0 and sh[-1][1] == len(costs)
        assert all(a <= b for a, b in sh) and all(sh[i][1] == sh[i + 1][0] for i in range(world - 1))
    big = np.random.default_rng(0).uniform(1, 2.3, 5000)
    sh = balanced_shards(big, 8)
    loads = [big[a:b].sum() for a, b in sh]
    assert max(loads) / min(loads) < 1.01


def _row_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from helpers import ragged_store
    from oracle import oracle as O
    from paper_2103_06393_b200.sharded import RowShardedStore, component_costs, row_pieces, slice_payload_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = (24, 7, 11)
        cc = ragged_store(dims, 3, 13, 1, 5, seed=43)
        ranks = np.asarray(cc.ranks).reshape(cc.m, cc.q, 3)
        layout = row_pieces(component_costs(dims, ranks, 2), dims[0], world, align=4, min_rows=8)
        m2 = 11
        rng = np.random.default_rng(3)
        v = rng.standard_normal((m2, cc.m)) + 1j * rng.standard_normal((m2, cc.m))
        pieces = []
        for k, a, b in layout[rank]:
            rk, pay = O.pack_tensors([cc.tensor(j, k) for j in range(cc.m)])
            rk = rk.reshape(cc.m, 1, 3)
            sub = O.Compressed((b - a, dims[1], dims[2]), 1, cc.m, rk, slice_payload_rows(dims, rk, pay, a, b))
            pieces.append((k, a, b, OracleShard(sub, np.asfortranarray(v))))
        sh = RowShardedStore(pieces, dims, cc.q, cc.m, layout, m2=m2)
        x = rng.standard_normal((cc.m, 2)) + 1j * rng.standard_normal((cc.m, 2))
        phi = rng.standard_normal((cc.rows, 2)) + 1j * rng.standard_normal((cc.rows, 2))
        xa = rng.standard_normal((m2, 2)) + 1j * rng.standard_normal((m2, 2))
        full = O.OracleStore(cc)

        def rel(a, b):
            return float(np.linalg.norm(a - b) / np.linalg.norm(b))
        y = sh.forward(torch.from_numpy(x), dst=world - 1)
        res = {"rank": rank, "pieces": layout,
               "ya": rel(sh.forward(torch.from_numpy(x), allreduce=True).numpy(), full.forward(x)),
               "z": rel(sh.adjoint(torch.from_numpy(phi)).numpy(), full.adjoint(phi)),
               "y1": rel(sh.forward(torch.from_numpy(x[:, 0]), allreduce=True).numpy(), full.forward(x[:, :1])[:, 0]),
               "aca_y": rel(sh.aca_forward(torch.from_numpy(xa), allreduce=True).numpy(), full.aca_forward(v, xa)),
               "aca_z": rel(sh.aca_adjoint(torch.from_numpy(phi)).numpy(), full.aca_adjoint(v, phi))}
        if rank == world - 1:
            res["y"] = rel(y.numpy(), full.forward(x))
        out_q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_row_sharded_products_gloo(world):
    """RowShardedStore (row-slab pieces) over gloo: forward
    assembled on one rank by point-to-point sends (and on every rank by an
    all-reduce of disjoint rows), adjoint by an all-reduce of the m x p
    partials, ACA products, 1-D inputs; cuts inside components."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(world)]
    if world != 3:  # (3 ranks over q = 3 components cut at the component boundaries)
        assert any(0 < a or b < 24 for lst in res[0]["pieces"] for _, a, b in lst)
    for r in res:
        for key in ("ya", "z", "y1", "aca_y", "aca_z"):
            assert r[key] < 1e-13, (key, r)
        if r["rank"] == world - 1:
            assert r["y"] < 1e-13
