"""Multi-GPU column sharding at the C ABI (tm_comm_* / tm_sharded_*) on the
one GPU of the test box: a real single-rank NCCL communicator ([0]) and an
emulated three-shard communicator ([0, 0, 0]: the collectives become
device-local copies / adds, every other part of the sharded path — cost-
balanced column split, per-shard stores, per-component completion events,
reduce / broadcast / gather order, host and device I/O — runs as on 8 GPUs).
Results vs the CPU oracle at the north_star tolerances."""
import numpy as np
import pytest

from conftest import rel
from helpers import cn01, ragged_store

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}


def _r(a, dtype):
    return a.astype(np.complex64).astype(np.complex128) if dtype == "c64" else a


@pytest.mark.parametrize("devices", [[0], [0, 0, 0]])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("dims,q,m,p", [((16, 12, 40), 3, 17, 1), ((64, 64, 64), 12, 10, 3), ((9, 5, 7), 1, 2, 2)])
def test_sharded_products(oracle, product, devices, dtype, dims, q, m, p):
    import torch
    from paper_2103_06393_b200.multigpu import Comm, ShardedDeviceStore
    O = oracle
    cc = ragged_store(dims, q, m, 2, 9, seed=m + q)
    comm = Comm(devices)
    assert comm.emulated == (len(set(devices)) != len(devices))
    ss = ShardedDeviceStore.from_compressed(comm, cc, dtype)
    rng = ss.shard_ranges
    assert rng[0][0] == 0 and rng[-1][1] == m and all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
    ref = O.OracleStore(cc.rounded_c64() if dtype == "c64" else cc)
    x = _r(cn01(m, p, 1), dtype)
    phi = _r(cn01(cc.rows, p, 2), dtype)
    yo, zo = ref.forward(x), ref.adjoint(phi)
    # host buffers
    ops = {}
    assert rel(ss.forward(x, ops), yo) <= TOL[dtype]
    assert rel(ss.adjoint(phi), zo) <= TOL[dtype]
    d = ref.opcounts(p)
    assert ops["decompress_madds"] == d[0] and ops["accumulate_madds"] == d[1]
    # device buffers on the root, twice (the second call reuses every work buffer)
    td = torch.complex64 if dtype == "c64" else torch.complex128
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).to(td).cuda().t()
    pd = torch.from_numpy(np.ascontiguousarray(phi.T)).to(td).cuda().t()
    for _ in range(2):
        y = ss.forward(xd)
        z = ss.adjoint(pd)
        torch.cuda.synchronize()
        assert rel(y.cpu().numpy(), yo) <= TOL[dtype]
        assert rel(z.cpu().numpy(), zo) <= TOL[dtype]


@pytest.mark.parametrize("devices", [[0], [0, 0]])
def test_sharded_aca(oracle, product, devices):
    from paper_2103_06393_b200.multigpu import Comm, ShardedDeviceStore
    O = oracle
    cc = ragged_store((20, 18, 30), 3, 9, 2, 6, seed=4)
    rng = np.random.default_rng(4)
    v = rng.standard_normal((23, 9)) + 1j * rng.standard_normal((23, 9))
    fac = O.Aca(cc.grid_dims, cc.q, cc.ranks, cc.payload, v)
    comm = Comm(devices)
    ss = ShardedDeviceStore.from_arrays(comm, fac.grid_dims, fac.q, fac.ranks, fac.payload, "c128", v=v)
    x = cn01(23, 2, 5)
    phi = cn01(fac.rows, 2, 6)
    assert rel(ss.aca_forward(x), O.aca_forward(fac, x)) <= 1e-12
    assert rel(ss.aca_adjoint(phi), O.aca_adjoint(fac, phi)) <= 1e-12


def test_forward_components(oracle, product):
    """tm_forward_components: component ranges of the forward write exactly
    their rows (tensor-core and CUDA-core paths)."""
    import torch
    P = product
    for dtype, dims in (("c64", (40, 36, 64)), ("c128", (9, 10, 11))):
        cc = ragged_store(dims, 12, 7, 2, 8, seed=3)
        ds = P.DeviceStore.from_compressed(cc, dtype)
        td = torch.complex64 if dtype == "c64" else torch.complex128
        x = torch.from_numpy(np.ascontiguousarray(_r(cn01(7, 2, 1), dtype).T)).to(td).cuda().t()
        full = ds.forward(x)
        nv = ds.num_voxels
        y = torch.full((2, ds.rows), 7.0 + 0j, dtype=td, device="cuda").t()
        ds.forward_components(x, 3, 8, y)
        torch.cuda.synchronize()
        # (the waves of a component range split their final partial wave
        # differently, so the c64 partial sums may round differently)
        tol = 1e-6 if dtype == "c64" else 1e-14

        def trel(a, b):
            return float(torch.linalg.vector_norm((a - b).reshape(-1)) / torch.linalg.vector_norm(b.reshape(-1)))
        assert trel(y[3 * nv:8 * nv], full[3 * nv:8 * nv]) <= tol
        assert bool((y[:3 * nv] == 7.0).all()) and bool((y[8 * nv:] == 7.0).all())
        for k0, k1 in ((0, 4), (4, 9), (9, 12)):
            ds.forward_components(x, k0, k1, y)
        torch.cuda.synchronize()
        assert trel(y, full) <= tol


def _overlap_worker(rank, world, port, path, out):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2103_06393_b200 as P
    from oracle import oracle as O
    from paper_2103_06393_b200.sharded import ShardedStore, balanced_shards, column_costs
    cc = O.load_ctc1(path)
    shards = balanced_shards(column_costs(cc.grid_dims, cc.ranks, 1), world)
    c0, c1 = shards[rank]
    off = O.tensor_offsets(cc.grid_dims, np.asarray(cc.ranks).reshape(-1, 3))
    sub = O.Compressed(cc.grid_dims, cc.q, c1 - c0, np.asarray(cc.ranks)[c0:c1],
                       cc.payload[off[c0 * cc.q]:off[c1 * cc.q]])
    ds = P.DeviceStore.from_compressed(sub, "c64", 0)
    sh = ShardedStore(ds, c0, c1, cc.m, shards=shards)
    x = torch.from_numpy(np.ascontiguousarray(cn01(cc.m, 2, 9).astype(np.complex64).T)).cuda().t()
    y = sh.forward(x, dst=0)  # component groups, async reduces
    if rank == 0:
        np.save(out, y.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_forward_overlaps_component_reduces(oracle, product, tmp_path):
    """sharded.py (one process per GPU, here two ranks on one GPU over gloo —
    a functional check): the forward in component groups with asynchronous
    per-group reduces equals the oracle's product."""
    import socket
    import torch.multiprocessing as mp
    O = oracle
    cc = ragged_store((32, 20, 64), 12, 9, 2, 7, seed=12)
    path = str(tmp_path / "s.ctc1")
    O.save_ctc1(path, cc)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "y.npy")
    mp.spawn(_overlap_worker, args=(2, port, path, out), nprocs=2, join=True)
    y = np.load(out)
    x = cn01(cc.m, 2, 9).astype(np.complex64).astype(np.complex128)
    assert rel(y, O.OracleStore(cc.rounded_c64()).forward(x)) <= 1e-5
