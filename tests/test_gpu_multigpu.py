"""Multi-GPU sharding at the C ABI (tm_comm_* / tm_sharded_*), by columns and
by row slabs (TM_SHARD_ROWS), on the one GPU of the test box: a real single-rank NCCL communicator ([0]) and an
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


def _check_pieces(ss, cc, ndev):
    """rows mode: the pieces tile the q * n1 slabs in shard order."""
    n1 = cc.grid_dims[0]
    got = [(k * n1 + a, k * n1 + b) for _, k, a, b in ss.pieces]
    assert got[0][0] == 0 and got[-1][1] == cc.q * n1
    assert all(x[1] == y[0] for x, y in zip(got, got[1:]))
    assert [d for d, *_ in ss.pieces] == sorted(d for d, *_ in ss.pieces)
    assert all(0 <= d < ndev for d, *_ in ss.pieces)


@pytest.mark.parametrize("mode", ["columns", "rows"])
@pytest.mark.parametrize("devices", [[0], [0, 0, 0]])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("dims,q,m,p", [((16, 12, 40), 3, 17, 1), ((64, 64, 64), 12, 10, 3), ((9, 5, 7), 1, 2, 2)])
def test_sharded_products(oracle, product, mode, devices, dtype, dims, q, m, p):
    import torch
    from paper_2103_06393_b200.multigpu import Comm, ShardedDeviceStore
    O = oracle
    cc = ragged_store(dims, q, m, 2, 9, seed=m + q)
    comm = Comm(devices)
    assert comm.emulated == (len(set(devices)) != len(devices))
    ss = ShardedDeviceStore.from_compressed(comm, cc, dtype, mode=mode)
    rng = ss.shard_ranges
    end = m if mode == "columns" else q * dims[0]
    assert rng[0][0] == 0 and rng[-1][1] == end and all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
    if mode == "rows":
        _check_pieces(ss, cc, len(devices))
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


@pytest.mark.parametrize("mode", ["columns", "rows"])
@pytest.mark.parametrize("devices", [[0], [0, 0]])
def test_sharded_aca(oracle, product, devices, mode):
    from paper_2103_06393_b200.multigpu import Comm, ShardedDeviceStore
    O = oracle
    cc = ragged_store((20, 18, 30), 3, 9, 2, 6, seed=4)
    rng = np.random.default_rng(4)
    v = rng.standard_normal((23, 9)) + 1j * rng.standard_normal((23, 9))
    fac = O.Aca(cc.grid_dims, cc.q, cc.ranks, cc.payload, v)
    comm = Comm(devices)
    ss = ShardedDeviceStore.from_arrays(comm, fac.grid_dims, fac.q, fac.ranks, fac.payload, "c128", v=v, mode=mode)
    x = cn01(23, 2, 5)
    phi = cn01(fac.rows, 2, 6)
    assert rel(ss.aca_forward(x), O.aca_forward(fac, x)) <= 1e-12
    assert rel(ss.aca_adjoint(phi), O.aca_adjoint(fac, phi)) <= 1e-12


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0, 0]])
def test_row_sharding_slabs_inside_components(oracle, product, devices):
    """Row sharding whose cuts fall inside components (a 64-row grid, q = 3,
    low ranks: pieces of 8..56 i1 rows), c64 on the tensor cores: host and
    strided device I/O, OpCounts equal to the unsharded store's, a device
    with several pieces (partial adjoints summed on the device)."""
    import torch
    from paper_2103_06393_b200.multigpu import Comm, ShardedDeviceStore
    O = oracle
    cc = ragged_store((64, 40, 256), 3, 12, 1, 6, seed=21)
    comm = Comm(devices)
    ss = ShardedDeviceStore.from_compressed(comm, cc, "c64", mode="rows")
    _check_pieces(ss, cc, len(devices))
    assert any(0 < a or b < 64 for _, _, a, b in ss.pieces)  # some cut inside a component
    ref = O.OracleStore(cc.rounded_c64())
    x = _r(cn01(cc.m, 3, 1), "c64")
    phi = _r(cn01(cc.rows, 3, 2), "c64")
    ops = {}
    assert rel(ss.forward(x, ops), ref.forward(x)) <= 1e-5
    d = ref.opcounts(3)
    assert ops["decompress_madds"] == d[0] and ops["accumulate_madds"] == d[1]
    assert rel(ss.adjoint(phi), ref.adjoint(phi)) <= 1e-5
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).to(torch.complex64).cuda().t()
    pbig = torch.zeros((3, cc.rows + 7), dtype=torch.complex64, device="cuda")
    pbig[:, :cc.rows] = torch.from_numpy(np.ascontiguousarray(phi.T)).to(torch.complex64).cuda()
    pd = pbig.t()[:cc.rows]  # leading dimension rows + 7
    y = torch.full((3, cc.rows + 5), 9.0 + 0j, dtype=torch.complex64, device="cuda").t()[:cc.rows]
    z = torch.empty((3, cc.m + 2), dtype=torch.complex64, device="cuda").t()[:cc.m]
    ss.forward_into(xd, y)
    ss.adjoint_into(pd, z)
    torch.cuda.synchronize()
    assert rel(y.cpu().numpy(), ref.forward(x)) <= 1e-5
    assert rel(z.cpu().numpy(), ref.adjoint(phi)) <= 1e-5


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


@pytest.mark.parametrize("mode", ["columns", "rows"])
def test_sharded_empty_store(oracle, product, mode):
    """A store with no columns, sharded (src/matvec.cpp:28-38: zeros out)."""
    from paper_2103_06393_b200.multigpu import Comm, ShardedDeviceStore
    O = oracle
    cc = O.Compressed((16, 5, 17), 3, 0, np.zeros((0, 3, 3), np.int32), np.zeros(0, np.complex128))
    ss = ShardedDeviceStore.from_compressed(Comm([0, 0]), cc, "c64", mode=mode)
    y = ss.forward(np.zeros((0, 2)))
    assert y.shape == (cc.rows, 2) and not np.any(y)
    assert ss.adjoint(np.ones((cc.rows, 2))).shape == (0, 2)
