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
