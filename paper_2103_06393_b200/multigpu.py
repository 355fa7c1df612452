"""Single-process multi-GPU sharding through the C ABI (tm_comm_* /
tm_sharded_*, include/tuckmat_b200.h): one host thread drives the GPUs of one
box through an NCCL communicator (ncclCommInitAll).  Two partitions:

* columns (default): cost-balanced contiguous column ranges — the
  reference's parallel_for over columns (src/parallel.cpp:13-48) lifted to
  GPUs; the forward's partial y is reduced per component, overlapped with the
  later components' waves, the adjoint broadcasts Phi and gathers z rows.
  sharded.py is its torch.distributed counterpart (bench.py under torchrun).
* rows: cost-balanced (component, i1) slab ranges; each piece is
  a store on the sub-grid; the forward copies each GPU's rows of y into the
  output (no reduction), the adjoint reads each GPU's rows of Phi and
  reduces the m x p partial z.

A device list that repeats a device builds an emulated communicator (the
collectives become device-local copies and adds) — the tests use it to run
the sharded orchestration on one GPU.
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import StoreDesc, lib
from .matvec import _DT, ContractViolation, DeviceStore, _check


class Comm:
    """tm_comm: a single-process communicator over `devices` (devices[0] is the root)."""

    def __init__(self, devices):
        import torch  # noqa: F401  (torch's bundled NCCL is then the one tm_comm_init finds in-process)
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        self._h = ctypes.c_void_p()
        _check(lib().tm_comm_init(len(devices), devs, ctypes.byref(self._h)))
        self.devices = [int(d) for d in devices]
        nd, em = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().tm_comm_info(self._h, ctypes.byref(nd), ctypes.byref(em)))
        self.emulated = bool(em.value)

    @property
    def handle(self):
        if not self._h:
            raise ContractViolation("communicator is finalized")
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tm_comm_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def row_cuts(comp_costs, n1, ndev, align=8, min_rows=8):
    """The C ABI's row partition rule (tm_shard_row_cuts): ndev + 1 cut points
    over the q * n1 global slabs k * n1 + i1 (same rule as
    sharded.row_pieces; host only)."""
    cc = np.ascontiguousarray(np.asarray(comp_costs, dtype=np.float64))
    out = np.zeros(ndev + 1, np.int64)
    _check(lib().tm_shard_row_cuts(len(cc), int(n1), int(ndev), int(align), int(min_rows), cc.ctypes.data,
                                   out.ctypes.data))
    return out


class ShardedDeviceStore(DeviceStore):
    """A Tucker store sharded over a Comm's devices — by columns (mode
    "columns", the default) or by row slabs (mode "rows"); the
    products take host numpy blocks or torch tensors on the root device."""

    def __init__(self, handle, comm, q, ncols, dims, dtype, m2, mode="columns"):
        self._h = handle
        self.comm = comm  # keeps the communicator alive
        self.device = comm.devices[0]
        self.q, self.ncols, self.dims, self.dtype, self.m2 = q, ncols, tuple(dims), dtype, m2
        ns = ctypes.c_int32()
        nb = ctypes.c_int64()
        ranges = (ctypes.c_int64 * (2 * len(comm.devices)))()
        _check(lib().tm_sharded_info(handle, ctypes.byref(ns), ranges, ctypes.byref(nb)))
        self.shard_ranges = [(ranges[2 * i], ranges[2 * i + 1]) for i in range(ns.value)]
        self.device_bytes = nb.value
        self.mode = mode
        npc = ctypes.c_int32()
        _check(lib().tm_sharded_pieces(handle, ctypes.byref(npc), None))
        buf = (ctypes.c_int64 * max(4 * npc.value, 1))()
        _check(lib().tm_sharded_pieces(handle, ctypes.byref(npc), buf))
        # rows mode: (shard, component k, i1 row a, i1 row b) per piece
        self.pieces = [tuple(int(buf[4 * i + e]) for e in range(4)) for i in range(npc.value)]

    @classmethod
    def from_arrays(cls, comm, grid_dims, q, ranks, payload, dtype="c64", v=None, mode="columns"):
        ranks = np.ascontiguousarray(np.asarray(ranks, dtype=np.int32).reshape(-1, 3))
        d = StoreDesc()
        d.q = int(q)
        d.ncols = ranks.shape[0] // q
        for g in range(3):
            d.dims[g] = int(grid_dims[g])
        d.ranks = ranks.ctypes.data
        pn = np.ascontiguousarray(np.asarray(payload, dtype=np.complex128))
        d.payload = pn.ctypes.data
        m2 = 0
        if v is not None:
            vn = np.asfortranarray(np.asarray(v, dtype=np.complex128))
            d.v = vn.ctypes.data
            d.m2 = m2 = vn.shape[0]
        h = ctypes.c_void_p()
        modes = {"columns": 0, "rows": 1}
        if mode not in modes:
            raise ContractViolation(f"unknown sharding mode {mode!r} (columns or rows)")
        _check(lib().tm_sharded_create_mode(ctypes.byref(d), comm.handle, _DT[dtype], modes[mode], ctypes.byref(h)))
        return cls(h, comm, int(q), d.ncols, tuple(int(x) for x in grid_dims), _DT[dtype], m2, mode)

    @classmethod
    def from_compressed(cls, comm, cc, dtype="c64", mode="columns"):
        return cls.from_arrays(comm, cc.grid_dims, cc.q, cc.ranks, cc.payload, dtype, getattr(cc, "v", None), mode)

    def close(self):
        if getattr(self, "_h", None):
            lib().tm_sharded_destroy(self._h)
            self._h = None

    def forward(self, x, ops=None):
        return self._call(lib().tm_sharded_forward, x, self.rows, ops, True)

    def adjoint(self, phi, ops=None):
        return self._call(lib().tm_sharded_adjoint, phi, self.ncols, ops, True)

    def aca_forward(self, x):
        return self._call(lib().tm_sharded_aca_forward, x, self.rows, None, False)

    def aca_adjoint(self, phi):
        return self._call(lib().tm_sharded_aca_adjoint, phi, self.m2, None, False)

    def forward_into(self, x, out, stream=None):
        return self._call_device(lib().tm_sharded_forward, x, self.rows, None, True, out=out, stream=stream)

    def adjoint_into(self, phi, out, stream=None):
        return self._call_device(lib().tm_sharded_adjoint, phi, self.ncols, None, True, out=out, stream=stream)

    def _single_store_only(self, *a, **k):
        raise ContractViolation("not available on a sharded store (use a shard's DeviceStore)")

    row_block = element = opcounts = kernel_paths = _single_store_only
