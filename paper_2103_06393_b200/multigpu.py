"""Single-process multi-GPU column sharding through the C ABI (tm_comm_* /
tm_sharded_*, include/tuckmat_b200.h): one host thread drives the GPUs of one
box through an NCCL communicator (ncclCommInitAll); the forward's partial y is
reduced per component, overlapped with the later components' waves, the
adjoint broadcasts Phi and gathers z rows.  This is the C-ABI counterpart of
sharded.py (one process per GPU over torch.distributed, used by bench.py under
torchrun); both shard by cost-balanced contiguous column ranges, the
reference's parallel_for over columns (src/parallel.cpp:13-48) lifted to GPUs.

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


class ShardedDeviceStore(DeviceStore):
    """A Tucker column store sharded by columns over a Comm's devices; the
    products take host numpy blocks or torch tensors on the root device."""

    def __init__(self, handle, comm, q, ncols, dims, dtype, m2):
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

    @classmethod
    def from_arrays(cls, comm, grid_dims, q, ranks, payload, dtype="c64", v=None):
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
        _check(lib().tm_sharded_create(ctypes.byref(d), comm.handle, _DT[dtype], ctypes.byref(h)))
        return cls(h, comm, int(q), d.ncols, tuple(int(x) for x in grid_dims), _DT[dtype], m2)

    @classmethod
    def from_compressed(cls, comm, cc, dtype="c64"):
        return cls.from_arrays(comm, cc.grid_dims, cc.q, cc.ranks, cc.payload, dtype, getattr(cc, "v", None))

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
