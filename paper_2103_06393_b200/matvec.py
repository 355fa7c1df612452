"""Python face of the B200 Tucker-compressed coupling matvec.

Mirrors the reference C++ API of /root/reference/proj/include/tuckmat/matvec.hpp
(forward, adjoint, aca_forward, aca_adjoint, OpCounts) on top of the C ABI
(include/tuckmat_b200.h).  The reference's value types (CompressedCoupling,
AcaFactors) become a device-resident ``DeviceStore``; multivectors are numpy
arrays (host, column-major) or torch CUDA tensors (device, column-major, i.e.
``t.stride(0) == 1``).  Host inputs go through the C ABI's TM_HOST mode (copy
in, compute, copy out); device inputs are enqueued on torch's current stream.

Errors map onto the reference taxonomy (include/tuckmat/errors.hpp:10-48).
There is no CPU fallback: without the built library or a CUDA device every
product raises.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import TM_C64, TM_C128, TM_DEVICE, TM_HOST, StoreDesc, lib


class Error(RuntimeError):
    """tuckmat::Error (errors.hpp:10-13)."""


class ContractViolation(Error):
    """tuckmat::ContractViolation (errors.hpp:16-19)."""


class CapacityError(Error):
    """tuckmat::CapacityError (errors.hpp:27-30)."""


class ParseError(Error):
    """tuckmat::ParseError (errors.hpp:39-45)."""

    def __init__(self, msg):
        super().__init__(msg)
        self.byte_offset = 0
        key = "(byte offset "
        if key in msg:
            try:
                self.byte_offset = int(msg[msg.rindex(key) + len(key):].rstrip(")"))
            except ValueError:
                pass


class CudaError(Error):
    """Device / driver failure (no reference analogue)."""


class SingularityError(Error):
    """tuckmat::SingularityError (errors.hpp:21-24)."""


_ERRS = {_lib.TM_CONTRACT_VIOLATION: ContractViolation, _lib.TM_CAPACITY_ERROR: CapacityError,
         _lib.TM_PARSE_ERROR: ParseError, _lib.TM_CUDA_ERROR: CudaError,
         _lib.TM_SINGULARITY_ERROR: SingularityError}


def _check(st):
    if st != _lib.TM_OK:
        msg = lib().tm_last_error().decode(errors="replace")
        raise _ERRS.get(st, Error)(msg)


_DT = {"c64": TM_C64, "complex64": TM_C64, TM_C64: TM_C64, "c128": TM_C128, "complex128": TM_C128, TM_C128: TM_C128}
_NP = {TM_C64: np.complex64, TM_C128: np.complex128}


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _torch_dtype(dt):
    import torch
    return torch.complex64 if dt == TM_C64 else torch.complex128


class OpCounts(dict):
    """OpCounts (matvec.hpp:17-20): counts are added (+=), as the reference does."""

    def __init__(self):
        super().__init__(decompress_madds=0, accumulate_madds=0)

    @property
    def decompress_madds(self):
        return self["decompress_madds"]

    @property
    def accumulate_madds(self):
        return self["accumulate_madds"]


class DeviceStore:
    """A Tucker column store resident in HBM (CompressedCoupling, or the
    Tucker U + V of AcaFactors)."""

    def __init__(self, handle, device):
        self._h = handle
        self.device = device
        q = ctypes.c_int32()
        ncols = ctypes.c_int64()
        dims = (ctypes.c_int64 * 3)()
        dt = ctypes.c_int32()
        m2 = ctypes.c_int64()
        nb = ctypes.c_int64()
        _check(lib().tm_store_info(handle, ctypes.byref(q), ctypes.byref(ncols), dims, ctypes.byref(dt),
                                   ctypes.byref(m2), ctypes.byref(nb)))
        self.q, self.ncols, self.dims = q.value, ncols.value, tuple(dims)
        self.dtype, self.m2, self.device_bytes = dt.value, m2.value, nb.value

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_arrays(cls, grid_dims, q, ranks, payload, dtype="c64", device=0, v=None):
        """ranks: (ncols, q, 3) int; payload: concatenated CTC1 tensor payloads
        (complex128, numpy host array or torch CUDA tensor); v: optional ACA V
        (m2 x r_c)."""
        ranks = np.ascontiguousarray(np.asarray(ranks, dtype=np.int32).reshape(-1, 3))
        if ranks.shape[0] % q:
            raise ContractViolation("ranks length is not a multiple of q")
        d = StoreDesc()
        d.q = int(q)
        d.ncols = ranks.shape[0] // q
        for g in range(3):
            d.dims[g] = int(grid_dims[g])
        d.ranks = ranks.ctypes.data
        keep = [ranks]
        if _is_torch(payload):
            import torch
            pt = payload.to(torch.complex128).contiguous()
            keep.append(pt)
            d.payload = pt.data_ptr()
            d.payload_on_device = 1
        else:
            pn = np.ascontiguousarray(np.asarray(payload, dtype=np.complex128))
            keep.append(pn)
            d.payload = pn.ctypes.data
        if v is not None:
            if _is_torch(v):
                import torch
                vt = v.to(torch.complex128).t().contiguous()  # column-major storage
                keep.append(vt)
                d.v = vt.data_ptr()
                d.v_on_device = 1
                d.m2 = v.shape[0]
            else:
                vn = np.asfortranarray(np.asarray(v, dtype=np.complex128))
                keep.append(vn)
                d.v = vn.ctypes.data
                d.m2 = vn.shape[0]
        h = ctypes.c_void_p()
        _check(lib().tm_store_create(ctypes.byref(d), int(device), _DT[dtype], ctypes.byref(h)))
        return cls(h, int(device))

    @classmethod
    def dense_aca(cls, u, v, dtype="c64", device=0):
        """AcaFactors with a dense U (m1 x r) and V (m2 x r): only aca_forward /
        aca_adjoint apply (src/matvec.cpp:158,173), on the device."""
        un = np.asfortranarray(np.asarray(u, dtype=np.complex128))
        vn = np.asfortranarray(np.asarray(v, dtype=np.complex128))
        if un.ndim != 2 or vn.ndim != 2 or un.shape[1] != vn.shape[1]:
            raise ContractViolation("dense ACA: U and V need the same column count")
        h = ctypes.c_void_p()
        _check(lib().tm_store_create_dense_aca(un.ctypes.data, un.shape[0], vn.ctypes.data, vn.shape[0], un.shape[1],
                                               0, int(device), _DT[dtype], ctypes.byref(h)))
        return cls(h, int(device))

    @classmethod
    def from_compressed(cls, cc, dtype="c64", device=0):
        """From any object with grid_dims, q, ranks, payload (and v for ACA)."""
        return cls.from_arrays(cc.grid_dims, cc.q, cc.ranks, cc.payload, dtype, device, getattr(cc, "v", None))

    @classmethod
    def load_ctc1(cls, path, dtype="c64", device=0):
        h = ctypes.c_void_p()
        _check(lib().tm_store_load_ctc1(str(path).encode(), int(device), _DT[dtype], ctypes.byref(h)))
        return cls(h, int(device))

    @classmethod
    def load_cta1(cls, path, dtype="c64", device=0):
        h = ctypes.c_void_p()
        _check(lib().tm_store_load_cta1(str(path).encode(), int(device), _DT[dtype], ctypes.byref(h)))
        return cls(h, int(device))

    def close(self):
        if getattr(self, "_h", None):
            lib().tm_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if not self._h:
            raise ContractViolation("store is closed")
        return self._h

    @property
    def num_voxels(self):
        return int(np.prod(self.dims))

    @property
    def rows(self):
        return self.q * self.num_voxels

    @property
    def np_dtype(self):
        return _NP[self.dtype]

    def row_block(self, indices):
        """Rows of the stored operator at global row indices (k*n_v + v):
        an (len(indices), ncols) array with entry [r, j] = T_jk[v] — the
        reference's element() per column (src/tensor.cpp:183-196), i.e.
        row_of_compressed_u (src/aca.cpp:234-244) on an ACA store."""
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.int64).reshape(-1))
        out = np.zeros((idx.size, self.ncols), dtype=self.np_dtype, order="F")
        _check(lib().tm_rows(self.handle, idx.ctypes.data, idx.size, out.ctypes.data, max(idx.size, 1), TM_HOST,
                             None))
        return out

    def element(self, j, k, i1, i2, i3):
        """element(tucker_jk, i1, i2, i3) (src/tensor.cpp:183-196)."""
        n1, n2, n3 = self.dims
        if not (0 <= j < self.ncols and 0 <= k < self.q and 0 <= i1 < n1 and 0 <= i2 < n2 and 0 <= i3 < n3):
            raise ContractViolation("element: index out of range")
        return self.row_block([k * self.num_voxels + i1 + n1 * (i2 + n2 * i3)])[0, j]

    def kernel_paths(self):
        """{'forward': 'tcgen05+warena' | 'tcgen05' | 'cuda-core', 'adjoint':
        'tcgen05+gemm' | 'tcgen05' | 'cuda-core'} for this
        store ('tcgen05+warena': the forward's A operand from the precomputed W
        arena; 'tcgen05+gemm': the adjoint as one GEMM on the transposed arena)."""
        f = ctypes.c_int32()
        a = ctypes.c_int32()
        _check(lib().tm_store_kernels(self.handle, ctypes.byref(f), ctypes.byref(a)))
        name = {3: "tcgen05+gemm", 2: "tcgen05+warena", 1: "tcgen05", 0: "cuda-core"}
        return {"forward": name[f.value], "adjoint": name[a.value]}  # adjoint 2: W tiles from the arena

    def opcounts(self, p=1):
        """Exact OpCounts of one product at p right-hand sides (matvec.cpp:10-15,50-51)."""
        dec = ctypes.c_int64()
        acc = ctypes.c_int64()
        _check(lib().tm_opcounts(self.handle, int(p), ctypes.byref(dec), ctypes.byref(acc)))
        return int(dec.value), int(acc.value)

    # -- products -------------------------------------------------------------
    def _call(self, fn, x, outrows, ops, with_ops):
        if _is_torch(x):
            return self._call_device(fn, x, outrows, ops, with_ops)
        a = np.asarray(x)
        squeeze = a.ndim == 1
        a = np.asfortranarray(a.reshape(-1, 1) if squeeze else a, dtype=self.np_dtype)
        inrows, p = a.shape
        out = np.zeros((outrows, p), dtype=self.np_dtype, order="F")
        o = np.zeros(2, np.int64)
        args = [self.handle, a.ctypes.data, max(inrows, 1), inrows, p, out.ctypes.data, max(outrows, 1), TM_HOST,
                None]
        if with_ops:
            args.append(o.ctypes.data)
        _check(fn(*args))
        if ops is not None:
            ops["decompress_madds"] = ops.get("decompress_madds", 0) + int(o[0])
            ops["accumulate_madds"] = ops.get("accumulate_madds", 0) + int(o[1])
        return out[:, 0] if squeeze else out

    def _call_device(self, fn, x, outrows, ops, with_ops, out=None, stream=None):
        import torch
        td = _torch_dtype(self.dtype)
        if x.device.type != "cuda" or x.device.index != self.device:
            raise ContractViolation(f"input is on {x.device}, store is on cuda:{self.device}")
        x_in = x
        squeeze = x.dim() == 1
        if squeeze:
            x = x.reshape(-1, 1)
        if x.dtype != td:
            x = x.to(td)
        # torch's lazy conjugate / negative views keep the raw memory
        # unconjugated: materialise them before handing the pointer over
        if x.is_conj():
            x = x.resolve_conj()
        if x.is_neg():
            x = x.resolve_neg()
        if x.stride(0) != 1 or (x.shape[1] > 1 and x.stride(1) < x.shape[0]):
            x = x.t().contiguous().t()
        inrows, p = x.shape
        ldx = x.stride(1) if p > 1 else max(inrows, 1)
        own_out = out is None
        if own_out:
            out = torch.empty((p, outrows), dtype=td, device=x.device).t()
        else:  # a caller's buffer: exact shape, dtype, device and column-major layout
            o2 = out.reshape(-1, 1) if out.dim() == 1 else out
            if (o2.dim() != 2 or tuple(o2.shape) != (outrows, p) or out.dtype != td
                    or out.device != x.device or o2.stride(0) != 1 or (p > 1 and o2.stride(1) < outrows)):
                raise ContractViolation(
                    f"out must be a column-major {td} tensor of shape ({outrows}, {p}) on {x.device}, got "
                    f"{tuple(out.shape)} {out.dtype} strides {tuple(out.stride())} on {out.device}")
            out = o2
        ldo = out.stride(1) if p > 1 else max(outrows, 1)
        if stream is not None:
            # work enqueued on a caller's stream: it first waits for torch's
            # current stream (where x was produced and temporaries were
            # allocated), and the allocator must not recycle those
            # temporaries before the caller's stream is done with them
            ext = torch.cuda.ExternalStream(stream, device=x.device)
            ext.wait_stream(torch.cuda.current_stream(x.device))
            if x.data_ptr() != x_in.data_ptr():
                x.record_stream(ext)
            if own_out:
                out.record_stream(ext)
        st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        o = np.zeros(2, np.int64)
        args = [self.handle, x.data_ptr(), ldx, inrows, p, out.data_ptr(), ldo, TM_DEVICE, st]
        if with_ops:
            args.append(o.ctypes.data)
        _check(fn(*args))
        if ops is not None:
            ops["decompress_madds"] = ops.get("decompress_madds", 0) + int(o[0])
            ops["accumulate_madds"] = ops.get("accumulate_madds", 0) + int(o[1])
        return out[:, 0] if squeeze else out

    def forward_components(self, x, k0, k1, out, stream=None):
        """Device forward restricted to components [k0, k1): rows k n_v ..
        (k + 1) n_v - 1 of `out` (column-major, rows x p) for k in the range;
        the other rows are untouched (tm_forward_components)."""
        import torch
        td = _torch_dtype(self.dtype)
        if x.device.type != "cuda" or x.device.index != self.device:
            raise ContractViolation(f"input is on {x.device}, store is on cuda:{self.device}")
        x = x.reshape(-1, 1) if x.dim() == 1 else x
        x = x.to(td).resolve_conj().resolve_neg()
        if x.stride(0) != 1 or (x.shape[1] > 1 and x.stride(1) < x.shape[0]):
            x = x.t().contiguous().t()
        o2 = out.reshape(-1, 1) if out.dim() == 1 else out
        inrows, p = x.shape
        if (tuple(o2.shape) != (self.rows, p) or out.dtype != td or out.device != x.device or o2.stride(0) != 1
                or (p > 1 and o2.stride(1) < self.rows)):
            raise ContractViolation(f"out must be a column-major {td} tensor of shape ({self.rows}, {p}) on {x.device}")
        st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        _check(lib().tm_forward_components(self.handle, x.data_ptr(), x.stride(1) if p > 1 else max(inrows, 1),
                                           inrows, p, o2.data_ptr(), o2.stride(1) if p > 1 else self.rows, int(k0),
                                           int(k1), st))
        return out

    def forward(self, x, ops=None):
        """Y = Zbc X (forward, src/matvec.cpp:132-138)."""
        return self._call(lib().tm_forward, x, self.rows, ops, True)

    def adjoint(self, phi, ops=None):
        """Z = Zbc^H Phi (adjoint, src/matvec.cpp:140-148)."""
        return self._call(lib().tm_adjoint, phi, self.ncols, ops, True)

    def aca_forward(self, x):
        """U (V^H x) (aca_forward, src/matvec.cpp:150-160)."""
        return self._call(lib().tm_aca_forward, x, self.rows, None, False)

    def aca_adjoint(self, phi):
        """V (U^H phi) (aca_adjoint, src/matvec.cpp:162-175)."""
        return self._call(lib().tm_aca_adjoint, phi, self.m2, None, False)

    def forward_into(self, x, out, stream=None):
        """Device-only forward writing into a preallocated column-major tensor."""
        return self._call_device(lib().tm_forward, x, self.rows, None, True, out=out, stream=stream)

    def adjoint_into(self, phi, out, stream=None):
        return self._call_device(lib().tm_adjoint, phi, self.ncols, None, True, out=out, stream=stream)


# Reference-named free functions (include/tuckmat/matvec.hpp:47-57).  The
# reference's `workers` (host threads) is accepted and ignored.
def forward(store, x, workers=1, ops=None):
    return store.forward(x, ops)


def adjoint(store, phi, workers=1, ops=None):
    return store.adjoint(phi, ops)


def aca_forward(store, x, workers=1):
    return store.aca_forward(x)


def aca_adjoint(store, phi, workers=1):
    return store.aca_adjoint(phi)


def load_ctc1(path, dtype="c64", device=0):
    return DeviceStore.load_ctc1(path, dtype, device)


def load_cta1(path, dtype="c64", device=0):
    return DeviceStore.load_cta1(path, dtype, device)
