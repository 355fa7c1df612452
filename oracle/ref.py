"""TEST INFRASTRUCTURE ONLY — ctypes face of oracle/_ref/libtuckmat_ref.so.

That library is the REFERENCE ITSELF: /root/reference/proj/src/{tensor,
matvec,compress,io,aca,parallel,memlog,scene}.cpp compiled unchanged against
the Eigen-API shim (oracle/eigen_shim), plus the C wrapper oracle/ref_capi.cpp
(see oracle/Makefile).  The reference's own unit tests (proj/tests/test_*.cpp)
are compiled against the same objects (oracle/_ref/test_*) and pass there,
which pins the shim.  Tests use this module to pin the CPU restatement
(oracle/oracle.py, oracle/tuckmat_oracle.cpp) and to check the GPU path
directly against reference code.  Nothing in the product imports it.

Built here by `make -C oracle ref` (needs /root/reference); the built .so
travels to the GPU box with the repo snapshot (oracle/_ref/ is git-ignored,
not gpurun-ignored).
"""
from __future__ import annotations

import ctypes
import os
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtuckmat_ref.so")
REF_SRC = "/root/reference/proj"

_lib = None
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def available():
    return os.path.exists(LIB_PATH)


def build():
    """Compile oracle/_ref from the reference sources (only where they exist)."""
    import subprocess
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "-j8", "ref"], check=True)
    return available()


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref, needs {REF_SRC})")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        for name in ("ref_cc_destroy", "ref_aca_destroy", "ref_scene_destroy"):
            getattr(L, name).restype = None
            getattr(L, name).argtypes = [_vp]
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _c(a):
    return np.ascontiguousarray(a).ctypes.data_as(_vp)


def _mv(a):
    """Column-major complex128 block (rows x p) as a Fortran-ordered copy
    (row counts are checked by the reference itself)."""
    a = np.asarray(a, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


def _ptr(a):
    return a.ctypes.data_as(_vp)


class RefCC:
    """The reference's CompressedCoupling (proj/include/tuckmat/compress.hpp:14-25)."""

    def __init__(self, handle):
        self.h = _vp(handle)
        q = ctypes.c_int()
        m = _i64()
        dims = (ctypes.c_int64 * 3)()
        _check(lib().ref_cc_info(self.h, ctypes.byref(q), ctypes.byref(m), dims))
        self.q, self.m, self.grid_dims = q.value, m.value, tuple(int(d) for d in dims)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_cc_destroy(self.h)
            self.h = None

    @property
    def rows(self):
        return self.q * int(np.prod(self.grid_dims))

    @classmethod
    def load_ctc1(cls, path):
        h = _vp()
        _check(lib().ref_load_ctc1(os.fsencode(path), ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def from_compressed(cls, cc):
        """From an oracle.Compressed (ranks (m, q, 3), CTC1-order payload)."""
        h = _vp()
        ranks = np.ascontiguousarray(np.asarray(cc.ranks, np.int32).reshape(-1))
        payload = np.ascontiguousarray(np.asarray(cc.payload, np.complex128))
        dims = np.asarray(cc.grid_dims, np.int64)
        _check(lib().ref_cc_from_arrays(ctypes.c_int(cc.q), _i64(cc.m), _c(dims), _ptr(ranks), _ptr(payload),
                                        ctypes.byref(h)))
        return cls(h.value)

    def save_ctc1(self, path):
        _check(lib().ref_save_ctc1(self.h, os.fsencode(path)))

    def to_compressed(self):
        """Round trip through the reference's save_ctc1 into an oracle.Compressed."""
        from oracle import oracle as O
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "cc.ctc1")
            self.save_ctc1(p)
            return O.load_ctc1(p)

    def forward(self, x, workers=1, ops=None):
        x = _mv(x)
        y = np.zeros((self.rows, x.shape[1]), np.complex128, order="F")
        o = np.zeros(2, np.int64)
        _check(lib().ref_forward(self.h, _ptr(x), _i64(x.shape[0]), _i64(x.shape[1]), ctypes.c_int(workers), _ptr(y), _ptr(o)))
        if ops is not None:
            ops[0] += int(o[0])
            ops[1] += int(o[1])
        return y

    def adjoint(self, phi, workers=1, ops=None):
        phi = _mv(phi)
        z = np.zeros((self.m, phi.shape[1]), np.complex128, order="F")
        o = np.zeros(2, np.int64)
        _check(lib().ref_adjoint(self.h, _ptr(phi), _i64(phi.shape[0]), _i64(phi.shape[1]), ctypes.c_int(workers), _ptr(z), _ptr(o)))
        if ops is not None:
            ops[0] += int(o[0])
            ops[1] += int(o[1])
        return z

    def element(self, j, k, i1, i2, i3):
        out = np.zeros(2, np.float64)
        _check(lib().ref_element(self.h, _i64(j), ctypes.c_int(k), _i64(i1), _i64(i2), _i64(i3), _ptr(out)))
        return complex(out[0], out[1])


class RefAca:
    """The reference's Cta1File / AcaFactors with a Tucker-stored U (proj/include/tuckmat/aca.hpp:24-41)."""

    def __init__(self, handle):
        self.h = _vp(handle)
        q = ctypes.c_int()
        rc, m2 = _i64(), _i64()
        dims = (ctypes.c_int64 * 3)()
        _check(lib().ref_aca_info(self.h, ctypes.byref(q), ctypes.byref(rc), ctypes.byref(m2), dims))
        self.q, self.rank, self.cols, self.grid_dims = q.value, rc.value, m2.value, tuple(int(d) for d in dims)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_aca_destroy(self.h)
            self.h = None

    @property
    def rows(self):
        return self.q * int(np.prod(self.grid_dims))

    @classmethod
    def load_cta1(cls, path):
        h = _vp()
        _check(lib().ref_load_cta1(os.fsencode(path), ctypes.byref(h)))
        return cls(h.value)

    def aca_forward(self, x, workers=1):
        x = _mv(x)
        y = np.zeros((self.rows, x.shape[1]), np.complex128, order="F")
        _check(lib().ref_aca_forward(self.h, _ptr(x), _i64(x.shape[0]), _i64(x.shape[1]), ctypes.c_int(workers), _ptr(y)))
        return y

    def aca_adjoint(self, phi, workers=1):
        phi = _mv(phi)
        z = np.zeros((self.cols, phi.shape[1]), np.complex128, order="F")
        _check(lib().ref_aca_adjoint(self.h, _ptr(phi), _i64(phi.shape[0]), _i64(phi.shape[1]), ctypes.c_int(workers), _ptr(z)))
        return z

    def row_of_compressed_u(self, i):
        out = np.zeros(self.rank, np.complex128)
        _check(lib().ref_row_of_compressed_u(self.h, _i64(i), _ptr(out)))
        return out


class RefScene:
    """The reference's SceneSpec (proj/include/tuckmat/scene.hpp:56-62), q = 3."""

    def __init__(self, handle, m):
        self.h = _vp(handle)
        self.m = m

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_scene_destroy(self.h)
            self.h = None

    @classmethod
    def from_scene(cls, sc):
        """From an oracle.Scene (sources (m, 7)); validated by the reference."""
        h = _vp()
        src = np.ascontiguousarray(np.asarray(sc.sources, np.float64))
        _check(lib().ref_scene_create(_c(np.asarray(sc.origin, np.float64)), ctypes.c_double(sc.spacing),
                                      _c(np.asarray(sc.dims, np.int64)), ctypes.c_int(sc.op),
                                      ctypes.c_double(sc.k0), _ptr(src), _i64(src.shape[0]), ctypes.byref(h)))
        return cls(h.value, src.shape[0])

    @classmethod
    def loop(cls, spacing, dims, radius, center, nseg, op, k0, grid_center=(0.0, 0.0, 0.0)):
        """make_centered_grid + make_loop_scene of the reference."""
        h = _vp()
        _check(lib().ref_loop_scene(ctypes.c_double(spacing), _c(np.asarray(dims, np.int64)),
                                    _c(np.asarray(grid_center, np.float64)), ctypes.c_double(radius),
                                    _c(np.asarray(center, np.float64)), ctypes.c_int(nseg), ctypes.c_int(op),
                                    ctypes.c_double(k0), ctypes.byref(h)))
        return cls(h.value, nseg)

    def sources(self):
        origin = np.zeros(3)
        sp = ctypes.c_double()
        src = np.zeros((self.m, 7))
        _check(lib().ref_scene_sources(self.h, _ptr(origin), ctypes.byref(sp), _ptr(src)))
        return origin, sp.value, src

    def compress(self, eps, workers=1):
        h = _vp()
        _check(lib().ref_compress(self.h, ctypes.c_double(eps), ctypes.c_int(workers), ctypes.byref(h)))
        return RefCC(h.value)

    def tucker_aca(self, eps, hosvd_eps, path):
        h = _vp()
        _check(lib().ref_tucker_aca(self.h, ctypes.c_double(eps), ctypes.c_double(hosvd_eps), os.fsencode(path),
                                    ctypes.byref(h)))
        return RefAca(h.value)

    def dense_forward(self, x, rows):
        x = _mv(x)
        y = np.zeros((rows, x.shape[1]), np.complex128, order="F")
        _check(lib().ref_dense_forward(self.h, _ptr(x), _i64(x.shape[1]), _ptr(y)))
        return y

    def dense_adjoint(self, phi):
        phi = np.asfortranarray(np.asarray(phi, np.complex128).reshape(phi.shape[0], -1))
        z = np.zeros((self.m, phi.shape[1]), np.complex128, order="F")
        _check(lib().ref_dense_adjoint(self.h, _ptr(phi), _i64(phi.shape[1]), _ptr(z)))
        return z
