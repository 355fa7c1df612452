"""TEST INFRASTRUCTURE ONLY — Python face of the CPU oracle.

This module restates the reference ``tuckmat`` library (C++20 + Eigen,
/root/reference/proj) closely enough to serve as the parity checker for the
B200 product path and as the timed CPU baseline.  It must never be imported by
the product package ``paper_2103_06393_b200``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / ``--impl
reference`` leg) may use it.

The hot-path restatement (mode products, reconstruct, stacked_forward /
stacked_adjoint with per-worker partials, forward / adjoint / aca_*, OpCounts,
scene kernels and dense assembly) is C++ in ``tuckmat_oracle.cpp`` (built to
``oracle/build/liboracle.so``).  The *producers* of the hot path's inputs —
HOSVD (src/tensor.cpp:122-174), compress_matrix (src/compress.cpp:7-35),
aca_dense / tucker_aca (src/aca.cpp:54-232) and the CTC1 / CTA1 containers
(src/io.cpp:121-279) — are restated here in numpy.  Eigen's BDCSVD is replaced
by LAPACK gesdd (numpy); singular vectors may differ by a phase, which changes
compressed factors bitwise but not the reconstruction — irrelevant to matvec
parity because both sides read the same store.

Complex data is numpy complex128; multivectors are (rows, p) arrays that are
Fortran-ordered (column-major) on the C side, as Eigen::MatrixXcd is.
"""
from __future__ import annotations

import ctypes
import math
import os
import struct
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None
_lib_lock = threading.Lock()

# Status codes (reference include/tuckmat/errors.hpp:10-48).
OK, CONTRACT_VIOLATION, CAPACITY_ERROR, PARSE_ERROR, SINGULARITY_ERROR, SCENE_ERROR = 0, 1, 2, 3, 4, 5


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ContractViolation(OracleError):
    pass


class SingularityError(OracleError):
    pass


class SceneError(OracleError):
    def __init__(self, msg, source):
        super().__init__(SCENE_ERROR, msg)
        self.source = source


class ParseError(OracleError):
    def __init__(self, msg, offset):
        super().__init__(PARSE_ERROR, f"{msg} (byte offset {offset})")
        self.byte_offset = offset


def build():
    """Compile liboracle.so (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            L = ctypes.CDLL(_LIB_PATH)
            vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
            L.orc_last_error.restype = ctypes.c_char_p
            L.orc_store_create.argtypes = [i32, i64, vp, vp, vp, ctypes.POINTER(vp)]
            L.orc_store_destroy.argtypes = [vp]
            L.orc_forward.argtypes = [vp, vp, i64, i64, vp, i32, vp]
            L.orc_adjoint.argtypes = [vp, vp, i64, i64, vp, i32, vp]
            L.orc_aca_forward.argtypes = [vp, vp, i64, vp, i64, i64, vp, i32]
            L.orc_aca_adjoint.argtypes = [vp, vp, i64, vp, i64, i64, vp, i32]
            L.orc_opcounts.argtypes = [vp, i64, vp, vp]
            L.orc_reconstruct.argtypes = [vp, i64, i32, vp]
            L.orc_element.argtypes = [vp, i64, i32, i64, i64, i64, vp]
            L.orc_mode_product.argtypes = [vp, vp, vp, i64, i64, i32, vp]
            L.orc_assemble_column.argtypes = [vp, dbl, vp, i32, dbl, i32, vp, i64, i64, vp]
            L.orc_assemble_full.argtypes = [vp, dbl, vp, i32, dbl, i32, vp, i64, i32, vp]
            L.orc_eval_kernel.argtypes = [i32, dbl, vp, vp, vp]
            L.orc_random_multivector.argtypes = [i64, i64, ctypes.c_uint64, vp]
            L.orc_randn_tests.argtypes = [i64, ctypes.c_uint64, vp]
            _lib = L
    return _lib


def _check(code):
    if code != OK:
        msg = lib().orc_last_error().decode()
        if code == CONTRACT_VIOLATION:
            raise ContractViolation(code, msg)
        if code == SINGULARITY_ERROR:
            raise SingularityError(code, msg)
        raise OracleError(code, msg)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _fortran_c128(a, rows=None):
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a.astype(np.complex128, copy=False))


def default_workers():
    return max(1, os.cpu_count() or 1)


# ---------------------------------------------------------------- stores --
def tensor_sizes(dims, ranks):
    """Scalars per tensor: r1 r2 r3 + sum_g n_g r_g (src/tensor.cpp:198-203)."""
    r = np.asarray(ranks, dtype=np.int64).reshape(-1, 3)
    n = np.asarray(dims, dtype=np.int64)
    return r[:, 0] * r[:, 1] * r[:, 2] + r @ n


def tensor_offsets(dims, ranks):
    s = tensor_sizes(dims, ranks)
    off = np.zeros(len(s) + 1, dtype=np.int64)
    np.cumsum(s, out=off[1:])
    return off


def split_tensor(dims, ranks_t, flat):
    """(core (r1,r2,r3) Fortran, U1, U2, U3) views of one tensor payload."""
    r1, r2, r3 = (int(v) for v in ranks_t)
    n1, n2, n3 = (int(v) for v in dims)
    o = 0
    core = flat[o:o + r1 * r2 * r3].reshape((r1, r2, r3), order="F"); o += r1 * r2 * r3
    u1 = flat[o:o + n1 * r1].reshape((n1, r1), order="F"); o += n1 * r1
    u2 = flat[o:o + n2 * r2].reshape((n2, r2), order="F"); o += n2 * r2
    u3 = flat[o:o + n3 * r3].reshape((n3, r3), order="F")
    return core, u1, u2, u3


def pack_tensors(tensors):
    """Flatten a list of (core, U1, U2, U3) into (ranks int32 (n,3), payload)."""
    ranks = np.array([t[0].shape for t in tensors], dtype=np.int32).reshape(-1, 3)
    parts = []
    for core, u1, u2, u3 in tensors:
        parts += [np.ravel(core, order="F"), np.ravel(u1, order="F"), np.ravel(u2, order="F"),
                  np.ravel(u3, order="F")]
    payload = np.concatenate(parts).astype(np.complex128) if parts else np.zeros(0, np.complex128)
    return ranks, payload


@dataclass
class Compressed:
    """CompressedCoupling stand-in (reference include/tuckmat/compress.hpp:14-25).

    ``ranks`` is (m, q, 3) int32 and ``payload`` the concatenated CTC1 tensor
    payloads in [column][component] order (src/io.cpp:121-129,204-208)."""
    grid_dims: tuple
    q: int
    m: int
    ranks: np.ndarray
    payload: np.ndarray
    kernel_op: int = 0
    k0: float = 0.0
    eps: float = 0.0

    @property
    def num_voxels(self):
        return int(np.prod(self.grid_dims))

    @property
    def rows(self):
        return self.q * self.num_voxels

    def tensor(self, j, k):
        off = tensor_offsets(self.grid_dims, self.ranks)
        i = j * self.q + k
        return split_tensor(self.grid_dims, self.ranks.reshape(-1, 3)[i], self.payload[off[i]:off[i + 1]])

    def rounded_c64(self):
        """The c64 store: factors rounded once, then read back as c128 (SURVEY §0 gap 3)."""
        return Compressed(self.grid_dims, self.q, self.m, self.ranks,
                          self.payload.astype(np.complex64).astype(np.complex128), self.kernel_op, self.k0,
                          self.eps)


@dataclass
class Aca:
    """AcaFactors stand-in with a Tucker-stored U (include/tuckmat/aca.hpp:24-41):
    U columns l = 0..r_c-1, each q tensors (ranks (r_c, q, 3)); V is (m2, r_c)."""
    grid_dims: tuple
    q: int
    ranks: np.ndarray
    payload: np.ndarray
    v: np.ndarray
    eps: float = 0.0
    hosvd_eps: float = 0.0
    converged: bool = False
    final_stat: float = 0.0

    @property
    def rank(self):
        return int(self.v.shape[1])

    @property
    def rows(self):
        return self.q * int(np.prod(self.grid_dims))

    @property
    def cols(self):
        return int(self.v.shape[0])

    def store(self):
        return Compressed(self.grid_dims, self.q, self.rank, self.ranks, self.payload)

    def rounded_c64(self):
        return Aca(self.grid_dims, self.q, self.ranks, self.payload.astype(np.complex64).astype(np.complex128),
                   self.v.astype(np.complex64).astype(np.complex128), self.eps, self.hosvd_eps, self.converged,
                   self.final_stat)


class OracleStore:
    """Owns the C++ oracle's copy of a Tucker column store."""

    def __init__(self, cc):
        self.q = int(cc.q)
        self.dims = tuple(int(d) for d in cc.grid_dims)
        ranks = np.ascontiguousarray(np.asarray(cc.ranks, dtype=np.int32).reshape(-1, 3))
        self.ncols = ranks.shape[0] // self.q
        payload = np.ascontiguousarray(np.asarray(cc.payload, dtype=np.complex128))
        dims = np.array(self.dims, dtype=np.int64)
        h = ctypes.c_void_p()
        _check(lib().orc_store_create(self.q, self.ncols, _ptr(dims), _ptr(ranks), _ptr(payload), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_store_destroy(self._h)
            self._h = None

    @property
    def rows(self):
        return self.q * int(np.prod(self.dims))

    def forward(self, x, workers=1, ops=None):
        x = _fortran_c128(x)
        y = np.zeros((self.rows, x.shape[1]), dtype=np.complex128, order="F")
        o = np.zeros(2, dtype=np.int64)
        _check(lib().orc_forward(self._h, _ptr(x), x.shape[0], x.shape[1], _ptr(y), workers, _ptr(o)))
        if ops is not None:
            ops["decompress_madds"] = ops.get("decompress_madds", 0) + int(o[0])
            ops["accumulate_madds"] = ops.get("accumulate_madds", 0) + int(o[1])
        return y

    def adjoint(self, phi, workers=1, ops=None):
        phi = _fortran_c128(phi)
        z = np.zeros((self.ncols, phi.shape[1]), dtype=np.complex128, order="F")
        o = np.zeros(2, dtype=np.int64)
        _check(lib().orc_adjoint(self._h, _ptr(phi), phi.shape[0], phi.shape[1], _ptr(z), workers, _ptr(o)))
        if ops is not None:
            ops["decompress_madds"] = ops.get("decompress_madds", 0) + int(o[0])
            ops["accumulate_madds"] = ops.get("accumulate_madds", 0) + int(o[1])
        return z

    def aca_forward(self, v, x, workers=1):
        v = _fortran_c128(v)
        x = _fortran_c128(x)
        y = np.zeros((self.rows, x.shape[1]), dtype=np.complex128, order="F")
        _check(lib().orc_aca_forward(self._h, _ptr(v), v.shape[0], _ptr(x), x.shape[0], x.shape[1], _ptr(y),
                                     workers))
        return y

    def aca_adjoint(self, v, phi, workers=1):
        v = _fortran_c128(v)
        phi = _fortran_c128(phi)
        z = np.zeros((v.shape[0], phi.shape[1]), dtype=np.complex128, order="F")
        _check(lib().orc_aca_adjoint(self._h, _ptr(v), v.shape[0], _ptr(phi), phi.shape[0], phi.shape[1],
                                     _ptr(z), workers))
        return z

    def opcounts(self, p):
        d = np.zeros(1, np.int64)
        a = np.zeros(1, np.int64)
        _check(lib().orc_opcounts(self._h, p, _ptr(d), _ptr(a)))
        return int(d[0]), int(a[0])

    def reconstruct(self, j, k):
        out = np.zeros(int(np.prod(self.dims)), dtype=np.complex128)
        _check(lib().orc_reconstruct(self._h, j, k, _ptr(out)))
        return out.reshape(self.dims, order="F")

    def column(self, j):
        return np.concatenate([self.reconstruct(j, k).ravel(order="F") for k in range(self.q)])

    def element(self, j, k, i1, i2, i3):
        out = np.zeros(2, np.float64)
        _check(lib().orc_element(self._h, j, k, i1, i2, i3, _ptr(out)))
        return complex(out[0], out[1])


def forward(cc, x, workers=1, ops=None):
    """forward(cc, x) (reference src/matvec.cpp:132-138)."""
    return OracleStore(cc).forward(x, workers, ops)


def adjoint(cc, phi, workers=1, ops=None):
    """adjoint(cc, phi) (reference src/matvec.cpp:140-148)."""
    return OracleStore(cc).adjoint(phi, workers, ops)


def aca_forward(fac, x, workers=1):
    """aca_forward (src/matvec.cpp:150-160); dense-U fallback (:158) included."""
    x = _fortran_c128(x)
    if x.shape[0] != fac.cols:
        raise ContractViolation(CONTRACT_VIOLATION, f"aca_forward: x has {x.shape[0]} rows, expected {fac.cols}")
    if isinstance(fac, DenseAca):
        return fac.u @ (fac.v.conj().T @ x)
    if fac.rank == 0:
        return np.zeros((fac.rows, x.shape[1]), np.complex128)
    return OracleStore(fac.store()).aca_forward(fac.v, x, workers)


def aca_adjoint(fac, phi, workers=1):
    """aca_adjoint (src/matvec.cpp:162-175)."""
    phi = _fortran_c128(phi)
    if phi.shape[0] != fac.rows:
        raise ContractViolation(CONTRACT_VIOLATION, f"aca_adjoint: phi has {phi.shape[0]} rows, expected {fac.rows}")
    if isinstance(fac, DenseAca):
        return fac.v @ (fac.u.conj().T @ phi)
    if fac.rank == 0:
        return np.zeros((fac.cols, phi.shape[1]), np.complex128)
    return OracleStore(fac.store()).aca_adjoint(fac.v, phi, workers)


def mode_product(t, m, mode):
    """mode_product (src/tensor.cpp:89-120) on numpy arrays."""
    t = np.asfortranarray(t, dtype=np.complex128)
    m = np.asfortranarray(m, dtype=np.complex128)
    od = list(t.shape)
    if 1 <= mode <= 3:
        od[mode - 1] = m.shape[0]
    out = np.zeros(int(np.prod(od)) if 1 <= mode <= 3 else 1, np.complex128)
    dims = np.array(t.shape, np.int64)
    _check(lib().orc_mode_product(_ptr(t), _ptr(dims), _ptr(m), m.shape[0], m.shape[1], mode, _ptr(out)))
    return out.reshape(od, order="F")


def reconstruct(core, u1, u2, u3):
    out = mode_product(core, u1, 1)
    out = mode_product(out, u2, 2)
    return mode_product(out, u3, 3)


def reconstruct_madds(dims, ranks):
    """reconstruct_madds (src/matvec.cpp:10-15)."""
    n1, n2, n3 = dims
    r1, r2, r3 = ranks
    return n1 * r1 * r2 * r3 + n1 * n2 * r2 * r3 + n1 * n2 * n3 * r3


def mode_product_loops(t, m, mode):
    """Plain loop n-mode product (reference tests/oracles.hpp:69-88)."""
    od = list(t.shape)
    od[mode - 1] = m.shape[0]
    out = np.zeros(od, np.complex128)
    for i3 in range(od[2]):
        for i2 in range(od[1]):
            for i1 in range(od[0]):
                acc = 0j
                for c in range(m.shape[1]):
                    if mode == 1:
                        acc += t[c, i2, i3] * m[i1, c]
                    elif mode == 2:
                        acc += t[i1, c, i3] * m[i2, c]
                    else:
                        acc += t[i1, i2, c] * m[i3, c]
                out[i1, i2, i3] = acc
    return out


# ------------------------------------------------------------ random data --
def random_multivector(rows, cols, seed):
    """random_multivector (src/experiments.cpp:26-33): mt19937_64 + N(0,1), re then im, column-major."""
    out = np.zeros(rows * cols, np.complex128)
    lib().orc_random_multivector(rows, cols, seed, _ptr(out))
    return out.reshape((rows, cols), order="F")


def randn_c(n, seed):
    """n draws of tests/oracles.hpp randn_c from one mt19937_64(seed)."""
    out = np.zeros(n, np.complex128)
    lib().orc_randn_tests(n, seed, _ptr(out))
    return out


def random_matrix(rows, cols, seed):
    """tests/oracles.hpp:31-37."""
    return randn_c(rows * cols, seed).reshape((rows, cols), order="F")


def random_tensor(dims, seed):
    """tests/oracles.hpp:24-29."""
    return randn_c(int(np.prod(dims)), seed).reshape(dims, order="F")


# ----------------------------------------------------------------- scenes --
def wavenumber_from_mhz(f_mhz):
    """include/tuckmat/scene.hpp:20-22."""
    return 2.0 * math.pi * f_mhz * 1e6 / 299792458.0


@dataclass
class Scene:
    """SceneSpec (include/tuckmat/scene.hpp:24-67).  sources is (m, 7):
    midpoint xyz, unit direction xyz, weight."""
    origin: np.ndarray
    spacing: float
    dims: tuple
    sources: np.ndarray
    op: int = 0
    k0: float = 0.0
    q: int = 3

    @property
    def num_voxels(self):
        return int(np.prod(self.dims))

    @property
    def num_sources(self):
        return int(self.sources.shape[0])

    @property
    def rows(self):
        return self.q * self.num_voxels


def make_centered_grid(center, spacing, dims):
    """make_centered_grid (src/scene.cpp:27-41): returns (origin, spacing, dims)."""
    if not spacing > 0:
        raise ContractViolation(CONTRACT_VIOLATION, "voxel grid spacing must be positive")
    if min(dims) <= 0:
        raise ContractViolation(CONTRACT_VIOLATION, "voxel grid dims must be positive")
    origin = np.array([center[a] - 0.5 * spacing * dims[a] for a in range(3)], np.float64)
    return origin, float(spacing), tuple(int(d) for d in dims)


def separation(origin, spacing, dims, point):
    """Distance to the nearest voxel centre (src/scene.cpp:13-23)."""
    nearest = np.zeros(3)
    for a in range(3):
        cell = (point[a] - origin[a]) / spacing - 0.5
        idx = min(max(round(cell), 0.0), float(dims[a] - 1))
        nearest[a] = origin[a] + spacing * (idx + 0.5)
    return float(np.linalg.norm(np.asarray(point) - nearest))


def validate_scene(sc, allow_pwl=True):
    """validate_scene (src/scene.cpp:43-74); q = 12 is this build's PWL extension."""
    if not sc.spacing > 0 or min(sc.dims) <= 0:
        raise ContractViolation(CONTRACT_VIOLATION, "scene grid is invalid")
    if sc.q != 3 and not (allow_pwl and sc.q == 12):
        raise ContractViolation(CONTRACT_VIOLATION, "kernel q must be 3 (one field vector per voxel)")
    if sc.k0 < 0:
        raise ContractViolation(CONTRACT_VIOLATION, "wavenumber k0 must be non-negative")
    if sc.op == 0 and not sc.k0 > 0:
        raise ContractViolation(CONTRACT_VIOLATION, "electric-field kernel requires k0 > 0")
    if sc.num_sources == 0:
        raise ContractViolation(CONTRACT_VIOLATION, "scene needs at least one source")
    for j, s in enumerate(sc.sources):
        if not s[6] > 0:
            raise SceneError(f"source {j} has non-positive weight", j)
        if abs(np.linalg.norm(s[3:6]) - 1.0) > 1e-12:
            raise SceneError(f"source {j} direction is not a unit vector", j)
        sep = separation(sc.origin, sc.spacing, sc.dims, s[0:3])
        if sep < 2.0 * sc.spacing:
            raise SceneError(f"source {j} violates the separation guard: distance {sep} m < 2h", j)


def make_loop_scene(radius, center, n_segments, grid, op=0, k0=0.0, q=3):
    """make_loop_scene (src/scene.cpp:177-202): tangential edges in the x-z plane."""
    if n_segments < 3:
        raise ContractViolation(CONTRACT_VIOLATION, "make_loop_scene: need at least 3 segments")
    chord = 2.0 * radius * math.sin(math.pi / n_segments)
    src = np.zeros((n_segments, 7))
    for s in range(n_segments):
        th = 2.0 * math.pi * (s + 0.5) / n_segments
        src[s, 0:3] = np.asarray(center) + radius * np.array([math.cos(th), 0.0, math.sin(th)])
        src[s, 3:6] = [-math.sin(th), 0.0, math.cos(th)]
        src[s, 6] = chord
    sc = Scene(grid[0], grid[1], grid[2], src, op, k0, q)
    validate_scene(sc)
    return sc


def make_plate_scene(side, center, edges_per_side, grid, op=0, k0=0.0, q=3):
    """make_plate_scene (src/scene.cpp:204-231)."""
    pitch = side / edges_per_side
    src = []
    for a in range(edges_per_side):
        for b in range(edges_per_side):
            u = pitch * (a + 0.5) - 0.5 * side
            w = pitch * (b + 0.5) - 0.5 * side
            d = [1, 0, 0] if (a + b) % 2 == 0 else [0, 0, 1]
            src.append(list(np.asarray(center) + np.array([u, 0.0, w])) + d + [pitch])
    sc = Scene(grid[0], grid[1], grid[2], np.array(src, np.float64), op, k0, q)
    validate_scene(sc)
    return sc


def _scene_args(sc):
    return (np.ascontiguousarray(sc.origin, np.float64), float(sc.spacing), np.array(sc.dims, np.int64),
            np.ascontiguousarray(sc.sources, np.float64))


def assemble_column(sc, j):
    """assemble_column (src/scene.cpp:127-150) as one component-major vector (q n_v)."""
    o, h, d, s = _scene_args(sc)
    out = np.zeros(sc.rows, np.complex128)
    _check(lib().orc_assemble_column(_ptr(o), h, _ptr(d), sc.op, sc.k0, sc.q, _ptr(s), sc.num_sources, j, _ptr(out)))
    return out


def assemble_full(sc, workers=None, mem_cap_bytes=4 << 30):
    """assemble_full (src/scene.cpp:156-175): dense (q n_v x m), Fortran order."""
    nbytes = 16 * sc.rows * sc.num_sources
    if nbytes > mem_cap_bytes:
        raise OracleError(CAPACITY_ERROR, f"assemble_full: dense matrix needs {nbytes} bytes")
    o, h, d, s = _scene_args(sc)
    out = np.zeros((sc.rows, sc.num_sources), np.complex128, order="F")
    _check(lib().orc_assemble_full(_ptr(o), h, _ptr(d), sc.op, sc.k0, sc.q, _ptr(s), sc.num_sources,
                                   workers or default_workers(), _ptr(out)))
    return out


def dense_forward(sc, x):
    """dense_forward (src/matvec.cpp:177-186)."""
    x = _fortran_c128(x)
    if x.shape[0] != sc.num_sources:
        raise ContractViolation(CONTRACT_VIOLATION, "dense_forward: x rows mismatch")
    return assemble_full(sc) @ x


def dense_adjoint(sc, phi):
    """dense_adjoint (src/matvec.cpp:188-196)."""
    phi = _fortran_c128(phi)
    if phi.shape[0] != sc.rows:
        raise ContractViolation(CONTRACT_VIOLATION, "dense_adjoint: phi rows mismatch")
    return assemble_full(sc).conj().T @ phi


def eval_kernel(op, k0, src7, obs):
    out = np.zeros(6)
    s = np.ascontiguousarray(src7, np.float64)
    o = np.ascontiguousarray(obs, np.float64)
    _check(lib().orc_eval_kernel(op, k0, _ptr(s), _ptr(o), _ptr(out)))
    return out[0::2] + 1j * out[1::2]


# ----------------------------------------------------------------- HOSVD --
def unfold(t, mode):
    """unfold (src/tensor.cpp:67-87): mode-g rows, remaining modes in increasing order as columns."""
    n1, n2, n3 = t.shape
    if mode == 1:
        return t.reshape((n1, n2 * n3), order="F")
    if mode == 2:
        return np.transpose(t, (1, 0, 2)).reshape((n2, n1 * n3), order="F")
    return t.reshape((n1 * n2, n3), order="F").T


def hosvd(t, eps):
    """Truncated HOSVD (src/tensor.cpp:122-174): per mode keep the smallest rank
    whose discarded energy stays below eps^2/3 |t|^2; a (near-)zero tensor is a
    rank-(1,1,1) zero core with e1 factors."""
    if not 0.0 < eps < 1.0:
        raise ContractViolation(CONTRACT_VIOLATION, "hosvd: eps must lie in (0,1)")
    t = np.asarray(t, np.complex128)
    fro = float(np.linalg.norm(t))
    dims = t.shape
    if fro < 1e-300:
        core = np.zeros((1, 1, 1), np.complex128)
        us = []
        for g in range(3):
            u = np.zeros((dims[g], 1), np.complex128)
            u[0, 0] = 1.0
            us.append(u)
        return core, us[0], us[1], us[2]
    budget = (eps * eps / 3.0) * fro * fro
    us = []
    for mode in (1, 2, 3):
        a = unfold(t, mode)
        u, sv, _ = np.linalg.svd(a, full_matrices=False)
        r = sv.size
        discarded = 0.0
        while r > 1:
            nxt = discarded + sv[r - 1] * sv[r - 1]
            if nxt > budget:
                break
            discarded = nxt
            r -= 1
        us.append(np.asfortranarray(u[:, :r]))
    core = np.einsum("abc,ai,bj,ck->ijk", t, us[0].conj(), us[1].conj(), us[2].conj(), optimize=True)
    return np.asfortranarray(core), us[0], us[1], us[2]


def compress_matrix(sc, eps, workers=None):
    """compress_matrix (src/compress.cpp:7-35): assemble each column, HOSVD each of its q tensors."""
    if not 0.0 < eps < 1.0:
        raise ContractViolation(CONTRACT_VIOLATION, "compress_matrix: eps must lie in (0,1)")
    validate_scene(sc)
    nv = sc.num_voxels
    dims = tuple(sc.dims)

    def one(j):
        col = assemble_column(sc, j)
        return [hosvd(col[k * nv:(k + 1) * nv].reshape(dims, order="F"), eps) for k in range(sc.q)]

    with ThreadPoolExecutor(max_workers=workers or default_workers()) as ex:
        cols = list(ex.map(one, range(sc.num_sources)))
    ranks, payload = pack_tensors([t for c in cols for t in c])
    return Compressed(dims, sc.q, sc.num_sources, ranks.reshape(sc.num_sources, sc.q, 3), payload, sc.op, sc.k0,
                      eps)


def householder_q(a):
    """Thin orthonormal basis of a's columns (Eigen::HouseholderQR ... * Identity)."""
    q, _ = np.linalg.qr(a)
    return np.asfortranarray(q)


def synthetic_compression(n, m, rank, seed, q=3):
    """Uniform-rank store with random cores and QR-orthonormal factors
    (reference tests/test_compress.cpp:21-45)."""
    dims = tuple(n) if isinstance(n, (tuple, list)) else (n, n, n)
    rk = tuple(rank) if isinstance(rank, (tuple, list)) else (rank, rank, rank)
    s = seed
    tensors = []
    for _ in range(m):
        for _ in range(q):
            core = random_tensor(rk, s); s += 1
            us = []
            for g in range(3):
                us.append(householder_q(random_matrix(dims[g], rk[g], s))); s += 1
            tensors.append((core, us[0], us[1], us[2]))
    ranks, payload = pack_tensors(tensors)
    return Compressed(dims, q, m, ranks.reshape(m, q, 3), payload, 0, 1.0, 1e-8)


# ------------------------------------------------------------------- ACA --
@dataclass
class DenseAca:
    """AcaFactors with dense U (include/tuckmat/aca.hpp:24-41)."""
    u: np.ndarray
    v: np.ndarray
    eps: float = 0.0
    converged: bool = False
    final_stat: float = 0.0

    @property
    def rank(self):
        return int(self.v.shape[1])

    @property
    def rows(self):
        return int(self.u.shape[0])

    @property
    def cols(self):
        return int(self.v.shape[0])


_ZERO_PIVOT = 1e-300
_NOISE_FLOOR = 1e-14


def _next_pivot_row(x, used):
    ax = np.abs(x)
    ax[used] = 0.0
    return int(np.argmax(ax))


def aca_dense(row_fn, col_fn, m1, m2, eps=1e-3):
    """aca_dense (src/aca.cpp:54-124): partially pivoted ACA with dense U."""
    if not 0.0 < eps < 1.0:
        raise ContractViolation(CONTRACT_VIOLATION, "aca: eps must lie in (0,1)")
    kmax = min(m1, m2)
    us, vs = [], []
    used = np.zeros(m1, bool)
    i, s, row_scale = 0, 0.0, 0.0
    fac = DenseAca(np.zeros((m1, 0), np.complex128), np.zeros((m2, 0), np.complex128), eps)
    for k in range(kmax):
        exhausted = False
        while True:
            r = np.array(row_fn(i), np.complex128)
            row_scale = max(row_scale, float(np.max(np.abs(r))))
            if k > 0:
                r = r - np.array([u[i] for u in us]) @ np.array(vs).conj()
            j = int(np.argmax(np.abs(r)))
            rmax = abs(r[j])
            if rmax > max(_ZERO_PIVOT, _NOISE_FLOOR * row_scale):
                break
            if k > 0:
                exhausted = True
                break
            used[i] = True
            free = np.flatnonzero(~used)
            if free.size == 0:
                exhausted = True
                break
            i = int(free[0])
        if exhausted:
            fac.converged = True
            fac.final_stat = 0.0
            break
        y = (r / r[j]).conj()
        x = np.array(col_fn(j), np.complex128)
        if k > 0:
            U = np.array(us).T
            V = np.array(vs).T
            x = x - U @ V[j, :].conj()
        nx, ny = float(np.linalg.norm(x)), float(np.linalg.norm(y))
        s += (nx * ny) ** 2
        if k > 0:
            s += 2.0 * float(np.sum(((U.conj().T @ x) * (V.conj().T @ y)).real))
        us.append(x)
        vs.append(y)
        scale = math.sqrt(max(s, 0.0))
        fac.final_stat = nx * ny / scale if scale > 0 else 0.0
        fac.u = np.array(us).T
        fac.v = np.array(vs).T
        if nx * ny <= eps * scale:
            fac.converged = True
            break
        used[i] = True
        i = _next_pivot_row(x, used)
    return fac


def tucker_aca(row_fn, col_fn, m1, m2, grid_dims, q, eps=1e-3, hosvd_eps=0.0):
    """tucker_aca (Algorithm 3, src/aca.cpp:126-232): accepted columns are
    HOSVD-compressed per component; residual rows come from element-wise
    decompression and the residual column update runs through the compressed
    stacked_forward / stacked_adjoint products."""
    if not 0.0 < eps < 1.0:
        raise ContractViolation(CONTRACT_VIOLATION, "aca: eps must lie in (0,1)")
    if hosvd_eps <= 0.0:
        hosvd_eps = min(3.0 * eps, 0.99)
    nv = int(np.prod(grid_dims))
    if m1 != q * nv:
        raise ContractViolation(CONTRACT_VIOLATION, f"tucker_aca: oracle has {m1} rows, expected q*n_v = {q * nv}")
    kmax = min(m1, m2)
    dims = tuple(grid_dims)
    tensors = []  # [(l, k)] in l-major order
    vs = []
    used = np.zeros(m1, bool)
    i, s, row_scale = 0, 0.0, 0.0
    converged, final_stat = False, 0.0

    def current(k):
        ranks, payload = pack_tensors(tensors)
        return Compressed(dims, q, k, ranks.reshape(k, q, 3), payload)

    store = None
    for k in range(kmax):
        exhausted = False
        while True:
            r = np.array(row_fn(i), np.complex128)
            row_scale = max(row_scale, float(np.max(np.abs(r))))
            if k > 0:
                comp, v = divmod(i, nv)
                i1, rest = v % dims[0], v // dims[0]
                i2, i3 = rest % dims[1], rest // dims[1]
                t = np.array([store.element(l, comp, i1, i2, i3) for l in range(k)])
                r = r - t @ np.array(vs).conj()
            j = int(np.argmax(np.abs(r)))
            if abs(r[j]) > max(_ZERO_PIVOT, _NOISE_FLOOR * row_scale):
                break
            if k > 0:
                exhausted = True
                break
            used[i] = True
            free = np.flatnonzero(~used)
            if free.size == 0:
                exhausted = True
                break
            i = int(free[0])
        if exhausted:
            converged, final_stat = True, 0.0
            break
        y = (r / r[j]).conj()
        x = np.array(col_fn(j), np.complex128)
        if k > 0:
            V = np.array(vs).T
            x = x - store.forward(V[j, :].conj().reshape(-1, 1))[:, 0]
        nx, ny = float(np.linalg.norm(x)), float(np.linalg.norm(y))
        s += (nx * ny) ** 2
        if k > 0:
            s += 2.0 * float(np.sum((store.adjoint(x.reshape(-1, 1))[:, 0] * (V.conj().T @ y)).real))
        for comp in range(q):
            tensors.append(hosvd(x[comp * nv:(comp + 1) * nv].reshape(dims, order="F"), hosvd_eps))
        vs.append(y)
        store = OracleStore(current(k + 1))
        scale = math.sqrt(max(s, 0.0))
        final_stat = nx * ny / scale if scale > 0 else 0.0
        if nx * ny <= eps * scale:
            converged = True
            break
        used[i] = True
        i = _next_pivot_row(x, used)
    rc = len(vs)
    ranks, payload = pack_tensors(tensors)
    v = np.array(vs).T if rc else np.zeros((m2, 0), np.complex128)
    return Aca(dims, q, ranks.reshape(rc, q, 3), payload, np.asfortranarray(v), eps, hosvd_eps, converged, final_stat)


def coupling_oracle(sc):
    """coupling_oracle (src/aca.cpp:246-273): row / column providers of a scene."""
    validate_scene(sc)
    nv = sc.num_voxels

    def col(j):
        return assemble_column(sc, j)

    def row(i):
        comp, v = divmod(i, nv)
        i1, rest = v % sc.dims[0], v // sc.dims[0]
        i2, i3 = rest % sc.dims[1], rest // sc.dims[1]
        if sc.q == 3:
            obs = sc.origin + sc.spacing * (np.array([i1, i2, i3], float) + 0.5)
            return np.array([eval_kernel(sc.op, sc.k0, s, obs)[comp] for s in sc.sources])
        # PWL rows: one-voxel sub-scene per source (slow path, tests only)
        sub = Scene(sc.origin + sc.spacing * np.array([i1, i2, i3], float), sc.spacing, (1, 1, 1), sc.sources,
                    sc.op, sc.k0, 12)
        return assemble_full(sub, workers=1)[comp, :]

    return row, col, sc.rows, sc.num_sources


# -------------------------------------------------------------------- io --
_KVERSION = 1


def _write_header(buf, tag, q, m, dims, k0, eps, op):
    buf += tag
    buf += struct.pack("<IIIIIIddB", _KVERSION, q, m, dims[0], dims[1], dims[2], k0, eps, op)


def save_ctc1(path, cc):
    """save_ctc1 (src/io.cpp:198-210): 45-byte header, then per tensor r1 r2 r3 u32 + f64 pairs."""
    buf = bytearray()
    _write_header(buf, b"CTC1", cc.q, cc.m, cc.grid_dims, cc.k0, cc.eps, cc.kernel_op)
    off = tensor_offsets(cc.grid_dims, cc.ranks)
    rk = np.asarray(cc.ranks, np.uint32).reshape(-1, 3)
    pay = np.asarray(cc.payload, np.complex128)
    for i in range(rk.shape[0]):
        buf += rk[i].astype("<u4").tobytes()
        buf += pay[off[i]:off[i + 1]].astype("<c16").tobytes()
    with open(path, "wb") as f:
        f.write(buf)


def _read_header(data, tag):
    if len(data) < 4:
        raise ParseError("truncated while reading magic", 0)
    if data[:4] != tag:
        raise ParseError(f"bad magic, expected {tag.decode()}", 0)
    if len(data) < 45:
        raise ParseError("truncated while reading header", 4)
    version, q, m, n1, n2, n3, k0, eps, op = struct.unpack_from("<IIIIIIddB", data, 4)
    if version != _KVERSION:
        raise ParseError(f"unsupported version {version}", 8)
    if q < 1 or m < 1 or min(n1, n2, n3) < 1:
        raise ParseError("non-positive header dimensions", 45)
    if op > 1:
        raise ParseError(f"unknown kernel id {op}", 45)
    return q, m, (n1, n2, n3), k0, eps, op


def _read_tensors(data, pos, count, dims):
    ranks = np.zeros((count, 3), np.int32)
    parts = []
    n = np.array(dims)
    for i in range(count):
        if len(data) - pos < 12:
            raise ParseError("truncated while reading u32", pos)
        r = struct.unpack_from("<III", data, pos)
        for g in range(3):
            if r[g] == 0 or r[g] > dims[g]:
                raise ParseError(f"tucker rank {r[g]} out of range for mode {g + 1}", pos + 4 * (g + 1))
        pos += 12
        cnt = r[0] * r[1] * r[2] + int(np.dot(r, n))
        if len(data) - pos < 16 * cnt:
            raise ParseError("truncated while reading f64", pos)
        parts.append(np.frombuffer(data, "<c16", cnt, pos))
        pos += 16 * cnt
        ranks[i] = r
    payload = np.concatenate(parts).astype(np.complex128) if parts else np.zeros(0, np.complex128)
    return ranks, payload, pos


def load_ctc1(path):
    """load_ctc1 (src/io.cpp:212-230)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ParseError(f"cannot open '{path}'", 0)
    q, m, dims, k0, eps, op = _read_header(data, b"CTC1")
    ranks, payload, pos = _read_tensors(data, 45, m * q, dims)
    if pos != len(data):
        raise ParseError(f"{len(data) - pos} trailing bytes", pos)
    return Compressed(dims, q, m, ranks.reshape(m, q, 3), payload, op, k0, eps)


def save_cta1(path, fac, k0, op):
    """save_cta1 (src/io.cpp:232-247): CTC1 payload of the U store, then V column-major."""
    buf = bytearray()
    _write_header(buf, b"CTA1", fac.q, fac.rank, fac.grid_dims, k0, fac.eps, op)
    off = tensor_offsets(fac.grid_dims, fac.ranks)
    rk = np.asarray(fac.ranks, np.uint32).reshape(-1, 3)
    for i in range(rk.shape[0]):
        buf += rk[i].astype("<u4").tobytes()
        buf += np.asarray(fac.payload[off[i]:off[i + 1]], np.complex128).astype("<c16").tobytes()
    buf += np.asfortranarray(fac.v, np.complex128).ravel(order="F").astype("<c16").tobytes()
    with open(path, "wb") as f:
        f.write(buf)


def load_cta1(path):
    """load_cta1 (src/io.cpp:249-279): m2 recovered from the remaining length."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ParseError(f"cannot open '{path}'", 0)
    q, rc, dims, k0, eps, op = _read_header(data, b"CTA1")
    ranks, payload, pos = _read_tensors(data, 45, rc * q, dims)
    rest = len(data) - pos
    col_bytes = 16 * rc
    if col_bytes == 0 or rest % col_bytes != 0 or rest // col_bytes == 0:
        raise ParseError(f"V block of {rest} bytes is not a positive multiple of 16*r_c", pos)
    m2 = rest // col_bytes
    v = np.frombuffer(data, "<c16", m2 * rc, pos).reshape((m2, rc), order="F").astype(np.complex128)
    fac = Aca(dims, q, ranks.reshape(rc, q, 3), payload, np.asfortranarray(v), eps)
    return fac, k0, op


def rel_err(a, b):
    """Relative Frobenius error |a-b| / |b| (src/experiments.cpp:547-548)."""
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))
