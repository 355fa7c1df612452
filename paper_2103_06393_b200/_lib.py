"""ctypes binding of the C ABI (include/tuckmat_b200.h).

Loads the in-tree ``libtuckmat_b200.so``.  There is no fallback: if the
library is missing or cannot be loaded the import of the product path fails
loudly.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtuckmat_b200.so")
# A/B experiments: load an alternative in-tree build (e.g. libtuckmat_b200_a.so)
if os.environ.get("TMB_LIB_VARIANT"):
    LIB_PATH = os.path.join(HERE, "libtuckmat_b200_%s.so" % os.environ["TMB_LIB_VARIANT"])

TM_OK, TM_CONTRACT_VIOLATION, TM_CAPACITY_ERROR, TM_PARSE_ERROR, TM_CUDA_ERROR, TM_ERROR = 0, 1, 2, 3, 6, 9
TM_SINGULARITY_ERROR = 4
TM_C64, TM_C128 = 0, 1
TM_HOST, TM_DEVICE = 0, 1
TM_SHARD_COLUMNS, TM_SHARD_ROWS = 0, 1

EXPORTED = [
    "tm_store_create", "tm_store_create_dense_aca", "tm_store_load_ctc1", "tm_store_load_cta1", "tm_store_destroy", "tm_store_info", "tm_store_kernels",
    "tm_forward", "tm_forward_components", "tm_adjoint", "tm_aca_forward", "tm_aca_adjoint", "tm_opcounts", "tm_rows", "tm_last_error",
    "tm_assemble_columns",
    "tm_comm_init", "tm_comm_finalize", "tm_comm_info", "tm_sharded_create", "tm_sharded_destroy", "tm_sharded_info",
    "tm_sharded_forward", "tm_sharded_adjoint", "tm_sharded_aca_forward", "tm_sharded_aca_adjoint",
    "tm_sharded_create_mode", "tm_sharded_pieces", "tm_shard_row_cuts",
    "tm_launch_count", "tm_version",
]


class StoreDesc(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_int32),
        ("ncols", ctypes.c_int64),
        ("dims", ctypes.c_int64 * 3),
        ("ranks", ctypes.c_void_p),
        ("payload", ctypes.c_void_p),
        ("payload_on_device", ctypes.c_int32),
        ("v", ctypes.c_void_p),
        ("m2", ctypes.c_int64),
        ("v_on_device", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library (raises if it is not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2103_06393_b200.build` "
                    "(or __graft_entry__.build()); there is no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
            L.tm_store_create.argtypes = [ctypes.POINTER(StoreDesc), i32, i32, ctypes.POINTER(vp)]
            L.tm_store_load_ctc1.argtypes = [ctypes.c_char_p, i32, i32, ctypes.POINTER(vp)]
            L.tm_store_load_cta1.argtypes = [ctypes.c_char_p, i32, i32, ctypes.POINTER(vp)]
            if hasattr(L, "tm_store_create_dense_aca"):  # (older A/B variants lack the newer entry points)
                L.tm_store_create_dense_aca.argtypes = [vp, i64, vp, i64, i64, i32, i32, i32, ctypes.POINTER(vp)]
            L.tm_store_destroy.argtypes = [vp]
            L.tm_store_info.argtypes = [vp, vp, vp, vp, vp, vp, vp]
            if hasattr(L, "tm_store_kernels"):
                L.tm_store_kernels.argtypes = [vp, vp, vp]
            L.tm_forward.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp, vp]
            L.tm_adjoint.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp, vp]
            if hasattr(L, "tm_forward_components"):
                L.tm_forward_components.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, i32, vp]
            L.tm_aca_forward.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp]
            L.tm_aca_adjoint.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp]
            L.tm_opcounts.argtypes = [vp, i64, vp, vp]
            L.tm_rows.argtypes = [vp, vp, i64, vp, i64, i32, vp]
            L.tm_assemble_columns.argtypes = [vp, ctypes.c_double, vp, i32, i32, ctypes.c_double, vp, i64, vp, i64,
                                              vp, vp]
            if hasattr(L, "tm_comm_init"):
                L.tm_comm_init.argtypes = [i32, vp, ctypes.POINTER(vp)]
                L.tm_comm_finalize.argtypes = [vp]
                L.tm_comm_info.argtypes = [vp, vp, vp]
                L.tm_sharded_create.argtypes = [ctypes.POINTER(StoreDesc), vp, i32, ctypes.POINTER(vp)]
                L.tm_sharded_destroy.argtypes = [vp]
                L.tm_sharded_info.argtypes = [vp, vp, vp, vp]
                L.tm_sharded_forward.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp, vp]
                L.tm_sharded_adjoint.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp, vp]
                L.tm_sharded_aca_forward.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp]
                L.tm_sharded_aca_adjoint.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, vp]
                L.tm_sharded_create_mode.argtypes = [ctypes.POINTER(StoreDesc), vp, i32, i32, ctypes.POINTER(vp)]
                L.tm_sharded_pieces.argtypes = [vp, vp, vp]
                L.tm_shard_row_cuts.argtypes = [i32, i64, i32, i64, i64, vp, vp]
            L.tm_last_error.restype = ctypes.c_char_p
            L.tm_launch_count.restype = ctypes.c_int64
            _lib = L
    return _lib


def launch_count():
    return int(lib().tm_launch_count())
