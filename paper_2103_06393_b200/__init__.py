"""B200-native Tucker-compressed VSIE coupling matvec (arXiv 2103.06393 hot path).

Product = ``libtuckmat_b200.so`` (C ABI ``include/tuckmat_b200.h``, CUDA
kernels for sm_100a, C++ drop-in ``include/tuckmat_b200/tuckmat.hpp``); this
package is its Python face plus the multi-GPU column sharding.
"""
from .matvec import (CapacityError, ContractViolation, CudaError, DeviceStore, Error, OpCounts, ParseError,
                     aca_adjoint, aca_forward, adjoint, forward, load_cta1, load_ctc1)
from ._lib import LIB_PATH, launch_count

__all__ = [
    "DeviceStore", "OpCounts", "forward", "adjoint", "aca_forward", "aca_adjoint", "load_ctc1", "load_cta1",
    "Error", "ContractViolation", "CapacityError", "ParseError", "CudaError", "LIB_PATH", "launch_count",
]
