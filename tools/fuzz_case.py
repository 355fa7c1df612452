import sys, os, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from helpers import ragged_store, cn01
from test_gpu_fuzz import _case
import paper_2103_06393_b200 as P
from oracle import oracle as O
seed = int(sys.argv[1])
dims, q, m, rmin, rmax, dtype, p = _case(seed)
cc = ragged_store(dims, q, m, rmin, rmax, seed=seed)
ds = P.DeviceStore.from_compressed(cc, dtype)
ref = O.OracleStore(cc.rounded_c64() if dtype == "c64" else cc)
x = cn01(m, p, 3 + seed).astype(np.complex64).astype(np.complex128)
phi = cn01(cc.rows, p, 5 + seed).astype(np.complex64).astype(np.complex128)
y = ds.forward(x); print("fwd", np.linalg.norm(y - ref.forward(x)) / np.linalg.norm(ref.forward(x)), flush=True)
z = ds.adjoint(phi); print("adj", np.linalg.norm(z - ref.adjoint(phi)) / np.linalg.norm(ref.adjoint(phi)), flush=True)
