#!/usr/bin/env python
"""Generate the committed golden fixtures (test infrastructure).

The reference stores no golden vectors: every reference test
derives its expectations from seeds, dense assembly or loop oracles.  These
fixtures freeze, as files, inputs built exactly like the reference's own
matvec tests and the CPU oracle's outputs on them, so the GPU tests and the
oracle tests read identical bytes:

  loop8.ctc1   test_scene(8, 10, 0.8) of proj/tests/test_matvec.cpp:11-16,
               compress_matrix at eps 1e-6 (test_matvec.cpp:50-58)
  aca8.cta1    distant_loop(8, 12, 0.9) of proj/tests/test_aca.cpp:21-26,
               tucker_aca at eps 1e-4 (test_aca.cpp:102-140)
  pwl.ctc1     ragged random q = 12 store (PWL component count)
plus seeded x / phi blocks (the reference generator, src/experiments.cpp:26-33)
and the oracle's y = forward, z = adjoint (complex128, workers = 1), and the
dense-matrix products for the loop scene.  Run from the repo root:
    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402


def save(name, arr):
    np.save(os.path.join(HERE, name), arr)


def main():
    # loop scene, PWC q = 3, c128
    g = O.make_centered_grid((0, 0, 0), 0.05, (8, 8, 8))
    sc = O.make_loop_scene(0.5, (0, 0.8, 0), 10, g, 0, O.wavenumber_from_mhz(298.06), 3)
    cc = O.compress_matrix(sc, 1e-6, workers=1)
    O.save_ctc1(os.path.join(HERE, "loop8.ctc1"), cc)
    x = O.random_multivector(cc.m, 8, 31)
    phi = O.random_multivector(cc.rows, 8, 77)
    st = O.OracleStore(cc)
    save("loop8_x.npy", x)
    save("loop8_phi.npy", phi)
    save("loop8_y.npy", st.forward(x, 1))
    save("loop8_z.npy", st.adjoint(phi, 1))
    save("loop8_ydense.npy", O.dense_forward(sc, x))
    save("loop8_zdense.npy", O.dense_adjoint(sc, phi))

    # ACA store (CTA1), PWC q = 3
    g = O.make_centered_grid((0, 0, 0), 0.04, (8, 8, 8))
    sc2 = O.make_loop_scene(0.5, (0, 0.9, 0), 12, g, 0, O.wavenumber_from_mhz(123.0), 3)
    row, col, m1, m2 = O.coupling_oracle(sc2)
    fac = O.tucker_aca(row, col, m1, m2, sc2.dims, 3, 1e-4)
    O.save_cta1(os.path.join(HERE, "aca8.cta1"), fac, sc2.k0, sc2.op)
    xa = O.random_multivector(m2, 4, 17)
    pa = O.random_multivector(m1, 4, 18)
    save("aca8_x.npy", xa)
    save("aca8_phi.npy", pa)
    save("aca8_y.npy", O.aca_forward(fac, xa))
    save("aca8_z.npy", O.aca_adjoint(fac, pa))

    # ragged PWL-width store (q = 12); expectations on the c64-rounded factors
    from helpers import ragged_store
    pw = ragged_store((12, 9, 20), 12, 5, 1, 7, seed=2103)
    O.save_ctc1(os.path.join(HERE, "pwl.ctc1"), pw)
    r64 = pw.rounded_c64()
    xp = O.random_multivector(pw.m, 2, 5).astype(np.complex64).astype(np.complex128)
    pp = O.random_multivector(pw.rows, 2, 6).astype(np.complex64).astype(np.complex128)
    s64 = O.OracleStore(r64)
    save("pwl_x.npy", xp)
    save("pwl_phi.npy", pp)
    save("pwl_y64.npy", s64.forward(xp, 1))
    save("pwl_z64.npy", s64.adjoint(pp, 1))
    s128 = O.OracleStore(pw)
    save("pwl_y128.npy", s128.forward(xp, 1))
    save("pwl_z128.npy", s128.adjoint(pp, 1))

    manifest = {}
    for f in sorted(os.listdir(HERE)):
        if f.endswith((".npy", ".ctc1", ".cta1")):
            with open(os.path.join(HERE, f), "rb") as fh:
                manifest[f] = hashlib.sha256(fh.read()).hexdigest()
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print(f"wrote {len(manifest)} golden files; loop8 m={cc.m}, aca8 r_c={fac.rank}")


if __name__ == "__main__":
    main()
