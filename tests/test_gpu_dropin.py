"""The C++ drop-in (include/tuckmat_b200/tuckmat.hpp) on the GPU, value-checked:
a C++ program written against the reference API (forward, adjoint,
stacked_forward / stacked_adjoint over TuckerColumns, element,
aca_forward / aca_adjoint with Tucker and dense U, row_of_compressed_u,
load_ctc1 / load_cta1, and the multi-GPU ShardedStore by columns and by rows) runs on the committed golden fixtures and its outputs
are compared with the golden arrays (the oracle's, pinned to the reference
by tests/test_ref_pin_cpu.py) at 1e-12 (the drop-in's default is complex128).
It also rebuilds a CompressedCoupling with different values at the same
address in a loop — the content-keyed store cache must not serve stale data.
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")

PROG = r"""
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>
#include <tuckmat_b200/tuckmat.hpp>
using namespace tuckmat;

static MultiVector rd(const std::string& f, Index rows, Index cols) {
    MultiVector m(rows, cols);
    std::ifstream in(f, std::ios::binary);
    in.read(reinterpret_cast<char*>(m.data()), sizeof(Complex) * rows * cols);
    if (!in) { std::fprintf(stderr, "short read %s\n", f.c_str()); std::exit(9); }
    return m;
}
static void wr(const std::string& f, const MultiVector& m) {
    std::ofstream out(f, std::ios::binary);
    out.write(reinterpret_cast<const char*>(m.data()), sizeof(Complex) * m.rows() * m.cols());
}

int main(int argc, char** argv) {
    const std::string g = argv[1], o = argv[2];
    CompressedCoupling cc = load_ctc1(g + "/loop8.ctc1");
    MultiVector x = rd(o + "/x.bin", cc.m, 8), phi = rd(o + "/phi.bin", cc.rows(), 8);
    OpCounts ops;
    wr(o + "/y.bin", forward(cc, x, 1, &ops));
    wr(o + "/z.bin", adjoint(cc, phi, 4, &ops));
    std::printf("ops %lld %lld\n", (long long)ops.decompress_madds, (long long)ops.accumulate_madds);
    TuckerColumns z;
    z.tensor = [&](Index j, int k) -> const TuckerTensor& { return cc.columns[j][k]; };
    z.ncols = cc.m;
    z.q = cc.q;
    z.grid_dims = cc.grid_dims;
    wr(o + "/ys.bin", stacked_forward(z, x));
    wr(o + "/zs.bin", stacked_adjoint(z, phi));
    MultiVector el(1, 1);
    el(0, 0) = element(cc.columns[3][1], 2, 5, 7);
    wr(o + "/el.bin", el);

    Cta1File af = load_cta1(g + "/aca8.cta1");
    const AcaFactors& fac = af.factors;
    MultiVector xa = rd(o + "/xa.bin", fac.cols(), 4), pa = rd(o + "/pa.bin", fac.rows(), 4);
    wr(o + "/ya.bin", aca_forward(fac, xa));
    wr(o + "/za.bin", aca_adjoint(fac, pa));
    wr(o + "/row.bin", row_of_compressed_u(fac, 5));

    AcaFactors dense;
    dense.dense_u = rd(o + "/du.bin", 300, 7);
    dense.v = rd(o + "/dv.bin", 40, 7);
    wr(o + "/yd.bin", aca_forward(dense, rd(o + "/dx.bin", 40, 2)));
    wr(o + "/zd.bin", aca_adjoint(dense, rd(o + "/dp.bin", 300, 2)));

    // the columns sharded over an (emulated, one-GPU) two-shard communicator
    {
        b200::Communicator comm({0, 0});
        b200::ShardedStore ss(cc, comm);
        wr(o + "/ysh.bin", forward(ss, x));
        wr(o + "/zsh.bin", adjoint(ss, phi));
        b200::ShardedStore sa(fac, comm);
        wr(o + "/yash.bin", aca_forward(sa, xa));
        // row (voxel-slab) sharding
        b200::ShardedStore sr(cc, comm, TM_C128, TM_SHARD_ROWS);
        wr(o + "/ysr.bin", forward(sr, x));
        wr(o + "/zsr.bin", adjoint(sr, phi));
        b200::ShardedStore sar(fac, comm, TM_C128, TM_SHARD_ROWS);
        wr(o + "/yasr.bin", aca_forward(sar, xa));
        wr(o + "/zasr.bin", aca_adjoint(sar, pa));
    }

    // the same stack slot, different contents each iteration
    for (int it = 0; it < 3; ++it) {
        CompressedCoupling c2 = cc;
        for (auto& col : c2.columns)
            for (auto& tt : col)
                for (Index i = 0; i < tt.core.size(); ++i) tt.core[i] *= double(it + 1);
        wr(o + "/yit" + std::to_string(it) + ".bin", forward(c2, x));
    }
    return 0;
}
"""


def _w(path, a):
    np.asfortranarray(a, dtype=np.complex128).ravel(order="F").tofile(path)


def _r(path, rows, cols):
    return np.fromfile(path, dtype=np.complex128).reshape((rows, cols), order="F")


def test_cpp_dropin_values(product, oracle, tmp_path):
    from paper_2103_06393_b200 import _lib
    src = tmp_path / "prog.cpp"
    src.write_text(PROG)
    exe = tmp_path / "prog"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe), _lib.LIB_PATH,
                    f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}", "-lpthread"], check=True)
    ld = lambda f: np.load(os.path.join(GOLD, f))  # noqa: E731
    x, phi = ld("loop8_x.npy"), ld("loop8_phi.npy")
    xa, pa = ld("aca8_x.npy"), ld("aca8_phi.npy")
    rng = np.random.default_rng(4)
    du = rng.standard_normal((300, 7)) + 1j * rng.standard_normal((300, 7))
    dv = rng.standard_normal((40, 7)) + 1j * rng.standard_normal((40, 7))
    dx = rng.standard_normal((40, 2)) + 1j * rng.standard_normal((40, 2))
    dp = rng.standard_normal((300, 2)) + 1j * rng.standard_normal((300, 2))
    for name, a in (("x", x), ("phi", phi), ("xa", xa), ("pa", pa), ("du", du), ("dv", dv), ("dx", dx), ("dp", dp)):
        _w(str(tmp_path / f"{name}.bin"), a)
    r = subprocess.run([str(exe), GOLD, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    m, rows = x.shape[0], phi.shape[0]
    y, z = _r(tmp_path / "y.bin", rows, 8), _r(tmp_path / "z.bin", m, 8)
    assert rel(y, ld("loop8_y.npy")) <= 1e-12
    assert rel(z, ld("loop8_z.npy")) <= 1e-12
    assert rel(_r(tmp_path / "ys.bin", rows, 8), ld("loop8_y.npy")) <= 1e-12
    assert rel(_r(tmp_path / "zs.bin", m, 8), ld("loop8_z.npy")) <= 1e-12
    st = oracle.OracleStore(oracle.load_ctc1(os.path.join(GOLD, "loop8.ctc1")))
    want = st.element(3, 1, 2, 5, 7)
    assert abs(_r(tmp_path / "el.bin", 1, 1)[0, 0] - want) <= 1e-12 * abs(want)
    ops = {}
    st.forward(x, 1, ops)
    st.adjoint(phi, 1, ops)
    assert f"ops {ops['decompress_madds']} {ops['accumulate_madds']}" in r.stdout
    fac = oracle.load_cta1(os.path.join(GOLD, "aca8.cta1"))[0]
    assert rel(_r(tmp_path / "ya.bin", fac.rows, 4), ld("aca8_y.npy")) <= 1e-12
    assert rel(_r(tmp_path / "za.bin", fac.cols, 4), ld("aca8_z.npy")) <= 1e-12
    sa = oracle.OracleStore(fac.store())
    i = 5
    want = np.array([sa.element(l, 0, i % 8, (i // 8) % 8, i // 64) for l in range(fac.rank)])
    assert rel(_r(tmp_path / "row.bin", 1, fac.rank)[0], want) <= 1e-12
    assert rel(_r(tmp_path / "yd.bin", 300, 2), du @ (dv.conj().T @ dx)) <= 1e-12
    assert rel(_r(tmp_path / "zd.bin", 40, 2), dv @ (du.conj().T @ dp)) <= 1e-12
    assert rel(_r(tmp_path / "ysh.bin", rows, 8), ld("loop8_y.npy")) <= 1e-12
    assert rel(_r(tmp_path / "zsh.bin", m, 8), ld("loop8_z.npy")) <= 1e-12
    assert rel(_r(tmp_path / "yash.bin", fac.rows, 4), ld("aca8_y.npy")) <= 1e-12
    assert rel(_r(tmp_path / "ysr.bin", rows, 8), ld("loop8_y.npy")) <= 1e-12
    assert rel(_r(tmp_path / "zsr.bin", m, 8), ld("loop8_z.npy")) <= 1e-12
    assert rel(_r(tmp_path / "yasr.bin", fac.rows, 4), ld("aca8_y.npy")) <= 1e-12
    assert rel(_r(tmp_path / "zasr.bin", fac.cols, 4), ld("aca8_z.npy")) <= 1e-12
    for it in range(3):
        assert rel(_r(tmp_path / f"yit{it}.bin", rows, 8), (it + 1) * ld("loop8_y.npy")) <= 1e-12
