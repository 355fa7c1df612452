"""The C ABI library on a host without a GPU: loads, exports every symbol the
header declares, validates arguments with the reference's error taxonomy,
parses CTC1 / CTA1 natively, and fails loudly (no CPU fallback) once it needs
the device.  Also builds and runs the C++ drop-in (include/tuckmat_b200/tuckmat.hpp)."""
import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT, has_cuda

HEADER = os.path.join(ROOT, "include", "tuckmat_b200.h")
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"TM_API\s+[\w\s\*]+?\b(tm_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(product):
    from paper_2103_06393_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 12
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    assert set(_lib.EXPORTED) <= set(syms)
    assert L.tm_version() == 1
    assert _lib.launch_count() >= 0


def test_nm_exports_match_header(product):
    from paper_2103_06393_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tm_\w+)", out))
    assert set(declared_symbols()) <= exported


def _desc(dims, q, ranks, payload):
    from paper_2103_06393_b200._lib import StoreDesc
    d = StoreDesc()
    d.q = q
    d.ncols = ranks.shape[0] // q
    for g in range(3):
        d.dims[g] = dims[g]
    d.ranks = ranks.ctypes.data
    d.payload = payload.ctypes.data
    return d


def test_store_validation_errors(product):
    from paper_2103_06393_b200._lib import TM_CONTRACT_VIOLATION, lib
    L = lib()
    h = ctypes.c_void_p()
    ranks = np.array([[3, 3, 9]], np.int32)  # r3 = 9 > n3 = 4: out of range
    pay = np.zeros(200, np.complex128)
    d = _desc((4, 4, 4), 1, ranks, pay)
    assert L.tm_store_create(ctypes.byref(d), 0, 0, ctypes.byref(h)) == TM_CONTRACT_VIOLATION
    assert b"out of range for mode 3" in L.tm_last_error()
    d.dims[0] = 0
    assert L.tm_store_create(ctypes.byref(d), 0, 0, ctypes.byref(h)) == TM_CONTRACT_VIOLATION
    assert L.tm_store_create(ctypes.byref(d), 0, 7, ctypes.byref(h)) == TM_CONTRACT_VIOLATION  # bad dtype
    assert L.tm_forward(None, None, 1, 1, 1, None, 1, 0, None, None) == TM_CONTRACT_VIOLATION


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(product, oracle):
    """Without a device every compute path fails loudly."""
    P = product
    cc = oracle.synthetic_compression(5, 2, 2, 1)
    with pytest.raises(P.CudaError):
        P.DeviceStore.from_compressed(cc, "c64")
    with pytest.raises(P.CudaError):
        P.load_ctc1(os.path.join(GOLD, "loop8.ctc1"))  # parses fine, then needs the device


def test_native_ctc1_parse_errors(product, tmp_path):
    """ParseError with byte offsets, as tuckmat::ParseError (src/io.cpp:44-119)."""
    P = product
    with pytest.raises(P.ParseError) as e:
        P.load_ctc1(str(tmp_path / "missing.ctc1"))
    assert e.value.byte_offset == 0
    bad = tmp_path / "bad.ctc1"
    bad.write_bytes(b"NOPE12345678")
    with pytest.raises(P.ParseError, match="bad magic"):
        P.load_ctc1(str(bad))
    data = open(os.path.join(GOLD, "loop8.ctc1"), "rb").read()
    t = tmp_path / "t.ctc1"
    t.write_bytes(data[:1000])
    with pytest.raises(P.ParseError) as e:
        P.load_ctc1(str(t))
    assert e.value.byte_offset > 45
    t.write_bytes(data + b"\x01\x02")
    with pytest.raises(P.ParseError, match="2 trailing bytes"):
        P.load_ctc1(str(t))
    v = bytearray(data)
    v[4] = 2  # version
    t.write_bytes(bytes(v))
    with pytest.raises(P.ParseError, match="unsupported version"):
        P.load_ctc1(str(t))
    cta = open(os.path.join(GOLD, "aca8.cta1"), "rb").read()
    t.write_bytes(cta[:-8])
    with pytest.raises(P.ParseError, match="V block"):
        P.load_cta1(str(t))


DROPIN_TEST = r"""
#include <cstdio>
#include <tuckmat_b200/tuckmat.hpp>
int main(int argc, char** argv) {
    using namespace tuckmat;
    CompressedCoupling cc = load_ctc1(argv[1]);
    std::printf("loaded m=%lld q=%d rows=%lld\n", (long long)cc.m, cc.q, (long long)cc.rows());
    try {
        forward(cc, MultiVector(cc.m + 1, 1));
        return 3;
    } catch (const ContractViolation& e) {
        std::printf("contract: %s\n", e.what());
    }
    try {
        load_ctc1(std::string(argv[1]) + ".missing");
        return 4;
    } catch (const ParseError& e) {
        std::printf("parse: offset %llu\n", (unsigned long long)e.byte_offset);
    }
    MultiVector x(cc.m, 2);
    for (Index j = 0; j < cc.m; ++j) x(j, 0) = x(j, 1) = Complex(1.0, -0.5 * j);
    OpCounts ops;
    try {
        MultiVector y = forward(cc, x, 1, &ops);
        std::printf("gpu forward ok rows=%lld norm=%.17g dec=%lld\n", (long long)y.rows(), y.norm(),
                    (long long)ops.decompress_madds);
        MultiVector z = adjoint(cc, y, 1, &ops);
        std::printf("gpu adjoint ok norm=%.17g\n", z.norm());
        const Complex e = element(cc.columns[3][1], 2, 5, 7);
        std::printf("element %.17g %.17g\n", e.real(), e.imag());
        try {
            element(cc.columns[3][1], 2, 5, 99);
            return 6;
        } catch (const ContractViolation& e2) {
            std::printf("contract: %s\n", e2.what());
        }
    } catch (const Error& e) {
        std::printf("device error: %s\n", e.what());
        return 5;
    }
    return 0;
}
"""


def build_dropin_test(tmp_path):
    from paper_2103_06393_b200 import _lib
    src = tmp_path / "dropin.cpp"
    src.write_text(DROPIN_TEST)
    exe = tmp_path / "dropin"
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe), _lib.LIB_PATH,
           f"-Wl,-rpath,{libdir}", "-lpthread"]
    subprocess.run(cmd, check=True)
    return exe


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_dropin_compiles_and_validates(product, tmp_path):
    exe = build_dropin_test(tmp_path)
    r = subprocess.run([str(exe), os.path.join(GOLD, "loop8.ctc1")], capture_output=True, text=True)
    assert "loaded m=10 q=3 rows=1536" in r.stdout
    assert "contract: forward: x has 11 rows, expected m = 10" in r.stdout
    assert "parse: offset 0" in r.stdout
    if has_cuda():
        assert r.returncode == 0, r.stdout + r.stderr
    else:
        assert r.returncode == 5 and "device error" in r.stdout  # no CPU fallback


def test_row_partition_rule_matches_python(product):
    """tm_shard_row_cuts (the C ABI's row-sharding partition) and
    sharded.row_pieces implement the same rule: identical cuts on random
    component costs, grid heights, device counts, alignments and minimum
    piece heights; every piece honours the alignment / minimum-height rule."""
    from paper_2103_06393_b200.multigpu import row_cuts
    from paper_2103_06393_b200.sharded import row_pieces
    rng = np.random.default_rng(0)
    for _ in range(500):
        q, n1, nd = int(rng.integers(1, 14)), int(rng.integers(1, 300)), int(rng.integers(1, 10))
        cc = rng.random(q) * float(rng.choice([1.0, 1e6, 1e12]))
        al, mr = int(rng.choice([1, 4, 8])), int(rng.integers(1, 40))
        cuts = row_cuts(cc, n1, nd, al, mr)
        pcs = row_pieces(cc, n1, nd, al, mr)
        want = np.cumsum([0] + [sum(b - a for _, a, b in p) for p in pcs])
        assert list(cuts) == list(want)
        assert cuts[0] == 0 and cuts[-1] == q * n1 and np.all(np.diff(cuts) >= 0)
        for p in pcs:
            for k, a, b in p:
                for e in (a, b):  # a cut inside a component: aligned, >= max(min_rows, align) from both ends
                    if 0 < e < n1:
                        assert e % al == 0 and min(e, n1 - e) >= max(mr, al)
