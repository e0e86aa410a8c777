"""CPU tests of the boundary: the C-ABI library loads, exports every symbol
include/fmp.h declares, its host-side generators match the reference's,
and the product package refuses to run without its CUDA library."""
import os
import re
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(fmp_[a-z0-9_]+)\s*\(", txt)))


def _exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_library_exports_every_declared_symbol(fmp):
    names = _declared("fmp.h")
    assert len(names) >= 25
    missing = [n for n in names if n not in _exported(fmp.LIB_PATH)]
    assert not missing, missing


def test_library_loads_without_gpu(fmp):
    assert fmp._lib.fmp_version() == 1
    assert fmp.crossover_iteration("fourier", 4096) == 11
    assert fmp.crossover_iteration("hadamard", 65536) == 17
    assert fmp.crossover_iteration("fourier", 1 << 24) == 21


def test_host_generators_match_reference(fmp, oracle):
    # make_row_selection / derive_seed / make_instance draw order (sensing.cpp:119-153)
    for n, m, s in ((128, 32, 7), (4096, 1024, 99)):
        assert np.array_equal(fmp.make_row_selection(n, m, s), oracle.make_row_selection(n, m, s))
    for b, i in ((0, 1), (7, 9), (2024, 1 << 40)):
        assert fmp.derive_seed(b, i) == oracle.derive_seed(b, i)
    for kind in ("fourier", "hadamard"):
        n, m, k = 256, 64, 6
        om = oracle.make_row_selection(n, m, 5)
        Y, X, nn = fmp.make_batch(kind, n, om, k, 3, base_seed=11, noise_stddev=0.05, want_x=True)
        for b in range(3):
            x, y, e = oracle.make_instance(kind, n, om, k, 0.05, oracle.derive_seed(11, b))
            assert np.array_equal(X[b], x)
            assert np.abs(Y[b] - y).max() < 1e-12
            assert abs(nn[b] - np.linalg.norm(e)) < 1e-12
        Y, X, _ = fmp.make_batch(kind, n, om, k, 2, base_seed=3, real=True, want_x=True)
        for b in range(2):
            x, y = oracle.make_real_instance(kind, n, om, k, oracle.derive_seed(3, b))
            assert np.array_equal(X[b], x)
            assert np.abs(Y[b] - y).max() < 1e-12


def test_package_fails_loudly_without_library(tmp_path):
    pkg = tmp_path / "paper_1205_4139_b200"
    pkg.mkdir()
    src = open(os.path.join(ROOT, "paper_1205_4139_b200", "__init__.py")).read()
    (pkg / "__init__.py").write_text(src)
    r = subprocess.run([sys.executable, "-c", "import paper_1205_4139_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "libfmp_cuda.so is missing" in r.stderr


def test_sm100a_code_in_library(fmp):
    out = subprocess.run(["cuobjdump", "--list-elf", fmp.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
