"""The C++ drop-in facade (include/fastmp_b200/fastmp.hpp, libfastmp_b200.so):
builds and links here (CPU), runs the reference's test recipes on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1205_4139_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "_test_facade")


def build_exe():
    src = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
    lib = os.path.join(PKG, "libfastmp_b200.so")
    cmd = ["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), src, "-o", EXE,
           lib, os.path.join(PKG, "libfmp_cuda.so"), "-ldl", f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_facade_builds_and_exports():
    exe = build_exe()
    assert os.path.exists(exe)
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(PKG, "libfastmp_b200.so")],
                         capture_output=True, text=True).stdout
    for sym in ("fastmp::omp_solve(", "fastmp::fast_update(", "fastmp::compute_kernel(",
                "fastmp::least_squares(", "fastmp::cosamp_solve(",
                "fastmp::save_instance(", "fastmp::load_instance(", "fastmp::save_result(",
                "fastmp::IncrementalQR::push_column(", "fastmp::IncrementalQR::solve(", "fastmp::SensingOperator::apply_adjoint("):
        assert sym in out, sym


@pytest.mark.gpu
def test_facade_reference_recipes(oracle):
    exe = build_exe()
    r = subprocess.run([exe, os.path.join(ROOT, "oracle", "_build", "libfmp_oracle.so"),
                        os.path.join(ROOT, "tests", "golden")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
