"""The C++ drop-in facade (include/phylograd_b200/engine.hpp): compiles against
the C-ABI library on CPU; runs the reference call pattern on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_facade_test(tmpdir):
    exe = os.path.join(str(tmpdir), "facade_test")
    libdir = os.path.join(ROOT, "paper_1905_12146_b200", "_build")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "facade_test.cpp"), "-L", libdir, "-lphylograd_b200",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(build_facade_test(tmp_path))


@pytest.mark.gpu
def test_facade_runs_reference_call_pattern(tmp_path):
    exe = build_facade_test(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
