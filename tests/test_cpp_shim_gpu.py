"""include/hetfuzz/*.hpp (the reference's C++ names over the C-ABI): compile a restatement of
the reference's own unit tests against it with g++ and run it on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(tmp):
    exe = os.path.join(tmp, "shim_test")
    lib_dir = os.path.join(ROOT, "paper_2603_12485_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), "-o", exe,
           "-L", lib_dir, "-l:libhfz.so", f"-Wl,-rpath,{lib_dir}"]
    subprocess.run(cmd, check=True)
    return exe


def test_shim_compiles(tmp_path):
    """CPU box: the headers are self-contained C++17 and link against libhfz.so."""
    assert os.path.exists(build(str(tmp_path)))


@pytest.mark.gpu
def test_shim_runs(tmp_path):
    exe = build(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
