"""The drop-in C++ API (include/sparseforge_b200/sparseforge.hpp): reference
style code compiles against it (CPU) and matches the reference goldens (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2403_05802_b200", "_lib")


def build(tmp_path):
    exe = str(tmp_path / "test_api")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lsfg", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                   check=True, capture_output=True, text=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs_on_gpu(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe, os.path.join(ROOT, "tests", "golden", "mm")], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout
