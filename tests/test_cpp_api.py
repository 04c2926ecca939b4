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


IO_SRC = os.path.join(ROOT, "tests", "cpp", "test_io.cpp")
IO_GOLDEN = os.path.join(ROOT, "tests", "golden", "io")


def build_io(tmp_path):
    exe = str(tmp_path / "test_io")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    IO_SRC, "-L", LIBDIR, "-lsfg", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                   check=True, capture_output=True, text=True)
    return exe


def test_io_text_utilities_match_reference(tmp_path):
    """write_matrix_market / write_vector_text / read_tns (io.hpp) byte-for-byte
    and message-for-message against the reference's outputs (host only)."""
    exe = build_io(tmp_path)
    out = subprocess.run([exe, IO_GOLDEN, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_io_dense_round_trips_on_gpu(tmp_path):
    exe = build_io(tmp_path)
    out = subprocess.run([exe, IO_GOLDEN, str(tmp_path), "--gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout
