"""The drop-in C++ headers (include/pot/) compile against the reference's
own test code shapes and run on the GPU through libpotgpu.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2601_17196_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR,
                    "-lpotgpu", "-Wl,-rpath," + LIBDIR, "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_dropin_headers_compile_and_link(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_dropin_reference_tests_pass_on_gpu(tmp_path):
    exe = build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "OK (0 failures)" in res.stdout
