"""The C++ drop-in header (include/dreg_b200/dreg.hpp) used the way a reference `dreg`
client uses the original library (tests/cpp/reference_style.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "reference_style.cpp")
LIBDIR = os.path.join(ROOT, "paper_2109_12688_b200", "lib")


def build(out):
    subprocess.run(
        ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
         f"-L{LIBDIR}", "-ldreg_cuda", f"-Wl,-rpath,{LIBDIR}", "-o", out],
        check=True,
    )


def test_header_compiles_and_links(tmp_path):
    build(str(tmp_path / "client"))


@pytest.mark.gpu
def test_reference_style_client_runs(tmp_path):
    exe = str(tmp_path / "client")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "OK" in r.stdout
