"""Build the C++ re-expression of the reference hot-path tests against the
drop-in header and library; run it where a GPU exists."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1911_09723_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")


def build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT}/include", SRC, "-o", exe,
           f"-L{LIB}", "-lspcv_b200", "-lspcv_cu", f"-Wl,-rpath,{LIB}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_dropin_reference_tests_pass_on_device(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all" in r.stdout and "checks passed" in r.stdout
