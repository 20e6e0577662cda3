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
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
           SRC, "-o", exe, f"-L{LIB}", "-lspcv_b200", "-lspcv_cu", f"-Wl,-rpath,{LIB}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
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


MODEL_SRC = os.path.join(ROOT, "tests", "cpp", "test_model.cpp")


def build_model_test(tmp_path):
    exe = str(tmp_path / "test_model")
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", MODEL_SRC, "-o", exe,
           f"-L{LIB}", "-lspcv_b200", "-lspcv_cu", f"-Wl,-rpath,{LIB}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_model_dropin_compiles_and_links(tmp_path):
    build_model_test(tmp_path)


@pytest.mark.gpu
def test_model_dropin_run_network_bit_exact(tmp_path, ref):
    """spcv::DeviceModel::load + spcv::run_network (C++ mirror) reproduce the
    reference run_network's logits bit for bit; model errors are typed."""
    import numpy as np

    exe = build_model_test(tmp_path)
    data = ref.model_bytes("mbv2", 0.35, 0.8, 5)
    x = np.random.default_rng(2).uniform(-1, 1, (1, 224, 224, 3)).astype(np.float32)
    want = ref.run_model(data, x)
    (tmp_path / "m.spcv").write_bytes(data)
    (tmp_path / "x.f32").write_bytes(x.tobytes())
    (tmp_path / "y.f32").write_bytes(want.tobytes())
    r = subprocess.run([exe, str(tmp_path / "m.spcv"), str(tmp_path / "x.f32"), str(tmp_path / "y.f32")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all" in r.stdout
