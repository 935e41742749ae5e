"""The header-only C++ layer compiles against include/ and links the C ABI
library; on a GPU box the same binary trains a small bundle."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "abi_smoke.cpp")
LIBDIR = os.path.join(ROOT, "paper_1708_08640_b200")


def build(tmp_path):
    from paper_1708_08640_b200 import _abi
    _abi.lib()  # builds the library if needed
    exe = str(tmp_path / "abi_smoke")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                        "-L", LIBDIR, "-lcmtf_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_layer_compiles_and_links(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    # 0 on a GPU box, 3 (CudaError: no device) here -- never a CPU fallback
    assert r.returncode in (0, 3), r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_layer_trains_on_gpu(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "trained 3 epochs" in r.stdout
