"""The tcgen05 operand layouts and descriptors the kernels use (umma.cuh):
scripts/micro/umma_test.cu builds the three MMA patterns of hog3tm (T = U3 G,
g3 = P G, dG = P^T S) from K-major no-swizzle tiles and checks them against a
host GEMM on the device."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_umma_descriptor_patterns(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "umma_test")
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                        "-I", os.path.join(ROOT, "paper_1708_08640_b200", "csrc"),
                        os.path.join(ROOT, "scripts", "micro", "umma_test.cu"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "UMMA descriptors: ok" in r.stdout, r.stdout + r.stderr
