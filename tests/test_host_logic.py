"""Host-side logic of the CUDA path that needs no GPU: the trailing-update tile
enumeration (SyrkMap: every lower 128-block of the requested column range exactly
once, pointers consistent with the panel layout), compiled with nvcc as host code; and
the MLE's quadratic-model trust-region minimiser (trust_region.h) on functions with known
minimisers (box-active optimum, +inf region, Rosenbrock), compiled with g++."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_syrkmap_enumeration(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "test_syrkmap")
    subprocess.check_call([nvcc, "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I",
                           os.path.join(ROOT, "paper_1708_02835_b200", "csrc"), "-o", exe,
                           os.path.join(ROOT, "tools", "test_syrkmap.cu")])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK")


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_2d_block_cyclic_layout_and_enumeration(tmp_path):
    """P x Q grids (2x1, 2x2, 2x4, 4x2, 3x2, 4x1, 8x1, 2x3): local panel offsets, tile ownership
    (I mod P, J mod Q), every lower tile stored once, and the Syrk2DMap enumeration with its
    A/B/C pointers for every rank and step (tools/test_syrk2d.cu)."""
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "test_syrk2d")
    subprocess.check_call([nvcc, "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I",
                           os.path.join(ROOT, "paper_1708_02835_b200", "csrc"), "-o", exe,
                           os.path.join(ROOT, "tools", "test_syrk2d.cu")])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK")


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_trust_region_minimiser(tmp_path):
    exe = str(tmp_path / "test_trust_region")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", exe, os.path.join(ROOT, "tools", "test_trust_region.cpp")])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count(" ok") == 8, out.stdout
