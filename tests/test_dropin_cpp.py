"""The drop-in C++ headers rebuild a reference-style consumer unchanged.

tests/cpp/dropin_example.cpp uses the reference API (quantize_tensor, reshuffle,
gemm_auto, gemm_oracle -- proj/README.md:156-167) plus rtnq/device.hpp, and links
only librtnq_b200.so.  CPU: it compiles and links.  GPU: it runs and checks parity.
"""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
PKG = os.path.join(ROOT, "paper_2505_15909_b200")


def build(tmp_path):
    exe = str(tmp_path / "dropin_example")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
           "-I/usr/local/cuda/include", "-L", PKG, "-lrtnq_b200", "-L/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{PKG}", "-o", exe]
    p = subprocess.run(cmd, capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    return exe


def test_consumer_compiles_against_dropin_headers(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_consumer_runs_with_parity(tmp_path):
    exe = build(tmp_path)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
