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
def test_consumer_runs_with_parity(tmp_path, oracle):
    """The consumer's results, checked against the CPU oracle (not against this library's own
    gemm_oracle): quantize_tensor bytes and scales and reshuffle bytes bit-exact; gemm_auto
    (fused path) bit-exact with the oracle's gemm_fused; the device tensor-core linear within
    1e-5 of the f64 oracle on f16-rounded scales."""
    import numpy as np
    from oracle import KERNEL
    exe = build(tmp_path)
    out = tmp_path / "dump"
    out.mkdir()
    p = subprocess.run([exe, str(out)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    n, k, m = 384, 1024, 4
    ld = lambda name, dt: np.fromfile(out / name, dtype=dt)  # noqa: E731
    w, a = ld("w.f32", np.float32).reshape(n, k), ld("a.f32", np.float32).reshape(m, k)
    codes, scales = oracle.quantize(w, 4, 128)
    assert np.array_equal(ld("q_data.u8", np.uint8), oracle.pack(codes, 4))
    assert np.array_equal(ld("q_scales.f32", np.float32).reshape(n, -1), scales)
    kern = oracle.encode(codes, 4, KERNEL)
    assert np.array_equal(ld("qk_data.u8", np.uint8), kern)
    fused = oracle.gemm_fused(a, kern, n, 4, 128, scales)
    assert np.array_equal(ld("gemm_auto.f32", np.float32).view(np.uint32), fused.ravel().view(np.uint32))
    assert np.array_equal(ld("gemm_oracle.f32", np.float32), oracle.gemm_oracle(a, codes, 128, scales).ravel())
    s16 = oracle.f16_round(scales).view(np.float16).astype(np.float32)
    ref = oracle.gemm_oracle_f64(a, codes, 128, s16)
    dev = ld("device_linear.f32", np.float32).reshape(m, n).astype(np.float64)
    assert np.linalg.norm(dev - ref) / np.linalg.norm(ref) <= 1e-5
