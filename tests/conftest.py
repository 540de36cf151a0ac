import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden_qg():
    z = np.load(os.path.join(GOLDEN, "quant_gemm.npz"))
    cases = {}
    for name in z["names"]:
        cases[str(name)] = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/")}
    return cases


@pytest.fixture(scope="session")
def golden_f16():
    return np.load(os.path.join(GOLDEN, "f16.npz"))


@pytest.fixture(scope="session")
def golden_plan():
    return np.load(os.path.join(GOLDEN, "plan.npz"))


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _cases(fname):
    z = np.load(os.path.join(GOLDEN, fname))
    return {str(n): {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{n}/")}
            for n in z["names"]}


@pytest.fixture(scope="session")
def golden_ties():
    """f32 near-tie quantize fixtures (tests/golden/make_golden_r2.py)."""
    return _cases("quant_f32ties.npz")


@pytest.fixture(scope="session")
def golden_gemm_float():
    """gemm_float fixtures (tests/golden/make_golden_r2.py)."""
    return _cases("gemm_float.npz")
