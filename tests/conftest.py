import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_ref():
    import oracle

    if not oracle.available("ref"):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return oracle.Oracle("ref")


@pytest.fixture(scope="session")
def oracle_port():
    import oracle

    if not oracle.available("port"):
        oracle.build()
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def checker():
    """The strongest available oracle: the reference library itself when it
    was built (it travels to the GPU box as a prebuilt .so), else the port."""
    import oracle

    if oracle.available("ref"):
        return oracle.Oracle("ref")
    if not oracle.available("port"):
        oracle.build()
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def gpu_ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1404_0424_b200 import Context

    return Context(0)


def cplx_randn(rng, shape, var=1.0):
    return ((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(var / 2))
