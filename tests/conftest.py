import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    """The reference compiled from /root/reference (oracle/_ref); skips where it
    was never built."""
    import oracle
    r = oracle.reference()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not available on this host")
    return r


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_1411_3656_b200 import _lib
    _lib.load()
    return torch.device("cuda:0")


def max_err_over_rms(got, want):
    """The north-star metric: max |got - want| / RMS(want) over complex outputs."""
    g = np.asarray(got).reshape(-1).view(np.complex64).astype(np.complex128)
    w = np.asarray(want).reshape(-1).view(np.complex64).astype(np.complex128)
    rms = np.sqrt(np.mean(np.abs(w) ** 2)) if w.size else 0.0
    d = np.max(np.abs(g - w)) if w.size else 0.0
    return d / rms if rms > 0 else d


def bits(a):
    return np.ascontiguousarray(a).reshape(-1).view(np.uint32)


def uniform(rng, n_complex):
    return rng.uniform(-1.0, 1.0, size=2 * n_complex).astype(np.float32).view(np.complex64)
