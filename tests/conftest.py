import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "glu_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.build()
    return O.Oracle()


@pytest.fixture(scope="session")
def reference():
    import oracle as O
    O.build()
    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref/libglu_ref.so not built (needs /root/reference at build time)")
    return O.Reference()


@pytest.fixture(scope="session")
def glu():
    """The CUDA product path; fails loudly (no skip) when a GPU test runs without it."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2307_09582_b200 import build as B
    if not os.path.exists(B.CUDA_SO):
        B.build()
    import paper_2307_09582_b200 as G
    G._native.lib()  # raises if the native library cannot be loaded
    return G
