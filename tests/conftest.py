import os
import sys

import hypothesis
import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")

# same profile as the reference's tests (pkg/tests/conftest.py:5-7)
hypothesis.settings.register_profile("default", max_examples=25, deadline=None, derandomize=True)
hypothesis.settings.load_profile("default")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsphb.so")
    config.addinivalue_line("markers", "slow: full-size configuration")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def checkpoints(g, tag, field):
    """Steps at which a fixture stores `field` (1, 100 and the last step)."""
    pre = f"{tag}__{field}"
    return sorted(int(k[len(pre):]) for k in g
                  if k.startswith(pre) and k[len(pre):].isdigit())


@pytest.fixture(scope="session")
def gold():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = golden(name)
        return cache[name]

    return get


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
