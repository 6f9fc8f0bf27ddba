import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def hp_from(g, prefix=""):
    return dict(family=str(g[prefix + "family"]), s2=float(g[prefix + "s2"]),
                ls=np.atleast_1d(g[prefix + "ls"]).astype(np.float64),
                noise=float(g[prefix + "noise"]),
                mean=float(g[prefix + "mean"]) if prefix + "mean" in g else 0.0)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
