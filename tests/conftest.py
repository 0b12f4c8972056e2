import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    path = os.path.join(ROOT, "tests", "golden", "small_cases.npz")
    z = np.load(path)
    n = int(z["n_cases"])
    cases = []
    for i in range(n):
        pre = f"c{i}_"
        cases.append({k[len(pre):]: z[k] for k in z.files if k.startswith(pre)})
    return cases


@pytest.fixture(scope="session")
def digests():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "digests.json")) as f:
        return json.load(f)
