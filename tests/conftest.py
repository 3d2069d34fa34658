import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

try:
    from hypothesis import settings
    settings.register_profile("spdnn", deadline=None, max_examples=40)
    settings.load_profile("spdnn")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: minutes of CPU work")


def random_layer(rng, n, max_row_nnz, allow_negative=True, values=None):
    """Random canonical CSR layer, the reference's fixture recipe
    (tests/conftest.py:35-52 of the reference)."""
    from paper_2007_14152_b200.model import make_layer_csr
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(0, max_row_nnz + 1))
        if k == 0:
            continue
        c = rng.choice(n, size=min(k, n), replace=False)
        rows.extend([r] * len(c))
        cols.extend(c.tolist())
    if values is None:
        vals = rng.uniform(0.01, 1.0, size=len(rows)).astype(np.float32)
        if allow_negative:
            vals *= rng.choice([-1.0, 1.0], size=len(vals)).astype(np.float32)
    else:
        vals = np.full(len(rows), values, dtype=np.float32)
    return make_layer_csr(n, np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), vals)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
