import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhmf.so")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden_sgd():
    g = np.load(GOLDEN / "sgd_range.npz")
    cases = {}
    for key in g.files:
        name, field = key.split("__")
        cases.setdefault(name, {})[field] = g[key]
    return cases


def random_matrix(n_users, n_items, nnz, seed, lo=1.0, hi=5.0):
    """Unique-pair coordinate matrix (same construction as the reference's
    tests/conftest.py:15-26)."""
    from paper_2006_15980_b200.data import RatingMatrix
    rng = np.random.default_rng(seed)
    chosen = rng.permutation(n_users * n_items)[:nnz]
    return RatingMatrix(n_users, n_items, (chosen // n_items).astype(np.int32),
                        (chosen % n_items).astype(np.int32), rng.uniform(lo, hi, size=nnz))
