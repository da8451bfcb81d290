import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
GRIDS = GOLDEN / "grids"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libosph.so")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / name)

    return load


@pytest.fixture(scope="session")
def grid_of():
    from paper_1403_4661_b200 import load_grid

    cache = {}

    def get(L, ordering="condmin"):
        key = (L, ordering)
        if key not in cache:
            cache[key] = load_grid(GRIDS / f"grid-L{L}-uniform-{ordering}.txt")
        return cache[key]

    return get


@pytest.fixture
def rng():
    return np.random.default_rng(20240901)


@pytest.fixture(autouse=True, scope="module")
def _release_gpu_memory():
    """Cached plans (get_plan) of one test module can hold tens of GB of factor
    storage at L >= 2048; free them between modules so large-L tests see the
    whole GPU, as a fresh process would."""
    yield
    if not has_gpu():
        return
    import torch

    import paper_1403_4661_b200 as osp

    osp.clear_plans()
    torch.cuda.empty_cache()


@pytest.fixture
def fresh_gpu():
    """Drop cached plans and torch's cached blocks before a large-L test."""
    import torch

    import paper_1403_4661_b200 as osp

    osp.clear_plans()
    torch.cuda.empty_cache()
