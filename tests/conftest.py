import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product CUDA path")


@pytest.fixture(scope="session")
def golden_bounds():
    with open(os.path.join(GOLDEN, "bounds_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_objective():
    with open(os.path.join(GOLDEN, "objective_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_solver():
    with open(os.path.join(GOLDEN, "solver_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gosma():
    """The product package; GPU tests only (it has no CPU path)."""
    import paper_1812_01232_b200 as g
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return g
