import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def ops_golden():
    return dict(np.load(GOLDEN / "ops.npz"))


@pytest.fixture(scope="session")
def steps_golden():
    return dict(np.load(GOLDEN / "steps.npz")), json.loads((GOLDEN / "steps_plans.json").read_text())


@pytest.fixture(scope="session")
def c1_digest():
    return json.loads((GOLDEN / "c1_digest.json").read_text())
