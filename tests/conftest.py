import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "large: BASELINE-sized parity gates (minutes, host RAM)")


@pytest.fixture(scope="session")
def golden_index():
    return json.loads((GOLDEN / "index.json").read_text())


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def golden_names():
    idx = json.loads((GOLDEN / "index.json").read_text())
    return sorted(k for k in idx if not k.startswith("_"))
