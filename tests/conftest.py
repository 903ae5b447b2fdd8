import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"

# Parity tolerance of the north star: fp32 device results vs the fp64 oracle,
# per tensor max|a-b| / max(max|b|, floor).
TOL = 1e-4


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")


def max_rel(a, b, floor=1e-8):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(np.abs(b).max(), floor))


def load_golden(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def graph_cases():
    data = load_golden("graphs.npz")
    names = sorted({k.split("/")[0] for k in data if "/" in k})
    return data, names


@pytest.fixture(scope="session")
def graphs_golden():
    return graph_cases()
