"""Shared fixtures; registers the ``gpu`` marker (tests needing a B200)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    class G:
        def npz(self, name):
            return np.load(GOLDEN / name, allow_pickle=False)

        def json(self, name):
            return json.loads((GOLDEN / name).read_text())

    return G()


@pytest.fixture(scope="session")
def oracle():
    import sfcdd_oracle

    return sfcdd_oracle


def pytest_collection_modifyitems(config, items):
    """GPU tests get a hard per-test timeout (thread method: a stuck CUDA call
    cannot hang the whole job; the DAG kernel's own watchdog traps first)."""
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(900, method="thread"))
