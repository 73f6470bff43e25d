"""Shared pytest wiring.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz")

    return load


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    # The oracle's C restatement is test infrastructure; build it if missing.
    from oracle import build

    build.build_oracle()
    build.build_ref()
    build.build_ref_pkg()

