"""Shared test plumbing.

Markers: ``gpu`` tests need a B200 (run with ``-m gpu`` on the box); everything
else runs on CPU.  The oracle (``oracle/moe_oracle.py``) is the checker; the
golden fixtures in ``tests/golden`` pin it to the real reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN_DIR = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and libparm_b200.so")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices (torchrun)")


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN_DIR / "golden_meta.json").read_text())
    arrays = np.load(GOLDEN_DIR / "golden.npz")
    return meta, arrays


@pytest.fixture(scope="session")
def cuda_lib():
    """The CUDA path must be the one that runs: fail (never skip) when it is missing."""
    import torch

    from paper_2407_00599_b200 import _lib

    assert torch.cuda.is_available(), "gpu test needs a CUDA device"
    lib = _lib.load()
    return lib
