"""Test configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs on the CPU (oracle vs reference goldens, host logic,
C-ABI exports, gloo slab exchange); `-m gpu` runs the parity tests proper on
a B200 through the C ABI.
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden_small.npz")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden_meta.json").read_text())


@pytest.fixture(scope="session")
def built():
    """Build the CUDA library and the C oracle once per session."""
    import __graft_entry__
    __graft_entry__.build()
    return True


def rel_linf(a, b) -> float:
    """tests/helpers.py:96-100 of the reference."""
    scale = np.max(np.abs(b))
    if scale == 0.0:
        return float(np.max(np.abs(a - b)))
    return float(np.max(np.abs(a - b)) / scale)
