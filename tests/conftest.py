"""Shared fixtures.  `-m "not gpu"` tests run in the build container (no GPU);
`-m gpu` tests need a B200 and call the CUDA path through the C-ABI."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers",
                            "gpu: needs a B200 (sm_100a) and libdynpar.so")


def _ensure_built():
    lib = ROOT / "paper_2201_02789_b200" / "csrc" / "libdynpar.so"
    if not lib.exists():
        subprocess.run(["make", "-s", "-C", str(lib.parent)], check=True)
    orc = ROOT / "oracle" / "liboracle.so"
    if not orc.exists():
        subprocess.run(["make", "-s", "-C", str(orc.parent)], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "reference_golden.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "reference_arrays.npz") as z:
        return {k: z[k] for k in z.files}
