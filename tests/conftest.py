"""Shared fixtures.  GPU tests carry @pytest.mark.gpu (driver: -m gpu on a B200)."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
INITS = ["zero", "constant:0.7,-0.3,0.25", "shear:1.5", "taylor-green", "random:1"]
SMALL_DIMS = [(1, 1, 1), (2, 2, 2), (3, 2, 1), (3, 3, 3), (4, 4, 4)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device; run with -m gpu")


def dims_key(dims):
    return "x".join(map(str, dims))


def init_key(spec):
    return spec.split(":")[0]


@pytest.fixture(scope="session")
def golden_small():
    return np.load(GOLDEN / "rhs_small.npz")


@pytest.fixture(scope="session")
def golden_meshes():
    return np.load(GOLDEN / "meshes.npz")


@pytest.fixture(scope="session")
def golden_mid():
    return np.load(GOLDEN / "rhs_mid.npz")


@pytest.fixture(scope="session")
def golden_checksums():
    return np.load(GOLDEN / "checksums.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O
