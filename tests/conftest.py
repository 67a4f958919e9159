"""pytest configuration: `gpu` marker, repo on sys.path, shared helpers."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    g = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(g, "maps.json")) as f:
        meta = json.load(f)
    return {
        "lattice": dict(np.load(os.path.join(g, "lattice.npz"))),
        "maps": dict(np.load(os.path.join(g, "maps.npz"))),
        "maps_meta": meta,
        "analysis": dict(np.load(os.path.join(g, "analysis.npz"))),
    }
