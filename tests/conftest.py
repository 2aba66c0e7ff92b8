"""Shared pytest setup.

Markers: ``gpu`` -- needs a B200 and the built ``libpcnn.so``; the CPU suite
(``-m "not gpu"``) covers the oracle against the reference's golden vectors,
the host logic and the C-ABI symbol table.
"""

import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpcnn.so")


@pytest.fixture()
def rng() -> np.random.Generator:
    return np.random.default_rng(0)


@pytest.fixture(scope="session")
def golden():
    import json
    manifest = json.loads((GOLDEN / "manifest.json").read_text())
    arrays = dict(np.load(GOLDEN / "golden.npz"))
    return manifest, arrays


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
