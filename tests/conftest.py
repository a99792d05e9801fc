"""Shared pytest configuration.

Markers:
  gpu — needs a CUDA device (run on the B200 box: ``pytest -m gpu``).
Everything else runs on CPU (``pytest -m "not gpu"``).
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200)")


@pytest.fixture(scope="session")
def orc():
    """The plain-C restatement (oracle/liboracle.so) — the checker."""
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref). Skips if it was never
    built (no /root/reference and no prebuilt .so)."""
    from oracle.oracle import Reference
    try:
        return Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def sg():
    """The product package; GPU tests fail loudly if the library or the GPU
    is missing (no fallback)."""
    import paper_1902_09931_b200 as pkg
    from paper_1902_09931_b200 import _lib
    _lib.check(_lib.lib().sg_init(0))
    return pkg
