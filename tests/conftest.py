"""Shared test setup: markers, import path, golden-vector loaders."""

from __future__ import annotations

import hashlib
import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200); runs the engine kernels")


def digest(obj) -> str:
    """sha256 of the canonical JSON (same recipe as make_golden.py)."""
    return hashlib.sha256(json.dumps(obj, sort_keys=True,
                                     separators=(",", ":")).encode()).hexdigest()


@lru_cache(maxsize=None)
def golden(name: str) -> dict:
    return json.loads((GOLDEN / name).read_text())


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except ImportError:
        return False


@pytest.fixture(scope="session")
def require_gpu():
    if not cuda_available():
        pytest.skip("needs a CUDA device")
