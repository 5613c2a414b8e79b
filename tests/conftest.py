"""Shared fixtures. GPU tests carry ``@pytest.mark.gpu``; everything else runs
on CPU. Golden fixtures come from ``tests/golden/make_goldens.py`` (run once
in the build container against the reference)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long CPU test")


def load_golden(name):
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.skip(f"golden fixture {path.name} not generated")
    with np.load(path, allow_pickle=False) as data:
        return {k: data[k] for k in data.files}


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get


def _ensure_library():
    """Rebuild lib/libjgs2.so if any CUDA source is newer (no-op otherwise)."""
    try:
        from paper_2506_06494_b200 import build
        build.build()
    except Exception as exc:  # nvcc missing: tests that need the library fail loudly
        print(f"[conftest] library build skipped: {exc}")


_ensure_library()
