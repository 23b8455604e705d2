"""Shared test plumbing: the ``gpu`` marker and golden-fixture loading."""

from __future__ import annotations

import functools
import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@functools.lru_cache(maxsize=None)
def golden(name: str):
    """Load ``tests/golden/<name>.npz`` fully into memory (cached)."""
    with np.load(GOLDEN / f"{name}.npz") as z:
        return _Frozen({k: z[k] for k in z.files})


class _Frozen(dict):
    @property
    def files(self):
        return list(self.keys())


REFERENCE_SRC = Path("/root/reference/pkg/src")
HAVE_REFERENCE = REFERENCE_SRC.is_dir() and os.environ.get("LSDF_NO_REFERENCE") != "1"


@pytest.fixture(scope="session")
def reference():
    """The real reference package (build container only; skipped elsewhere)."""
    if not HAVE_REFERENCE:
        pytest.skip("reference not mounted (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import linksdf

    return linksdf
