"""Shared fixtures.  `gpu`-marked tests need a CUDA device (B200) and the
built libckf.so; everything else runs on a CPU-only box."""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden_v1.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libckf.so")
    config.addinivalue_line("markers", "slow: large-size GPU parity runs")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device on this host")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@lru_cache(maxsize=1)
def golden():
    z = np.load(GOLDEN)
    data = {k: z[k] for k in z.files}
    manifest = json.loads(bytes(data.pop("manifest")).decode())
    return data, manifest


@pytest.fixture(scope="session")
def gold():
    return golden()


def scenario_cfg(sc, cls):
    """FilterConfig (ours or the oracle's) of a golden scenario."""
    return cls(bucket_count=sc["m"], fingerprint_bits=sc["f"], bucket_slots=sc["b"],
               policy=sc["policy"], eviction=sc["eviction"], max_evictions=sc["max_evictions"],
               seed=sc["seed"])
