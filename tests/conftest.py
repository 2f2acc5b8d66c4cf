"""Shared test setup.

Markers: `gpu` = needs a real B200 (run on the box with `pytest -m gpu`);
everything else runs on the CPU container with `pytest -m "not gpu"`.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA GPU (B200)")


def _ensure_built():
    from oracle import bindings
    if not bindings.PORT_LIB.exists():
        bindings.build()
    from paper_1406_2628_b200 import build as nb
    if not nb.LIB.exists():
        nb.build()


_ensure_built()


@pytest.fixture(scope="session")
def kats():
    return json.loads((GOLDEN / "kats.json").read_text())


@pytest.fixture(scope="session")
def fixtures():
    return np.load(GOLDEN / "ref_fixtures.npz")


@pytest.fixture(scope="session")
def port():
    from oracle import bindings
    return bindings.port()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.fixture(autouse=True)
def _release_torch_cache():
    """The library allocates scratch from its own CUDA pool, which cannot
    reuse blocks torch's caching allocator keeps after a test (a full-size
    torch.sort leaves tens of GB cached): hand them back after every test so
    a later mp_sort / mp_merge never sees an out-of-memory that only the
    suite's order caused."""
    yield
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


def element_array(keys, tag_base=0):
    from oracle.bindings import ELEMENT_DTYPE
    e = np.zeros(len(keys), dtype=ELEMENT_DTYPE)
    e["key"] = np.asarray(keys, dtype=np.int64)
    e["tag"] = np.arange(tag_base, tag_base + len(keys), dtype=np.uint32)
    return e


def fixture_cases(fx, kind="m"):
    """Yield (S, case_id) for every recorded merge ('m') or sort ('s') case."""
    seen = set()
    for k in fx.files:
        parts = k.split("/")
        if len(parts) == 3 and parts[1].startswith(kind) and parts[1][1:].isdigit():
            if (parts[0], parts[1]) not in seen:
                seen.add((parts[0], parts[1]))
    return sorted(seen)


def same(x, y) -> bool:
    """Bit equality; `element` padding is not part of the value."""
    from oracle.bindings import ELEMENT_DTYPE
    x, y = np.asarray(x), np.asarray(y)
    if x.dtype == ELEMENT_DTYPE or y.dtype == ELEMENT_DTYPE:
        return (np.array_equal(x["key"], y["key"]) and np.array_equal(x["tag"], y["tag"]))
    return x.tobytes() == y.tobytes()


os.environ.setdefault("PYTHONHASHSEED", "0")
