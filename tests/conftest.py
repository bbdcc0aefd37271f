"""Shared fixtures.  `-m gpu` tests need a B200 and the built engine; every
other test runs on CPU (oracle vs golden vectors, host logic, C ABI symbols,
gloo multi-process paths)."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: long-running")


def decode_matrix(d):
    if d["kind"] == "int":
        return np.array(d["v"], dtype=np.int64)
    if d["kind"] == "float":
        return np.array(d["v"], dtype=np.float64)
    return np.array(d["re"], dtype=np.float64) + 1j * np.array(d["im"], dtype=np.float64)


def decode_value(v):
    if isinstance(v, dict):
        if "int" in v:
            return int(v["int"])
        if "float" in v:
            return float(v["float"])
        return complex(v["re"], v["im"])
    return v


def parity_case(c):
    """(matrix, algorithm, expected) from a parity.json entry."""
    if c["dtype"] == "int":
        a = np.array(c["matrix"], dtype=np.int64)
        exp = int(c["expected"]["value"])
    elif c["dtype"] == "float":
        a = np.array(c["matrix"], dtype=np.float64)
        exp = float(c["expected"]["value"])
    else:
        a = np.array([[complex(e["re"], e["im"]) for e in row] for row in c["matrix"]])
        exp = complex(c["expected"]["re"], c["expected"]["im"])
    return a, c["algorithm"], exp


@pytest.fixture(scope="session")
def parity_cases():
    return json.loads((GOLDEN / "parity.json").read_text())


@pytest.fixture(scope="session")
def ref_cases():
    return json.loads((GOLDEN / "ref_cases.json").read_text())


@pytest.fixture(scope="session")
def ref_int_walk():
    return json.loads((GOLDEN / "ref_int_walk.json").read_text())


@pytest.fixture
def rng():
    return np.random.default_rng(20240613)


def rel_err(x, y):
    """Metric (i) of SURVEY 8(c): |x-y| / max(|x|, |y|, 1e-300)."""
    return abs(x - y) / max(abs(x), abs(y), 1e-300)


def scaled_err(x, y, M):
    """Metric (ii): |x-y| / max(|x|, |y|, M), M = Glynn magnitude sum."""
    return abs(x - y) / max(abs(x), abs(y), M, 1e-300)
