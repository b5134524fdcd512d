"""Shared fixtures.  Tests marked ``gpu`` need a B200 (run with -m gpu); the
rest run on CPU (oracle vs goldens, host logic, ABI surface, gloo multi-rank)."""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


def h2f(h: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


def h2a(hs) -> np.ndarray:
    return np.array([h2f(h) for h in hs], dtype=np.float64)


def f2h(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def same_bits(a, b) -> bool:
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    return a.shape == b.shape and bool(np.all(a.view(np.uint64) == b.view(np.uint64)))


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def ctx():
    import paper_2202_01753_b200 as M

    return M.Context(0)


def words_value(words) -> list:
    """Exact integers denoted by an exchange buffer ([accumulator][MCB_XWORDS]
    radix-2^32 digit sums, after the MCB_XHEADER count words of a run's
    buffer: overflowed addends, finite samples, non-finite samples).
    Different partitions carry between words at different points, so compare
    VALUES, not word vectors."""
    a = np.asarray(words).astype(np.uint64)
    out = []
    if a.size % 67 == 3:  # a run's exchange buffer: [3 count words][accumulators]
        out += [int(v) for v in a[:3]]
        a = a[3:]
    a = a.reshape(-1, 67)
    for row in a:
        v = 0
        for i in range(66, -1, -1):
            v = (v << 32) + int(row[i])
        out.append(v)
    return out
