import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built libsdmk_b200.so")


def golden_index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def golden_case(name):
    meta = next(c for c in golden_index() if c["name"] == name)
    data = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    with open(os.path.join(GOLDEN, f"{name}.tree.txt")) as f:
        dump = f.read()
    return meta, data, dump


def parity_ok(u, ref, rtol=1e-10, floor=1e-3):
    """|u - ref| <= rtol * max(|ref|, floor * ||ref||_inf) per component."""
    u, ref = np.asarray(u), np.asarray(ref)
    scale = np.max(np.abs(ref)) if ref.size else 0.0
    err = np.abs(u - ref)
    bound = rtol * np.maximum(np.abs(ref), floor * scale)
    return bool(np.all(err <= bound)), float(np.max(err / np.maximum(bound, 1e-300)) * rtol) if ref.size else 0.0


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_2509_21471_b200 as g
    return g.Context(0)
