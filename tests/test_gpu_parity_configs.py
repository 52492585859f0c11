"""BASELINE cfg1 (N = 1e4 iid uniform, seed 0, 3D Stokeslet, eps = 1e-6) at its
full size against the compiled reference, through tools/parity_configs.py
(the same check profiles/round2/parity_full_size.jsonl records for every
BASELINE configuration): dump_tree text and permutations bit-exact, the
residual loop's in-support pair count exact, every pass (outgoing and
incoming proxies, far field, residual, u) within 1e-10 scaled per component
(SURVEY 8(d)), bitwise determinism, and the O(N^2) direct sum as the second
oracle (acceptance.cpp:451-474: the GPU's error against it equals the
reference's)."""
import os
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ref = pytest.importorskip("oracle.ref")
if not ref.available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_cfg1_full_size_parity(gpu_ctx):
    import parity_configs
    threads = ref.set_threads(os.cpu_count() or 1)
    line = parity_configs.run("cfg1", gpu_ctx, threads)
    assert line["tree_equal"] and line["perm_equal"]
    assert line["pairs_equal"], (line["ref_pairs"], line["gpu_pairs_in_support"])
    assert line["deterministic"]
    for k, v in line["max_scaled_err"].items():
        assert v <= 1e-10, (k, v)
    d = line["rel_l2_vs_direct"]
    assert d["gpu"] < 1e-6 and abs(d["gpu"] - d["ref"]) <= 1e-3 * d["ref"]
    assert line["pass"]
