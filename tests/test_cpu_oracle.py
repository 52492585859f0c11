"""Pins the CPU oracle restatement (oracle/restate.py) before it is trusted.

1. Against the reference's own known-answer rows for select_parameters
   (test_dmk.cpp:89-167 of the reference test suite).
2. Against the committed golden vectors produced by the compiled reference
   (tests/golden/make_golden.py): tree dump text bit-exact, evaluate output.
3. Against the live compiled reference (oracle/_ref) when it is available.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_case, golden_index, parity_ok
from oracle import restate as R

# (kernel, eps, window, p, N1, N_per) -- the reference's plan pins (test_dmk.cpp:96-115)
PLAN_ROWS = [
    (0, 1e-3, 0, 12, 19, 3), (0, 1e-6, 0, 23, 33, 5), (0, 1e-9, 0, 33, 49, 9), (0, 1e-12, 0, 44, 61, 11),
    (0, 1e-3, 1, 14, 27, 5), (0, 1e-6, 1, 28, 49, 9), (0, 1e-9, 1, 43, 75, 13), (0, 1e-12, 1, 58, 99, 17),
    (1, 1e-3, 0, 11, 17, 3), (1, 1e-6, 0, 22, 33, 5), (1, 1e-9, 0, 33, 49, 9), (1, 1e-12, 0, 44, 63, 11),
    (1, 1e-9, 1, 44, 79, 13), (2, 1e-3, 0, 8, 13, 3), (2, 1e-6, 0, 18, 27, 5), (2, 1e-9, 0, 28, 39, 7),
    (2, 1e-12, 0, 39, 53, 9), (2, 1e-12, 1, 53, 93, 15),
]


@pytest.mark.parametrize("row", PLAN_ROWS)
@pytest.mark.parametrize("dim", [2, 3])
def test_plan_rows(row, dim):
    k, eps, w, p, n1, nper = row
    plan = R.select_parameters(k, eps, w, dim)
    assert (plan["p"], plan["N1"], plan["N_per"]) == (p, n1, nper)
    if w == 0:
        assert abs(plan["c"] - (n1 + 1) // 2 * np.pi / 3.0) <= 1e-12 * plan["c"]


def test_plan_leaf_sizes_and_errors():
    assert R.select_parameters(0, 1e-3, 0, 3)["n_s"] == 600
    assert R.select_parameters(0, 1e-6, 0, 3)["n_s"] == 1200
    assert R.select_parameters(0, 1e-9, 0, 3)["n_s"] == 2000
    assert R.select_parameters(0, 1e-12, 0, 3)["n_s"] == 3000
    assert R.select_parameters(2, 1e-3, 1, 2)["n_s"] == 120
    assert R.select_parameters(1, 1e-6, 0, 2)["n_s"] == 240
    for bad in [(0, 0.5, 0, 3), (0, 1e-14, 0, 3), (0, 1e-6, 0, 4)]:
        with pytest.raises(ValueError):
            R.select_parameters(*bad)


@pytest.mark.parametrize("name", [c["name"] for c in golden_index()])
def test_restatement_matches_golden(name):
    meta, d, dump = golden_case(name)
    plan = meta["plan"]
    dim = meta["dim"]
    tabs = R.load_tables(os.path.join(GOLDEN, f"{name}.tables.bin"))
    src = d["sources"]
    tgt = d["targets"] if meta["ntgt"] else None
    per = meta["periodic"]
    xs = R.wrap_into_box(src) if per else src
    xt = None if tgt is None else (R.wrap_into_box(tgt) if per else tgt)
    T = R.build_tree(xs, xt, plan["n_s"], dim, per, plan["p"])
    assert R.dump_tree(T) == dump
    assert np.array_equal(T["sperm"], d["sperm"])
    if meta["n"] <= 3000 and meta["num_boxes"] <= 300:
        u = R.evaluate_with_plan(plan, tabs, dim, src, d["strengths"], tgt, per)
        ok, err = parity_ok(u, d["u"], rtol=1e-10)
        assert ok, err


def test_restatement_residual_matches_golden():
    meta, d, _ = golden_case("stokeslet3d_cluster")
    plan = meta["plan"]
    tabs = R.load_tables(os.path.join(GOLDEN, "stokeslet3d_cluster.tables.bin"))
    T = R.build_tree(d["sources"], None, plan["n_s"], 3, False, plan["p"])
    ok, err = parity_ok(R.residual_pass(T, plan, tabs, d["strengths"]), d["residual"], 1e-11)
    assert ok, err


def test_direct_sum_accuracy_of_golden():
    """The golden DMK output is within eps of the exact direct sum (acceptance.cpp:451-474)."""
    meta, d, _ = golden_case("stokeslet3d_uniform")
    ex = R.direct_sum(0, 3, d["sources"], d["strengths"])
    rel = np.linalg.norm(d["u"] - ex) / np.linalg.norm(ex)
    assert rel < meta["eps"]


def test_restatement_vs_live_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(7)
    x = rng.uniform(-0.5, 0.5, (1500, 3))
    s = rng.standard_normal((1500, 3))
    plan = ref.select_parameters(2, 1e-6, 0, 3)
    plan["n_s"] = 120
    P = ref.RefProblem(plan, 3, x, s)
    P.export_tables("/tmp/_sdmk_live.bin")
    tabs = R.load_tables("/tmp/_sdmk_live.bin")
    u = R.evaluate_with_plan(plan, tabs, 3, x, s)
    ur, _ = P.evaluate()
    ok, err = parity_ok(u, ur, 1e-10)
    assert ok, err
