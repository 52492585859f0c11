"""Proxy orders above the DMMA kernels' range (p = 33..64, 3D and 2D: the
Gaussian-window and eps <= 1e-10 rows of the plan table, params.cpp:21-38)
against the compiled reference: tree dump, upward pass, incoming(1), u."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2509_21471_b200 as g  # noqa: E402
from conftest import parity_ok  # noqa: E402
from oracle import ref  # noqa: E402

CASES = [  # kernel, dim, window, eps, n, n_s
    (0, 3, 0, 1e-13, 1500, 100),   # p = 48
    (0, 3, 1, 1e-10, 1500, 100),   # p = 48
    (1, 3, 1, 1e-10, 1200, 100),   # p = 50
    (2, 3, 1, 1e-12, 1200, 100),   # p = 53
    (0, 3, 1, 1e-12, 1200, 100),   # p = 58
    (1, 3, 1, 1e-12, 1000, 100),   # p = 60
    (0, 3, 1, 1e-13, 1000, 100),   # p = 63
    (0, 2, 1, 1e-13, 3000, 60),    # p = 63 (2D)
]
ctx = g.Context(0)
for kernel, dim, window, eps, n, n_s in CASES:
    rng = np.random.default_rng(5 + n + kernel)
    x = rng.uniform(-0.5, 0.5, (n, dim))
    s = rng.standard_normal((n, g.strength_components(kernel, dim)))
    plan = ref.select_parameters(kernel, eps, window, dim)
    plan["n_s"] = n_s
    row = {"kernel": kernel, "dim": dim, "window": window, "eps": eps, "n": n, "p": plan["p"], "N1": plan["N1"]}
    try:
        t0 = time.time()
        P = ref.RefProblem(plan, dim, x, s, None, False)
        ur, _ = P.evaluate()
        row["ref_s"] = round(time.time() - t0, 2)
        sys_ = g.ParticleSystem(dim, x, np.zeros(0), s)
        ctx.setup(g.DmkPlan(**plan), sys_, 0)
        row["tree_equal"] = ctx.tree_dump() == P.tree_dump()
        row["upward"] = parity_ok(ctx.upward_pass(), P.upward(), 1e-12)[1]
        row["incoming"] = parity_ok(ctx.incoming(1), P.incoming(1), 1e-11)[1]
        rep = {}
        u = ctx.evaluate_with_plan(g.DmkPlan(**plan), sys_, 0, rep)
        ok, err = parity_ok(u, ur, 1e-10)
        row.update(ok=ok, err=err, max_level=rep["max_level"], gpu_ms=round(rep["t_total"] * 1e3, 2))
    except Exception as e:  # noqa: BLE001
        row["error"] = f"{type(e).__name__}: {e}"
    print(json.dumps(row), flush=True)
