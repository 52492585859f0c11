"""Per-pass GPU vs reference comparison (debug driver; uses the oracle)."""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402
from oracle import ref  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.max(np.abs(b)) if b.size else 1.0
    return float(np.max(np.abs(a - b)) / (s if s > 0 else 1.0)) if a.size else 0.0


def case(kernel, dim, n, eps, periodic=False, seed=0, ntgt=0, n_s=None, window=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5, 0.5, (n, dim))
    sc = g.strength_components(kernel, dim)
    s = rng.standard_normal((n, sc))
    if kernel == 1:
        nn = rng.standard_normal((n, dim))
        nn /= np.linalg.norm(nn, axis=1, keepdims=True)
        s[:, dim:] = nn
    t = rng.uniform(-0.5, 0.5, (ntgt, dim)) if ntgt else None
    plan = ref.select_parameters(kernel, eps, window, dim)
    if n_s:
        plan["n_s"] = n_s
    R = ref.RefProblem(plan, dim, x, s, t, periodic)
    ctx = g.Context(0)
    sys_ = g.ParticleSystem(dim, x, t if t is not None else np.zeros(0), s)
    P = g.DmkPlan(**plan)
    ctx.setup(P, sys_, 1 if periodic else 0)
    out = {"kernel": kernel, "dim": dim, "n": n, "eps": eps, "periodic": periodic, "boxes": R.info["num_boxes"],
           "levels": R.info["max_level"]}
    out["tree_equal"] = ctx.tree_dump() == R.tree_dump()
    sp, tp = ctx.tree_perm()
    rsp, rtp = R.tree_perm()
    out["perm_equal"] = bool(np.array_equal(sp, rsp)) and (tp is None or bool(np.array_equal(tp, rtp)))
    out["upward"] = rel(ctx.upward_pass(), R.upward())
    out["incoming0"] = rel(ctx.incoming(0), R.incoming(0))
    out["incoming1"] = rel(ctx.incoming(1), R.incoming(1))
    out["target_far"] = rel(ctx.target_far_fields(), R.target_far())
    out["residual"] = rel(ctx.residual_pass(), R.residual())
    t0 = time.time()
    ur, rep_ref = R.evaluate()
    t1 = time.time()
    rep = {}
    u = ctx.evaluate_with_plan(P, sys_, 1 if periodic else 0, rep)
    t2 = time.time()
    out["evaluate"] = rel(u, ur)
    scale = np.max(np.abs(ur))
    err = np.abs(u - ur)
    out["percomp_ok"] = bool(np.all(err <= 1e-10 * np.maximum(np.abs(ur), 1e-3 * scale)))
    out["t_ref"] = t1 - t0
    out["t_gpu"] = t2 - t1
    out["gpu_total"] = rep.get("t_total")
    return out


if __name__ == "__main__":
    cases = [
        dict(kernel=0, dim=3, n=10000, eps=1e-6),
        dict(kernel=1, dim=3, n=6000, eps=1e-6),
        dict(kernel=2, dim=3, n=6000, eps=1e-6),
        dict(kernel=0, dim=2, n=8000, eps=1e-9),
        dict(kernel=1, dim=2, n=5000, eps=1e-6),
        dict(kernel=2, dim=2, n=5000, eps=1e-6),
        dict(kernel=0, dim=3, n=8000, eps=1e-8, periodic=True),
        dict(kernel=1, dim=3, n=4000, eps=1e-6, periodic=True),
        dict(kernel=0, dim=3, n=5000, eps=1e-6, ntgt=3000),
        dict(kernel=0, dim=3, n=3000, eps=1e-3),
    ]
    for c in cases:
        try:
            print(case(**c), flush=True)
        except Exception as e:  # noqa: BLE001
            print("FAILED", c, type(e).__name__, e, flush=True)
