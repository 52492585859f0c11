"""Every BASELINE.json configuration at its full size on one GPU.

For each config: seeded synthetic inputs of the stated shape (no public
dataset exists; the generators follow BASELINE.json's descriptions), two
warm evaluations through the host entry point (sdmk_evaluate_with_plan:
H2D, all passes, D2H), and two size-independent checks:
  * linearity: doubling the forces doubles u bit for bit (a power-of-two
    scale commutes with every rounding in the pipeline; the stresslet's
    normals stay fixed, it is bilinear in f and n);
  * accuracy (free space): 256 sampled targets against the exact sum on the
    GPU (sdmk_direct_sum, the reference's direct_sum), split as all sources
    outside the sample plus the sample's own pairs so no self pair appears.
    Periodic cfg2 has no O(N) exact reference (ewald_reference is O(N^2) on
    the CPU), so it reports linearity only.

usage: python tools/baseline_configs.py [cfg1,cfg2,...]  -> one JSON line per config
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402


def cfg_system(name):
    rng = np.random.default_rng({"cfg1": 0, "cfg2": 2, "cfg3": 3, "cfg4": 4, "cfg5": 5}[name])
    if name == "cfg1":
        x = rng.uniform(-0.5, 0.5, (10_000, 3))
        return dict(kernel=0, dim=3, eps=1e-6, periodic=0, x=x, s=rng.standard_normal((10_000, 3)))
    if name == "cfg2":
        n = 1_000_000
        x = rng.uniform(-0.5, 0.5, (n, 3))
        f = rng.standard_normal((n, 3))
        f -= f.mean(axis=0)  # zero net force
        return dict(kernel=0, dim=3, eps=1e-8, periodic=1, x=x, s=f)
    if name == "cfg3":
        n = 2_000_000
        c = rng.uniform(-0.4, 0.4, (64, 3))
        r = rng.uniform(0.01, 0.05, 64)
        k = rng.integers(0, 64, n)
        v = rng.standard_normal((n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        x = np.clip(c[k] + r[k, None] * v, -0.5, 0.5)
        s = np.concatenate([rng.standard_normal((n, 3)), v], axis=1)  # f, then the outward normal
        return dict(kernel=1, dim=3, eps=1e-6, periodic=0, x=x, s=s)
    if name == "cfg4":
        n = 4_000_000
        c = rng.uniform(-0.45, 0.45, (16, 2))
        sg = rng.uniform(1e-3, 1e-2, 16)
        k = rng.integers(0, 16, n)
        x = np.clip(c[k] + sg[k, None] * rng.standard_normal((n, 2)), -0.5, 0.5)
        return dict(kernel=0, dim=2, eps=1e-9, periodic=0, x=x, s=rng.standard_normal((n, 2)))
    if name == "cfg5":
        n = 16_000_000
        x = rng.uniform(-0.5, 0.5, (n, 3))
        h = n // 2
        c = rng.uniform(-0.4, 0.4, (8, 3))
        k = rng.integers(0, 8, h)
        x[:h] = np.clip(c[k] + 5e-3 * rng.standard_normal((h, 3)), -0.5, 0.5)
        return dict(kernel=0, dim=3, eps=1e-6, periodic=0, x=x, s=rng.standard_normal((n, 3)))
    raise ValueError(name)


def exact_at(ctx, kernel, dim, x, s, idx):
    """Exact u at sources idx (self pair excluded) from two GPU direct sums."""
    mask = np.ones(len(x), bool)
    mask[idx] = False
    far = ctx.direct_sum(kernel, g.ParticleSystem(dim, x[mask], x[idx], s[mask]))
    own = ctx.direct_sum(kernel, g.ParticleSystem(dim, x[idx], np.zeros(0), s[idx]))
    return (far + own).reshape(-1, dim)


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    ctx = g.Context(0)
    for name in names:
        c = cfg_system(name)
        kernel, dim, n = c["kernel"], c["dim"], len(c["x"])
        plan = g.select_parameters(kernel, c["eps"], g.PROLATE, dim)
        sysm = g.ParticleSystem(dim, c["x"], np.zeros(0), c["s"])
        rep = {}
        for _ in range(2):
            t0 = time.perf_counter()
            u = ctx.evaluate_with_plan(plan, sysm, c["periodic"], rep)
            wall = time.perf_counter() - t0
        s2 = c["s"].copy()
        s2[:, :dim] *= 2.0  # the force part: u is linear in f (the stresslet is bilinear in f and n)
        u2 = ctx.evaluate_with_plan(plan, g.ParticleSystem(dim, c["x"], np.zeros(0), s2), c["periodic"])
        line = {"config": name, "kernel": ["stokeslet", "stresslet", "rotlet"][kernel], "dim": dim, "n": n,
                "eps": c["eps"], "periodic": bool(c["periodic"]), "p": plan.p, "N1": plan.N1, "n_s": plan.n_s,
                "boxes": rep["num_boxes"], "max_level": rep["max_level"],
                "t_total_ms": rep["t_total"] * 1e3, "points_per_s": n / rep["t_total"], "wall_ms": wall * 1e3,
                "passes_ms": {k: round(rep[k] * 1e3, 2) for k in ("t_h2d", "t_tree", "t_upward", "t_root",
                                                                 "t_downward", "t_residual", "t_d2h")},
                "linearity_bitwise": bool(np.array_equal(u2, 2.0 * u))}
        if not c["periodic"]:
            idx = np.random.default_rng(99).choice(n, 256, replace=False)
            ex = exact_at(ctx, kernel, dim, c["x"], c["s"], idx)
            got = u.reshape(-1, dim)[idx]
            line["rel_l2_vs_exact_256"] = float(np.linalg.norm(got - ex) / np.linalg.norm(ex))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
