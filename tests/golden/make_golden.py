"""Generate the golden vectors in tests/golden/ from the compiled reference.

Run in the container that has /root/reference (oracle/_ref is built from it):
    python tests/golden/make_golden.py
Each case stores its seeded inputs, the plan, the reference's SDMKSPLT table
file, the reference's dump_tree text, its src permutation and the reference
evaluate_with_plan output (plus residual_pass and target_far_fields), so the
CPU suite can pin both the oracle restatement and the product's host code
without the reference sources, and the GPU suite can check the CUDA path.
"""
import json
import zlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref  # noqa: E402

CASES = [
    # name, kernel, dim, n, eps, periodic, ntgt, n_s override, window, distribution
    ("stokeslet3d_uniform", 0, 3, 3000, 1e-6, False, 0, 200, 0, "uniform"),
    ("stokeslet3d_cluster", 0, 3, 2500, 1e-6, False, 0, 60, 0, "cluster"),
    ("stresslet3d_uniform", 1, 3, 2000, 1e-6, False, 0, 300, 0, "uniform"),
    ("rotlet3d_eps3", 2, 3, 2000, 1e-3, False, 0, 100, 0, "uniform"),
    ("stokeslet2d_eps9", 0, 2, 3000, 1e-9, False, 0, 100, 0, "cluster"),
    ("stresslet2d", 1, 2, 2000, 1e-6, False, 0, 100, 0, "uniform"),
    ("rotlet2d", 2, 2, 2000, 1e-6, False, 0, 100, 0, "uniform"),
    ("stokeslet3d_periodic_eps8", 0, 3, 2000, 1e-8, True, 0, 300, 0, "uniform"),
    ("stresslet3d_periodic", 1, 3, 1500, 1e-6, True, 0, 300, 0, "uniform"),
    ("stokeslet3d_targets", 0, 3, 2000, 1e-6, False, 700, 250, 0, "uniform"),
    ("stokeslet3d_gaussian", 0, 3, 1000, 1e-6, False, 0, 150, 1, "uniform"),
    ("stokeslet2d_periodic", 0, 2, 2000, 1e-6, True, 0, 100, 0, "uniform"),
]


def points(rng, n, dim, dist, periodic):
    if dist == "uniform":
        x = rng.uniform(-0.5, 0.5, (n, dim))
    else:  # clusters: adaptive deep trees
        c = rng.uniform(-0.4, 0.4, (4, dim))
        x = c[rng.integers(0, 4, n)] + rng.normal(0, 0.02, (n, dim))
        x = np.clip(x, -0.5, 0.5)
    if periodic:
        x = x + rng.integers(-1, 2, (n, dim))  # exercise the wrap
    return x


def main():
    index = []
    for name, kernel, dim, n, eps, periodic, ntgt, n_s, window, dist in CASES:
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        x = points(rng, n, dim, dist, periodic)
        sc = {0: dim, 1: 2 * dim, 2: 3 if dim == 3 else 1}[kernel]
        s = rng.standard_normal((n, sc))
        if kernel == 1:
            nn = rng.standard_normal((n, dim))
            s[:, dim:] = nn / np.linalg.norm(nn, axis=1, keepdims=True)
        t = rng.uniform(-0.5, 0.5, (ntgt, dim)) if ntgt else np.zeros((0, dim))
        plan = ref.select_parameters(kernel, eps, window, dim)
        plan["n_s"] = n_s
        P = ref.RefProblem(plan, dim, x, s, t if ntgt else None, periodic)
        u, _ = P.evaluate()
        tab = os.path.join(HERE, f"{name}.tables.bin")
        P.export_tables(tab)
        sp, tp = P.tree_perm()
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), sources=x, strengths=s, targets=t, u=u,
                            residual=P.residual(), far=P.target_far(), sperm=sp,
                            tperm=tp if tp is not None else np.zeros(0, np.int32))
        with open(os.path.join(HERE, f"{name}.tree.txt"), "w") as f:
            f.write(P.tree_dump())
        index.append(dict(name=name, kernel=kernel, dim=dim, n=n, eps=eps, periodic=periodic, ntgt=ntgt,
                          window=window, plan=plan, num_boxes=P.info["num_boxes"], max_level=P.info["max_level"]))
        print(name, P.info, flush=True)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
