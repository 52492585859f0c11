"""Small evaluations for compute-sanitizer (racecheck / memcheck / synccheck).

Covers every kernel family of the evaluation at sizes the sanitizer finishes
in minutes: the 3D DMMA path (k_basis, k_anterp2, k_tensor_up/down, k_fwd_xy2,
k_zf2, k_acc_group with its TMA/mbarrier ring, k_zi2, k_inv_xy2,
k_interp_mma), the persistent residual kernel with its atomic work queue,
the FFMA paths (2D, and the periodic top levels on k_acc_sym), the tree
kernels and the GPU direct sums.

usage: compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402


def main():
    ctx = g.Context(0)
    rng = np.random.default_rng(7)
    cases = [
        ("stokeslet3d", 0, 3, 1e-6, 0, 40_000),
        ("stresslet3d_periodic", 1, 3, 1e-6, 1, 20_000),
        ("rotlet3d", 2, 3, 1e-3, 0, 20_000),
        ("stokeslet2d", 0, 2, 1e-9, 0, 30_000),
    ]
    for name, kernel, dim, eps, per, n in cases:
        x = rng.uniform(-0.5, 0.5, (n, dim))
        s = rng.standard_normal((n, g.strength_components(kernel, dim)))
        plan = g.select_parameters(kernel, eps, g.PROLATE, dim)
        rep = {}
        u = ctx.evaluate_with_plan(plan, g.ParticleSystem(dim, x, np.zeros(0), s), per, rep)
        assert np.all(np.isfinite(u)), name
        print(f"{name}: {rep['num_boxes']} boxes, {rep['kernel_launches']} launches", flush=True)
    xs = rng.uniform(-0.5, 0.5, (2000, 3))
    d = ctx.direct_sum(0, g.ParticleSystem(3, xs, np.zeros(0), rng.standard_normal((2000, 3))))
    assert np.all(np.isfinite(d))
    print("direct_sum ok", flush=True)


if __name__ == "__main__":
    main()
