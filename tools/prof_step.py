"""One warm DMK evaluation for profiling (ncu launch lists / --set full)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--eps", type=float, default=1e-6)
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--periodic", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cfg", default=None, help="a BASELINE configuration (tools/baseline_configs.py) instead")
a = ap.parse_args()
if a.cfg:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from baseline_configs import cfg_system
    c = cfg_system(a.cfg)
    x, s = c["x"], c["s"]
    a.kernel, a.dim, a.eps, a.periodic = c["kernel"], c["dim"], c["eps"], c["periodic"]
else:
    rng = np.random.default_rng(0)
    x = rng.uniform(-0.5, 0.5, (a.n, a.dim))
    sc = g.strength_components(a.kernel, a.dim)
    s = rng.standard_normal((a.n, sc))
ctx = g.Context(0)
plan = g.select_parameters(a.kernel, a.eps, g.PROLATE, a.dim)
sys_ = g.ParticleSystem(a.dim, x, np.zeros(0), s)
for i in range(a.reps):
    rep = {}
    ctx.evaluate_with_plan(plan, sys_, a.periodic, rep)
    print({k: (round(v, 5) if isinstance(v, float) else v) for k, v in rep.items()}, flush=True)
