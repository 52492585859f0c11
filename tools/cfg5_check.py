"""cfg5 shape (N=1.6e7: half uniform, half in 8 Gaussian clusters, sigma 5e-3), 3D Stokeslet eps=1e-6:
one warm evaluation, report + device memory high-water mark."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 16_000_000
rng = np.random.default_rng(5)
x = rng.uniform(-0.5, 0.5, (n, 3))
h = n // 2
c = rng.uniform(-0.4, 0.4, (8, 3))
k = rng.integers(0, 8, h)
x[:h] = np.clip(c[k] + 5e-3 * rng.standard_normal((h, 3)), -0.5, 0.5)
f = rng.standard_normal((n, 3))
ctx = g.Context(0)
plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
for _ in range(2):
    rep = {}
    u = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, np.zeros(0), f), 0, rep)
    print({k_: (round(v, 4) if isinstance(v, float) else v) for k_, v in rep.items()}, flush=True)
import torch  # noqa: E402
free, total = torch.cuda.mem_get_info()
print(f"device memory in use after: {(total - free) / 2**30:.1f} GiB of {total / 2**30:.1f}")
