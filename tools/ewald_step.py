"""One warm FFT-Ewald evaluation at BASELINE cfg2 (for ncu launch lists / captures)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2509_21471_b200 as g  # noqa: E402
from baseline_configs import cfg_system  # noqa: E402

c = cfg_system("cfg2")
ctx = g.Context(0)
plan = g.select_parameters(0, 1e-8, g.PROLATE, 3)
s = g.ParticleSystem(3, c["x"], np.zeros(0), c["s"])
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    info = {}
    ctx.ewald(plan, s, info=info)
    print(info, flush=True)
