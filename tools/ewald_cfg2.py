"""BASELINE cfg2 (3D periodic Stokeslet, N = 1e6 iid uniform, forces N(0,1)
shifted to zero net force, eps = 1e-8) through the FFT Ewald path
(include/sdmk.h sdmk_ewald) beside the GPU periodic DMK, at full size.

Per split level: the Ewald parameters (cells, grid, window width,
kappa_max), device times per phase, the e2e time, and the difference to the
DMK result (both approximate the periodic sum to eps; the Ewald at a 100x
tighter tolerance shows which side the difference is on).

usage: python tools/ewald_cfg2.py [--levels 3,4,5]   -> JSON lines
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2509_21471_b200 as g  # noqa: E402
from baseline_configs import cfg_system  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="-1,3,4,5")
    a = ap.parse_args()
    c = cfg_system("cfg2")
    x, f = c["x"], c["s"]
    n = len(x)
    ctx = g.Context(0)
    plan = g.select_parameters(0, 1e-8, g.PROLATE, 3)
    s = g.ParticleSystem(3, x, np.zeros(0), f)
    rep = {}
    ctx.evaluate_with_plan(plan, s, g.PERIODIC)
    u_dmk = ctx.evaluate_with_plan(plan, s, g.PERIODIC, rep)
    tight = g.select_parameters(0, 1e-10, g.PROLATE, 3)
    u_tight = ctx.ewald(tight, s)
    print(json.dumps({"config": "cfg2", "n": n, "method": "dmk_periodic", "eps": 1e-8,
                      "t_total_ms": rep["t_total"] * 1e3, "points_per_s": n / rep["t_total"],
                      "rel_vs_ewald_eps1e-10": rel(u_dmk, u_tight)}), flush=True)
    for L in [int(v) for v in a.levels.split(",")]:
        info = {}
        ctx.ewald(plan, s, level=L, info=info)  # warm (plans, buffers)
        t0 = time.perf_counter()
        u = ctx.ewald(plan, s, level=L, info=info)
        wall = time.perf_counter() - t0
        print(json.dumps({"config": "cfg2", "n": n, "method": "fft_ewald", "eps": 1e-8, **info,
                          "wall_ms": wall * 1e3, "points_per_s": n / (info["t_total_ms"] * 1e-3),
                          "rel_vs_dmk": rel(u, u_dmk), "rel_vs_ewald_eps1e-10": rel(u, u_tight)}), flush=True)


if __name__ == "__main__":
    main()
