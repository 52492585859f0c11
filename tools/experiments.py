"""Accuracy and scaling experiments on the GPU path, writing the reference
CLI's CSV layout (tools/cli_main.cpp:146-177: '#' header lines, then
kernel,dim,mode,window,eps,N,pass,seconds,rel_l2,c,p,N1,N_per,n_s with one
row per pass), so the reference's plotting / regression scripts read both.

  accuracy: DMK vs the exact sum (cli_main.cpp:217-238).  The exact sum is
            the GPU direct_sum (bitwise the reference's in 3D), so N is not
            capped at 5e4 as in the reference.
  scaling:  per-pass times over an ascending N list (cli_main.cpp:240-262).

Points are seeded uniform samples of the unit box (numpy), not the
reference's pointgen stream.  Free space only (the periodic accuracy
reference, ewald_reference, is an O(N^2) CPU routine).

usage: python tools/experiments.py accuracy --kernel stokeslet --dim 3 --eps 1e-6 --n 100000 [--out f.csv]
       python tools/experiments.py scaling --kernel stokeslet --dim 3 --eps 1e-6 --n-list 1e5,1e6,1e7
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402

PASSES = [("tree", "t_tree"), ("upward", "t_upward"), ("root", "t_root"), ("downward", "t_downward"),
          ("residual", "t_residual")]


def make_system(kernel, dim, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5, 0.5, (n, dim))
    s = rng.standard_normal((n, g.strength_components(kernel, dim)))
    if kernel == g.STRESSLET:
        nn = rng.standard_normal((n, dim))
        s[:, dim:] = nn / np.linalg.norm(nn, axis=1, keepdims=True)
    return g.ParticleSystem(dim, x, np.zeros(0), s)


def rel_l2(got, want):  # cli_main.cpp:92-101
    num, den = float(np.sum((got - want) ** 2)), float(np.sum(want ** 2))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return (num / den) ** 0.5


class Csv:
    def __init__(self, path):
        self.f = open(path, "w", newline="\n") if path else sys.stdout

    def header(self, a, plan, n):
        w = self.f.write
        w("# tool=sdmk-b200-experiments\n")
        w(f"# kernel={a.kernel} dim={a.dim} mode=free window={a.window} eps={a.eps!r}\n")
        w(f"# n={n} targets=0 gen=uniform seed={a.seed} repetitions={a.repetitions}\n")
        w(f"# plan: c={plan.c!r} sigma={plan.sigma!r} p={plan.p} N1={plan.N1} N_per={plan.N_per} "
          f"n_s={plan.n_s} table_tol={plan.table_tol!r}\n")
        w("kernel,dim,mode,window,eps,N,pass,seconds,rel_l2,c,p,N1,N_per,n_s\n")

    def row(self, a, plan, n, name, sec, rel):
        r = "" if rel is None else repr(float(rel))
        self.f.write(f"{a.kernel},{a.dim},free,{a.window},{a.eps!r},{n},{name},{sec!r},{r},{plan.c!r},{plan.p},"
                     f"{plan.N1},{plan.N_per},{plan.n_s}\n")
        self.f.flush()


def timed(ctx, plan, sysm, reps):  # best per pass over the repetitions (cli_main.cpp:186-204)
    best, u = None, None
    for _ in range(max(1, reps)):
        rep = {}
        u = ctx.evaluate_with_plan(plan, sysm, g.FREE_SPACE, rep)
        if best is None:
            best = rep
        else:
            for _, k in PASSES:
                best[k] = min(best[k], rep[k])
    return u, best


def emit(csv, a, plan, n, rep, rel):
    for name, key in PASSES:
        csv.row(a, plan, n, name, rep[key], rel)
    csv.row(a, plan, n, "total", sum(rep[k] for _, k in PASSES), rel)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["accuracy", "scaling"])
    ap.add_argument("--kernel", default="stokeslet", choices=list(g.KERNELS))
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--window", default="prolate", choices=["prolate", "gaussian"])
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--n-list", default="")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--repetitions", type=int, default=1)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    kernel = g.KERNELS[a.kernel]
    plan = g.select_parameters(kernel, a.eps, g.PROLATE if a.window == "prolate" else g.GAUSSIAN, a.dim)
    ctx = g.Context(0)
    csv = Csv(a.out)
    if a.mode == "accuracy":
        sysm = make_system(kernel, a.dim, a.n, a.seed)
        ref = ctx.direct_sum(kernel, sysm)
        u, rep = timed(ctx, plan, sysm, a.repetitions)
        rel = rel_l2(u, ref)
        csv.header(a, plan, a.n)
        emit(csv, a, plan, a.n, rep, rel)
        print(f"accuracy: rel_l2={rel:.3e} target={a.eps:g}  [{'pass' if rel <= a.eps else 'FAIL'}]", file=sys.stderr)
        return 0 if rel <= a.eps else 1
    ns = [int(float(v)) for v in a.n_list.split(",") if v]
    if not ns or ns != sorted(ns):
        raise SystemExit("scaling mode needs a nonempty ascending N list")
    csv.header(a, plan, ns[0])
    totals = []
    for n in ns:
        _, rep = timed(ctx, plan, make_system(kernel, a.dim, n, a.seed), a.repetitions)
        emit(csv, a, plan, n, rep, None)
        totals.append(sum(rep[k] for _, k in PASSES))
    for i in range(1, len(ns)):
        print(f"scaling: N {ns[i - 1]} -> {ns[i]}  time ratio = {totals[i] / totals[i - 1]:.4g}", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
