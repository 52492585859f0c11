"""Parity with the compiled reference at every BASELINE configuration, full size.

For each configuration the SAME seeded inputs go through
  * the reference (oracle/_ref: the unmodified stokesdmk core, all host
    threads): build_tree, then the passes of evaluate_with_plan once
    (dmk.cpp:1070-1084, shim ref_run_full) with u assembled as
    dmk.cpp:1086-1102 does, and a counting pass of the residual pair loop
    over the reference's own tree (dmk.cpp:941-1013, shim ref_count_pairs);
  * the GPU library through its C-ABI: the pass-level entry points
    (sdmk_setup, sdmk_upward_pass, sdmk_incoming(1), sdmk_target_far_fields,
    sdmk_residual_pass) on the same problem, then sdmk_evaluate_with_plan
    twice (u, determinism, the in-support pair count from its report).

Recorded per configuration (one JSON line):
  * sha256 of the dump_tree text on both sides (tree.cpp:325-354) and
    whether they are equal; whether src_perm (and tgt_perm) are equal;
  * max scaled error, |a - b| / max(|b|, 1e-3 ||b||_inf) over every
    component, for the outgoing proxies (upward), the incoming
    proxies after the downward pass, the target far field, the residual and
    u; the bar is 1e-10;
  * in-support pair counts: the reference's loop vs the GPU kernel's count;
  * bitwise determinism of two GPU evaluations;
  * reference pass times on this host (cores stated) and GPU e2e time.
cfg1 adds the exact O(N^2) sum (reference direct_sum) as a second oracle.

usage: python tools/parity_configs.py cfg1,cfg2,... [--out file.jsonl]
Needs oracle/_ref (built here by oracle/Makefile; it travels to the GPU box).
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2509_21471_b200 as g  # noqa: E402
from oracle import ref  # noqa: E402
from baseline_configs import cfg_system  # noqa: E402

TOL = 1e-10


def system(name):
    if name.startswith("metric_"):
        import bench
        kernel = {"metric_stokeslet": 0, "metric_stresslet": 1}[name]
        x, s = bench.make_system(kernel, 10_000_000, 0 + kernel)  # bench.py's inputs, seeds 0 / 1
        return dict(kernel=kernel, dim=3, eps=1e-6, periodic=0, x=x, s=s)
    return cfg_system(name)


def scaled_err(a, b, chunk=1 << 25):
    """max |a-b| / max(|b|, 1e-3 ||b||_inf), in chunks (arrays up to ~20 GB)."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    if a.shape != b.shape:
        return float("inf")
    if b.size == 0:
        return 0.0
    inf = 0.0
    for i in range(0, b.size, chunk):
        inf = max(inf, float(np.max(np.abs(b[i:i + chunk]))))
    floor = 1e-3 * inf
    err = 0.0
    for i in range(0, b.size, chunk):
        bb = b[i:i + chunk]
        d = np.abs(a[i:i + chunk] - bb) / np.maximum(np.abs(bb), floor if floor > 0 else 1e-300)
        err = max(err, float(np.max(d)))
    return err


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def run(name, ctx, threads):
    c = system(name)
    kernel, dim, n = c["kernel"], c["dim"], len(c["x"])
    x, s, mode = c["x"], c["s"], c["periodic"]
    plan = g.select_parameters(kernel, c["eps"], g.PROLATE, dim)
    line = {"config": name, "kernel": ["stokeslet", "stresslet", "rotlet"][kernel], "dim": dim, "n": n,
            "eps": c["eps"], "periodic": bool(mode), "p": plan.p, "N1": plan.N1, "N_per": plan.N_per,
            "n_s": plan.n_s, "tol": TOL}
    log = lambda m: print(f"[parity {name}] {m}", file=sys.stderr, flush=True)  # noqa: E731

    # ---- reference: tree, counting pass, the passes once ----
    t0 = time.perf_counter()
    R = ref.RefProblem(plan.__dict__, dim, x, s, periodic=bool(mode))
    line["ref_setup_s"] = time.perf_counter() - t0
    ref_dump = R.tree_dump()
    ref_sp, ref_tp = R.tree_perm()
    line["boxes"], line["max_level"] = R.info["num_boxes"], R.info["max_level"]
    t0 = time.perf_counter()
    tested, insup, zero = R.count_pairs()
    line["ref_pairs"] = {"tested": tested, "in_support": insup, "coincident": zero,
                         "count_s": time.perf_counter() - t0}
    log(f"reference tree {R.info['num_boxes']} boxes; pairs in support {insup}")
    t_tree = R.time_tree()
    far_r, res_r, u_r, rp = R.run_full()
    tot = t_tree + rp["t_upward"] + rp["t_root"] + rp["t_downward"] + rp["t_residual"]
    line["ref_time"] = {"cores": threads, "t_tree": t_tree, **{k: rp[k] for k in ("t_upward", "t_root", "t_downward",
                                                                                    "t_residual")},
                        "t_total": tot, "points_per_s": n / tot}
    log(f"reference passes {tot:.1f} s ({n / tot:.3g} points/s on {threads} threads)")

    # ---- GPU: the same problem through the pass-level C-ABI ----
    sysm = g.ParticleSystem(dim, x, np.zeros(0), s)
    ctx.setup(plan, sysm, mode)
    gpu_dump = ctx.tree_dump()
    sp, tp = ctx.tree_perm()
    line["tree_sha256"] = {"ref": sha(ref_dump), "gpu": sha(gpu_dump)}
    line["tree_equal"] = gpu_dump == ref_dump
    line["perm_equal"] = bool(np.array_equal(sp, ref_sp)) and (ref_tp is None or np.array_equal(tp, ref_tp))
    del gpu_dump, ref_dump
    errs = {}
    og = ctx.upward_pass()
    errs["upward"] = scaled_err(og, R.proxy(0))
    del og
    inc = ctx.incoming(1)
    errs["incoming"] = scaled_err(inc, R.proxy(1))
    del inc
    R.release()
    errs["far"] = scaled_err(ctx.target_far_fields(), far_r)
    errs["residual"] = scaled_err(ctx.residual_pass(), res_r)
    rep = {}
    ctx.evaluate_with_plan(plan, sysm, mode)  # warm
    t0 = time.perf_counter()
    u = ctx.evaluate_with_plan(plan, sysm, mode, rep)
    wall = time.perf_counter() - t0
    u2 = ctx.evaluate_with_plan(plan, sysm, mode)
    errs["u"] = scaled_err(u, u_r)
    line["max_scaled_err"] = errs
    line["gpu_pairs_in_support"] = int(rep["p2p_in_support"])
    line["pairs_equal"] = int(rep["p2p_in_support"]) == insup
    line["deterministic"] = bool(np.array_equal(u, u2))
    line["gpu_e2e_s"] = rep["t_total"]
    line["gpu_wall_s"] = wall
    line["gpu_points_per_s"] = n / rep["t_total"]
    if name == "cfg1":  # second oracle: the exact O(N^2) sum (acceptance.cpp:451-474)
        ex = R.direct_sum()
        line["rel_l2_vs_direct"] = {"gpu": float(np.linalg.norm(u - ex) / np.linalg.norm(ex)),
                                    "ref": float(np.linalg.norm(u_r - ex) / np.linalg.norm(ex))}
    line["pass"] = bool(line["tree_equal"] and line["perm_equal"] and line["pairs_equal"] and line["deterministic"]
                        and all(v <= TOL for v in errs.values()))
    log(f"errors {errs}; tree {line['tree_equal']} perm {line['perm_equal']} pairs {line['pairs_equal']}")
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="?", default="cfg1,cfg2,cfg3,cfg4,metric_stokeslet,metric_stresslet,cfg5")
    ap.add_argument("--out", default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    threads = ref.set_threads(a.threads)
    ctx = g.Context(0)
    for name in a.configs.split(","):
        line = run(name, ctx, threads)
        print(json.dumps(line), flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
