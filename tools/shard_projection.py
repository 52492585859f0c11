"""Projected strong scaling of the sharded evaluation, measured on ONE GPU.

gpurun gives one B200, so the ranks of an R-GPU run are executed one after
another on it in the library's manual-exchange mode (include/sdmk.h
sdmk_set_manual_exchange): each rank's evaluate_begin + evaluate_end is the
exact device work that rank does in an R-GPU run (tree, its cut subtrees,
halo pack/unpack, the boxes above the cut, its shard of the downward /
far-field / residual passes), timed with CUDA events on the library stream.
The NCCL transfers are NOT run; their bytes are reported and costed at an
assumed NVLink rate (--link-gbs) together with the all-gather of u (each
rank receives the other ranks' owned ranges, (R-1)/R of u).  The
projection is max over ranks of (device time + transfer estimate), and
"overlap" credits the library's schedule, where the halo exchange runs on a
side stream beside the residual pass; it is a model, not a multi-GPU
measurement.

usage: python tools/shard_projection.py [--n 1e7] [--dist uniform|cfg5] [--ranks 2,4,8]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21471_b200 as g  # noqa: E402


def system(n, dist, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5, 0.5, (n, 3))
    if dist == "cfg5":  # half uniform, half in 8 Gaussian clusters (sigma 5e-3), BASELINE cfg5
        h = n // 2
        c = rng.uniform(-0.4, 0.4, (8, 3))
        k = rng.integers(0, 8, h)
        x[:h] = np.clip(c[k] + 5e-3 * rng.standard_normal((h, 3)), -0.5, 0.5)
    return x, rng.standard_normal((n, 3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e7)
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--link-gbs", type=float, default=400.0, help="assumed per-GPU NVLink rate for the estimate")
    a = ap.parse_args()
    import torch
    n = int(a.n)
    x, f = system(n, a.dist, 0)
    dx, df = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    du = torch.empty(n * 3, dtype=torch.float64, device="cuda")
    plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    ctx = g.Context(0)
    rep = {}
    for _ in range(a.reps + 1):
        ctx.evaluate_device(plan, 3, n, dx.data_ptr(), 0, 0, df.data_ptr(), 0, du.data_ptr(), rep)
    t1 = rep["t_total"]
    out = {"n": n, "dist": a.dist, "t1_ms": t1 * 1e3, "link_gbs_assumed": a.link_gbs, "ranks": {}}
    print(json.dumps({"R": 1, "t_ms": t1 * 1e3, "tree_ms": rep["t_tree"] * 1e3}), flush=True)
    ctx.set_manual_exchange(True)
    for R in [int(v) for v in a.ranks.split(",")]:
        rows = []
        for r in range(R):
            ctx.set_shard(r, R)
            rr = None
            for k in range(a.reps):  # the fastest repetition: the host part (repair, lists) is noisy on a shared box
                r1 = {}
                ctx.evaluate_begin_device(plan, 3, n, dx.data_ptr(), 0, 0, df.data_ptr(), 0)
                ctx.evaluate_end(r1, d_u=du.data_ptr())
                if k > 0 and (rr is None or r1["t_total"] < rr["t_total"]):
                    rr = r1
            u_bytes = n * 3 * 8
            halo_s = rr["halo_bytes_recv"] / (a.link_gbs * 1e9)
            u_s = u_bytes * (R - 1) / R / (a.link_gbs * 1e9)  # all-gather of the owned ranges
            xfer = halo_s + u_s
            # with a communicator the halo exchange runs beside the residual pass
            # (engine.cpp evaluate: side stream, residual first); u's all-gather cannot
            hidden = max(0.0, halo_s - rr["t_residual"]) + u_s
            rows.append({"rank": r, "dev_ms": rr["t_total"] * 1e3, "tree_ms": rr["t_tree"] * 1e3,
                         "upward_ms": rr["t_upward"] * 1e3, "root_ms": rr["t_root"] * 1e3, "pack_unpack_ms": rr["t_exchange"] * 1e3,
                         "downward_ms": rr["t_downward"] * 1e3, "residual_ms": rr["t_residual"] * 1e3,
                         "halo_recv_MB": rr["halo_bytes_recv"] / 1e6, "xfer_est_ms": xfer * 1e3,
                         "xfer_exposed_ms": hidden * 1e3})
        # (no transfer between the sequential ranks: the received slabs hold stale
        # data, which changes values but not the work; correctness of the same
        # code path is tests/test_gpu_parity.py::test_halo_exchange_sums_to_single)
        worst = max(rows, key=lambda q: q["dev_ms"] + q["xfer_est_ms"])
        tR = worst["dev_ms"] + worst["xfer_est_ms"]
        tO = max(q["dev_ms"] + q["xfer_exposed_ms"] for q in rows)
        res = {"R": R, "projected_ms": tR, "projected_eff": t1 * 1e3 / (R * tR),
               "projected_overlap_ms": tO, "projected_overlap_eff": t1 * 1e3 / (R * tO),
               "max_dev_ms": max(q["dev_ms"] for q in rows), "min_dev_ms": min(q["dev_ms"] for q in rows),
               "per_rank": rows}
        out["ranks"][R] = res
        print(json.dumps({k: v for k, v in res.items() if k != "per_rank"}), flush=True)
    ctx.set_manual_exchange(False)
    ctx.set_shard(0, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
