#!/usr/bin/env python
"""Benchmark: DMK evaluate throughput (points/s) at the BASELINE metric.

Workload (BASELINE.json "metric"): N = 1e7 sources = targets, iid uniform in
[-1/2, 1/2]^3, free space, eps = 1e-6, prolate window; Stokeslet forces
f ~ N(0,1)^3 (headline `value`) and the stresslet (f ~ N(0,1)^3, n a random
unit vector) reported beside it.  Seeded synthetic data (no dataset exists).

  value  : N / (device time of one evaluate_with_plan) with inputs already in
           HBM (sdmk_evaluate_device), CUDA events on the library's stream.
  e2e    : same metric through the C-ABI sdmk_evaluate_with_plan from pinned
           HOST buffers (H2D of points+strengths and D2H of u inside).
  roofline: dominant kernel of the step (FP64-bound), achieved algorithmic
           FLOP/s over its CUDA-event time vs the measured DFMA peak.
  cpu_baseline: the reference (oracle/_ref, unmodified stokesdmk core, all
           host threads) on a bounded sample of the same workload.

--impl reference times the reference's own CPU implementation (oracle/_ref)
on a bounded sample per step (rank 0 only).

Multi-GPU (torchrun): the SAME N-point system is sharded (include/sdmk.h
sdmk_comm_init, paper_2509_21471_b200/distributed.py): every rank builds the
tree; the upward pass is split into cut subtrees owned by ranks, with one
NCCL group exchanging the outgoing expansions each rank reads (its halo) and
the cut boxes; each rank forms the downward pass, far fields and residual
for its own Morton run of target leaves, and an NCCL all-reduce assembles u
on every rank (strong scaling; the result is bitwise the 1-GPU result).  All
of it runs on the library's stream; the timed region (CUDA events on that
stream, the call blocking in between) has barriers on both sides and the
max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6551.7
# one metric string for both arms (the driver pairs the lines by it)
METRIC = "points/sec (3D Stokeslet DMK, N=1e7, eps=1e-6)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_system(kernel: int, n: int, seed: int):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5, 0.5, (n, 3))
    f = rng.standard_normal((n, 3))
    if kernel == 1:
        nn = rng.standard_normal((n, 3))
        nn /= np.linalg.norm(nn, axis=1, keepdims=True)
        s = np.concatenate([f, nn], axis=1)
    else:
        s = f
    return x, s


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def planewave_flops(plan, nbox_src, nbox_tgt, entries, nhalf, ncol, pz, nch, d):
    """Algorithmic FLOPs of the half-spectrum band-limited plane-wave stage."""
    p, M = plan.p, (plan.N1 - 1) // 2
    fwd = pz * (p * (M + 1) * p * 4 + ncol * p * 8) + nhalf * pz * 8
    inv = nhalf * pz * 8 + pz * (p * ncol * 8 + p * p * (M + 1) * 4)
    acc = entries * nch * nhalf * 2
    return nbox_src * nch * fwd + nbox_tgt * d * inv + acc


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2509_21471_b200 as g

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = g.Context(local_rank)
    use_comm = False
    if world > 1:  # the library's own NCCL communicator: halo exchange + u all-reduce on its stream
        try:
            obj = [g.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx.comm_init(rank, world, obj[0])
            ok = 1
        except Exception as e:  # keep the scaling run alive on the replicated-upward path
            log(f"[bench] rank {rank}: library NCCL communicator unavailable ({e}); "
                "falling back to sdmk_set_shard + torch all_reduce")
            ok = 0
        flag = torch.tensor([ok], device="cuda", dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        use_comm = bool(flag.item())
        if not use_comm:
            ctx = g.Context(local_rank)
            ctx.set_shard(rank, world)
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    n = args.n
    results = {}
    clocks = None
    for kname, kernel in (("stokeslet", 0), ("stresslet", 1)):
        if kname not in args.kernels:
            continue
        plan = g.select_parameters(kernel, args.eps, g.PROLATE, 3)
        x, s = make_system(kernel, n, args.seed + kernel)  # the same system on every rank
        d_x = torch.from_numpy(x).cuda()
        d_s = torch.from_numpy(s).cuda()
        d_u = torch.empty(n * 3, dtype=torch.float64, device="cuda")
        rep = {}

        def step_dev():  # at N > 1 every rank returns the assembled u (NCCL inside the call)
            ctx.evaluate_device(plan, 3, n, d_x.data_ptr(), 0, 0, d_s.data_ptr(), g.FREE_SPACE, d_u.data_ptr(), rep)
            if world > 1 and not use_comm:
                dist.all_reduce(d_u, op=dist.ReduceOp.SUM)

        tstream = stream if (world == 1 or use_comm) else torch.cuda.current_stream()

        for _ in range(args.warmup):
            step_dev()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local_rank)
        with sampler:
            e0.record(tstream)
            reps = []
            for _ in range(args.steps):
                step_dev()
                reps.append(dict(rep))
            e1.record(tstream)
            e1.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
        ms = max_over_ranks(ms)
        if kernel == 0:
            clocks = sampler.summary()
        # e2e: pinned host buffers through the public C-ABI (H2D + D2H inside)
        h_x = torch.from_numpy(x).pin_memory()
        h_s = torch.from_numpy(s).pin_memory()
        h_u = torch.empty(n * 3, dtype=torch.float64).pin_memory()
        sys_ = g.ParticleSystem(3, h_x.numpy(), np.zeros(0), h_s.numpy())
        cplan = plan.to_c()
        import ctypes as C
        lib = g.lib()

        def step_host():
            if world > 1 and not use_comm:  # host in, H2D, sharded evaluate, all-reduce, D2H
                d_x.copy_(h_x, non_blocking=True)
                d_s.copy_(h_s, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                step_dev()
                h_u.copy_(d_u)
                return None
            r = g.sdmk_report()
            code = lib.sdmk_evaluate_with_plan(ctx._h, C.byref(cplan), 3, n, g._dptr(sys_.sources), 0, g._dptr(None),
                                               g._dptr(sys_.strengths), 0, g._dptr(h_u.numpy()), C.byref(r))
            g._raise(code)
            return r

        for _ in range(max(1, args.warmup // 2)):
            step_host()
        barrier()
        e0.record(tstream)
        for _ in range(args.steps):
            step_host()
        e1.record(tstream)
        e1.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        # the same through pageable host arrays (what a C++ caller passing
        # std::vector gives the drop-in): staged copies inside the call
        e2e_pg_ms = None
        if world == 1 or use_comm:
            sys_pg = g.ParticleSystem(3, np.ascontiguousarray(x), np.zeros(0), np.ascontiguousarray(s))
            u_pg = np.empty(n * 3)

            def step_pageable():
                r = g.sdmk_report()
                code = lib.sdmk_evaluate_with_plan(ctx._h, C.byref(cplan), 3, n, g._dptr(sys_pg.sources), 0,
                                                   g._dptr(None), g._dptr(sys_pg.strengths), 0, g._dptr(u_pg),
                                                   C.byref(r))
                g._raise(code)

            step_pageable()
            barrier()
            e0.record(tstream)
            for _ in range(args.steps):
                step_pageable()
            e1.record(tstream)
            e1.synchronize()
            barrier()
            e2e_pg_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        # accuracy guard on rank 0: the device result equals the host-path result
        u_dev = d_u.cpu().numpy()
        same = float(np.max(np.abs(u_dev - h_u.numpy())))
        r0 = reps[-1]
        results[kname] = {"ms": ms, "e2e_ms": e2e_ms, "e2e_pageable_ms": e2e_pg_ms, "rep": r0, "plan": plan.__dict__, "dev_vs_host_maxabs": same,
                          "launches": int(r0["kernel_launches"])}
        log(f"[bench] {kname}: {ms:.2f} ms/step device, {e2e_ms:.2f} ms/step e2e; report {r0}")
        del d_x, d_s, d_u
        torch.cuda.empty_cache()

    # rooflines (FP64): the three largest kernels, each over the peak of the
    # pipe it runs on, measured live on this GPU (DFMA for the residual's
    # CUDA-core arithmetic, DMMA for the tensor-core contractions); the bench
    # line's roofline object is the dominant kernel (largest CUDA-event time)
    peak = ctx.fp64_peak_tflops()
    peak_mma = ctx.fp64_mma_peak_tflops()
    R = results.get("stokeslet") or next(iter(results.values()))
    rep = R["rep"]
    plan = g.DmkPlan(**R["plan"])
    hw_all = {}  # per-kernel ncu numbers of the same workload (profiles/round2/kernel_hw.json)
    try:
        with open(os.path.join(ROOT, "profiles", "round2", "kernel_hw.json")) as f:
            hw_all = json.load(f) if args.n == 10_000_000 else {}
    except (OSError, ValueError):
        hw_all = {}
    # residual kernel algorithmic FLOPs (SURVEY 8(d) convention, our tested-candidate count)
    F_in = 3 * (33 + 33) + 30
    res_flops = 8 * rep["p2p_candidates"] + F_in * rep["p2p_in_support"]
    pd = plan.p ** 3
    nch = 3  # Stokeslet channels / components in 3D
    cands = {
        "k_residual": {"t": rep["t_residual_kernel"], "flop": res_flops, "peak": peak, "pipe": "FP64 CUDA cores (DFMA)",
                       "work": "8 FLOP per tested pair + F_in = 3(33+33)+30 = 228 per in-support pair (the reference's "
                               "Clenshaw cost; an algorithm-equivalent rate: the kernel evaluates degree-6 piecewise "
                               "re-expansions, so it executes fewer FP64 operations than this counts)"},
        "k_interp_mma": {"t": rep.get("t_interp_kernel", 0.0), "flop": 2.0 * nch * pd * rep["num_targets"],
                         "peak": peak_mma, "pipe": "FP64 tensor cores (DMMA m8n8k4)",
                         "work": "2 d p^3 FLOP per target (u_j = sum W[j,iz,iy,ix] bz by bx)"},
        "k_anterp2": {"t": rep.get("t_anterp_kernel", 0.0), "flop": 2.0 * nch * pd * rep["num_sources"],
                      "peak": peak_mma, "pipe": "FP64 tensor cores (DMMA m8n8k4)",
                      "work": "2 nch p^3 FLOP per source (outgoing[ch,iz,iy,ix] += s_ch bz by bx)"},
    }
    kern = {}
    for name, c in cands.items():
        if c["t"] <= 0:
            continue
        ach = c["flop"] / c["t"] / 1e12
        hw = hw_all.get(name, {})
        kern[name] = {"ms": c["t"] * 1e3, "share_of_step": c["t"] / (R["ms"] * 1e-3), "achieved": ach,
                      "peak": c["peak"], "frac": ach / c["peak"], "pipe": c["pipe"], "work": c["work"],
                      "traffic": hw.get("dram_bytes_per_launch"), "tensor_pipe_pct": hw.get("tensor_pct"),
                      "fp64_pipe_pct": hw.get("fp64_pct"), "hw_fp64_tflops": hw.get("hw_fp64_tflops")}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    d = kern[dom]
    roof = {"bound": "fp64", "kernel": dom, "achieved": d["achieved"], "achieved_kind": d["work"],
            "peak": d["peak"], "unit": "TFLOP/s", "frac": d["frac"], "traffic": d["traffic"],
            "traffic_source": "profiles/round2/kernel_hw.json (ncu dram__bytes_read+write, one launch, same workload)",
            "peak_source": ("measured live: " + ("DMMA" if "mma" in d["pipe"].lower() or "DMMA" in d["pipe"]
                                                 else "DFMA") + " microbenchmark (sdmk_fp64_mma_peak / sdmk_fp64_peak); "
                            "MEASURED_PEAKS.json has no FP64 figure"),
            "pipe": d["pipe"], "share_of_step": d["share_of_step"],
            "planewave_share_of_step": rep["t_planewave"] / (R["ms"] * 1e-3),
            "peaks_measured": {"dfma_tflops": peak, "dmma_tflops": peak_mma},
            "kernels": kern}
    # the algorithmic figure counts the reference's operations; where ncu gave the executed FP64 rate, say so
    roof["frac_kind"] = "algorithmic FLOPs of the reference's formulation / time / measured peak"
    if d.get("hw_fp64_tflops"):
        roof["hw_fp64_tflops"] = d["hw_fp64_tflops"]
        roof["frac_hw"] = d["hw_fp64_tflops"] / d["peak"]
        roof["frac_hw_kind"] = "FP64 operations the kernel executed (ncu, profiles/round2/residual_hw.json) / time / measured peak"
    elif d.get("tensor_pipe_pct"):
        roof["frac_hw"] = d["tensor_pipe_pct"] / 100.0
        roof["frac_hw_kind"] = "FP64 tensor pipe utilisation (ncu, profiles/round2/kernel_hw.json)"
    roof["multi_gpu_path"] = ("library NCCL communicator" if use_comm else "set_shard + torch all_reduce") if world > 1 else None
    return results, roof, clocks


def cpu_reference_sample(n_sample: int, seed: int, threads: int):
    from oracle import ref
    ref.set_threads(threads)
    x, s = make_system(0, n_sample, seed)
    plan = ref.select_parameters(0, 1e-6, 0, 3)
    R = ref.RefProblem(plan, 3, x, s)
    _, rp = R.evaluate()
    t = rp["t_tree"] + rp["t_upward"] + rp["t_root"] + rp["t_downward"] + rp["t_residual"]
    return n_sample / t, t, rp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--kernels", default="stokeslet,stresslet")
    ap.add_argument("--cpu-sample", type=int, default=100_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    threads = os.cpu_count() or 1
    config = {"workload": f"metric: 3D free-space DMK, N={args.n:.0e} iid uniform in [-1/2,1/2]^3, eps={args.eps:g}, "
                          "prolate window, targets = sources",
              "kernels": args.kernels, "n_points": args.n, "eps": args.eps, "seed": args.seed,
              "parallelism": (f"target-leaf shards x{world} (replicated tree; owner-local upward pass with NCCL halo exchange of outgoing expansions; NCCL all-reduce of u)"
                              if world > 1 else "single GPU"),
              "l2": "inputs (>=480 MB) and proxy grids (>10 GB) exceed the 126 MB L2; no flush needed"}

    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import ref
        if not ref.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        vals = []
        for i in range(args.warmup + args.steps):
            v, t, _ = cpu_reference_sample(args.cpu_sample, args.seed, threads)
            if i >= args.warmup:
                vals.append((v, t))
        v = float(np.mean([a for a, _ in vals]))
        ms = float(np.mean([t for _, t in vals])) * 1e3
        rcfg = dict(config)
        rcfg.update({"workload": f"bounded sample of the metric workload: 3D free-space DMK, N={args.cpu_sample} "
                                 f"iid uniform in [-1/2,1/2]^3, eps={args.eps:g}, prolate window, targets = sources",
                     "n_points": args.cpu_sample, "sample_of": args.n, "kernels": "stokeslet",
                     "parallelism": f"CPU, OpenMP {threads} threads (rank 0 only)"})
        line = {"metric": METRIC, "value": v, "unit": "points/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded uniform points, N(0,1) forces)", "config": rcfg, "impl": "reference",
                "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "reference",
                                 "sample": f"evaluate_with_plan on N={args.cpu_sample} points of the same "
                                           "distribution per step; the full N=1e7 run on this host's 16 cores is "
                                           "in profiles/round2/parity_full_size.jsonl (ref_time)"},
                "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    results, roof, clocks = run_ours(args, rank, world, local_rank)
    if rank != 0:
        return
    R = results.get("stokeslet") or next(iter(results.values()))
    n = args.n
    value = n / (R["ms"] * 1e-3)  # one N-point system per step, all ranks together
    e2e = n / (R["e2e_ms"] * 1e-3)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            v, t, rp = cpu_reference_sample(args.cpu_sample, args.seed, threads)
            cpu = {"value": v, "unit": "points/s", "cores": threads, "kind": "reference",
                   "sample": f"stokesdmk evaluate_with_plan (oracle/_ref, unmodified core, OpenMP {threads} threads) "
                             f"on N={args.cpu_sample} uniform points, eps=1e-6: {t:.2f} s"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "points/s", "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    extra = {}
    for k, r in results.items():
        extra[k] = {"points_per_s": n / (r["ms"] * 1e-3), "ms_per_step": r["ms"],
                    "e2e_points_per_s": n / (r["e2e_ms"] * 1e-3), "e2e_ms": r["e2e_ms"],
                    "e2e_pageable_ms": r.get("e2e_pageable_ms"),
                    "p": r["plan"]["p"], "N1": r["plan"]["N1"], "num_boxes": r["rep"]["num_boxes"],
                    "max_level": r["rep"]["max_level"],
                    "pass_s": {k2: r["rep"][k2] for k2 in ("t_tree", "t_upward", "t_root", "t_downward",
                                                           "t_residual", "t_residual_kernel", "t_planewave")}}
    line = {"metric": METRIC, "value": value, "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": R["ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform points, N(0,1) forces; stresslet normals random unit)",
            "config": config, "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "points/s", "h2d_bytes_per_step": n * 6 * 8, "d2h_bytes_per_step": n * 3 * 8,
                    "host_buffers": "pinned"},
            "e2e_pageable": ({"value": n / (R["e2e_pageable_ms"] * 1e-3), "unit": "points/s",
                              "h2d_bytes_per_step": n * 6 * 8, "d2h_bytes_per_step": n * 3 * 8,
                              "host_buffers": "pageable (numpy / std::vector)"}
                             if R.get("e2e_pageable_ms") else None),
            "gpu_launches": R["launches"] * args.steps, "clocks": clocks, "kernels": extra}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
