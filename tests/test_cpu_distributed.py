"""Multi-GPU host logic on CPU: the target-leaf shard plan (SURVEY section
8(e)) and the all-reduce assembly, with torch.distributed over gloo at
world size 2 (no GPU needed).  The GPU side -- sum over shards bitwise equal
to the single-GPU result -- is tests/test_gpu_parity.py::test_shards_sum_to_single."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2509_21471_b200 as g
from oracle import restate as R


def _points(n, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5, 0.5, (n, 3))
    x[: n // 3] = 0.5 * x[: n // 3] * 0.1 + 0.2  # a dense cluster: uneven leaves
    q = R.quantize(x)
    return q[R.morton_order(q)]


@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
def test_shard_plan_tiles_targets(nranks):
    qs = _points(20000)
    plans = [g.host_shard_plan(3, False, 300, 10, qs, r, nranks) for r in range(nranks)]
    total = qs.shape[0]
    # contiguous Morton runs covering every target exactly once, in rank order
    assert plans[0]["t0"] == 0 and plans[-1]["t1"] == total
    for a, b in zip(plans, plans[1:]):
        assert a["t1"] == b["t0"]
    assert sum(p["owned_leaves"] for p in plans) == plans[0]["target_leaves"]
    # balanced to within one leaf (leaves hold <= n_s sources)
    for p in plans:
        assert abs((p["t1"] - p["t0"]) - total / nranks) <= 300
        assert p["needed_boxes"] >= p["owned_leaves"]
    if nranks == 1:
        assert plans[0]["owned_leaves"] == plans[0]["target_leaves"]


def test_shard_plan_rejects_bad_rank():
    qs = _points(1000)
    with pytest.raises(ValueError):
        g.host_shard_plan(3, False, 100, 8, qs, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, qs, out_q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    plan = g.host_shard_plan(3, False, 300, 10, qs, rank, world)
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    # each rank fills its owned Morton range of a per-target field; zeros elsewhere
    n = qs.shape[0]
    full = torch.arange(n * 3, dtype=torch.float64).reshape(n, 3).sin()
    part = torch.zeros_like(full)
    part[plan["t0"]:plan["t1"]] = full[plan["t0"]:plan["t1"]]
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    if rank == 0:
        out_q.put((plans, bool(torch.equal(part, full))))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_assembles_full_result():
    qs = _points(20000, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qs, q)) for r in range(2)]
    for p in procs:
        p.start()
    plans, equal = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert equal
    assert plans[0]["t0"] == 0 and plans[0]["t1"] == plans[1]["t0"] and plans[1]["t1"] == qs.shape[0]
