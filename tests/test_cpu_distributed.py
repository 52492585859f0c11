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
    # cost-balanced (host/tree.hpp shard_costs) to within one leaf's cost
    boxes = _parse_dump(g.host_topology_dump(3, False, 300, 10, qs))
    tl, w = _shard_costs(boxes)
    tb = [boxes[i]["tb"] for i in tl]
    for p in plans:
        c = sum(wi for t0, wi in zip(tb, w) if p["t0"] <= t0 < p["t1"])
        assert abs(c - sum(w) / nranks) <= max(w)
        assert p["needed_boxes"] >= p["owned_leaves"]
    if nranks == 1:
        assert plans[0]["owned_leaves"] == plans[0]["target_leaves"]


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_shard_bounds_equal_per_rank_plans(nranks):
    """sdmk_host_shard_bounds (the u all-gather layout) equals each rank's shard plan."""
    qs = _points(20000, seed=4)
    b = g.host_shard_bounds(3, False, 300, 10, qs, nranks)
    assert b[0] == 0 and b[-1] == qs.shape[0] and np.all(np.diff(b) >= 0)
    for r in range(nranks):
        p = g.host_shard_plan(3, False, 300, 10, qs, r, nranks)
        if p["t1"] > p["t0"]:
            assert (b[r], b[r + 1]) == (p["t0"], p["t1"])
        else:
            assert b[r] == b[r + 1]


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
    # the library's assembly (engine.cpp evaluate_end): pack the owned sorted
    # rows, all-gather them padded to the longest range, scatter to caller
    # order through the target permutation (here a random one)
    bounds = g.host_shard_bounds(3, False, 300, 10, qs, world)
    perm = torch.from_numpy(np.random.default_rng(9).permutation(n))
    caller = torch.empty_like(full)
    caller[perm] = full  # u in caller order: caller[perm[s]] = sorted row s
    maxc = int(max(bounds[r + 1] - bounds[r] for r in range(world)))
    snd = torch.zeros(maxc, 3, dtype=torch.float64)
    t0, t1 = int(bounds[rank]), int(bounds[rank + 1])
    snd[: t1 - t0] = caller[perm[t0:t1]]
    rcv = [torch.empty_like(snd) for _ in range(world)]
    dist.all_gather(rcv, snd)
    out = torch.full_like(full, float("nan"))
    for r in range(world):
        a, b = int(bounds[r]), int(bounds[r + 1])
        out[perm[a:b]] = rcv[r][: b - a]
    ok_ag = bool(torch.equal(out, caller)) and t0 == plan["t0"] and t1 == plan["t1"]
    # the halo exchange plan of the distributed upward pass: the same on both
    # processes, and its send / receive sizes pair up in an all-to-all (the
    # shape of the library's NCCL group of sends and receives)
    h = g.host_halo_plan(3, False, 300, 10, qs, world)
    hs = [None] * world
    dist.all_gather_object(hs, h["recv"].tolist())
    send = [int(h["recv"][rank, q]) for q in range(world)]
    recv = [int(h["recv"][f, rank]) for f in range(world)]
    payload = torch.full((sum(send),), float(rank + 1), dtype=torch.float64)
    got = torch.empty(sum(recv), dtype=torch.float64)
    dist.all_to_all_single(got, payload, output_split_sizes=recv, input_split_sizes=send)
    ok_x = hs[0] == hs[1] and bool((got == float(2 - rank)).all()) and sum(recv) > 0
    if rank == 0:
        out_q.put((plans, bool(torch.equal(part, full)) and ok_x and ok_ag))
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


# ---- distributed upward pass: the exchange plan, restated from the tree dump ----

def _parse_dump(text):
    boxes = []
    for line in text.splitlines()[1:]:
        f = line.split()
        lev = int(f[1][1:])
        anc = tuple(int(v) for v in f[2][2:].split(","))
        sb, se = (int(v) for v in f[4][5:-1].split(","))
        tb, te = (int(v) for v in f[5][5:-1].split(","))
        def lst(tag):
            body = line[line.index(tag + "={") + len(tag) + 2:line.index("}", line.index(tag + "={"))]
            out = []
            for e in body.split():
                bx, _, sh = e.partition("@")
                out.append((int(bx), tuple(int(v) for v in sh.split(",")) if sh else (0, 0, 0)))
            return out
        col, crs, fin = lst("col"), lst("crs"), lst("fin")
        boxes.append(dict(level=lev, a=anc, leaf=f[3] == "leaf", ns=se - sb, nt=te - tb, sb=sb, tb=tb,
                          col=[c for c, _ in col], colsh=col, crs=crs, fin=fin))
    key = {(b["level"], b["a"]): i for i, b in enumerate(boxes)}
    for i, b in enumerate(boxes):
        b["children"] = []
        if b["level"] == 0:
            b["parent"] = -1
            continue
        side = 1 << (30 - b["level"] + 1)
        b["parent"] = key[(b["level"] - 1, tuple(v - v % side for v in b["a"]))]
    for i, b in enumerate(boxes):
        if b["parent"] >= 0:
            boxes[b["parent"]]["children"].append(i)
    return boxes


def _shard_costs(boxes):
    """host/tree.hpp shard_costs: nt * (near sources + 1190) + sum over the
    leaf and its ancestors a of 860000 * nt // nt(a) per target leaf, near sources = own box + colleague leaves (not the
    zero-shift self entry) + coarse + fine neighbours (dmk.cpp:966-990)."""
    tl = sorted((i for i, b in enumerate(boxes) if b["leaf"] and b["nt"] > 0), key=lambda i: boxes[i]["tb"])
    w = []
    for i in tl:
        b = boxes[i]
        near = b["ns"]
        near += sum(boxes[c]["ns"] for c, sh in b["colsh"] if not (c == i and sh == (0, 0, 0)) and boxes[c]["leaf"])
        near += sum(boxes[c]["ns"] for c, _ in b["crs"]) + sum(boxes[c]["ns"] for c, _ in b["fin"])
        bw, a = 0, i
        while a >= 0:
            bw += 860000 * b["nt"] // boxes[a]["nt"]
            a = boxes[a]["parent"]
        w.append(b["nt"] * (near + 1190) + bw)
    return tl, w


def _halo_plan_restated(boxes, R_):
    """include/sdmk.h sdmk_comm_init: cut subtrees of <= N/(8R) sources dealt
    to ranks by source midpoint; rank r reads the colleagues of its plane-wave
    targets (targets whose parent it needs, the shard plan); it receives from
    f every box f owns that it reads, and every cut box."""
    total = boxes[0]["ns"]
    thr = max(1, total // (8 * R_))
    owner = [-2] * len(boxes)
    cut, stack = [], [0]
    while stack:
        b = stack.pop()
        if boxes[b]["ns"] == 0:
            continue
        if not boxes[b]["leaf"] and boxes[b]["ns"] > thr and R_ > 1:
            owner[b] = -1
            stack += boxes[b]["children"]
        else:
            cut.append(b)
    cut.sort(key=lambda b: boxes[b]["sb"])
    start = 0
    for c in cut:
        n = boxes[c]["ns"]
        r = 0 if R_ == 1 else min(R_ - 1, ((2 * start + n) * R_) // (2 * total))
        start += n
        st = [c]
        while st:
            x = st.pop()
            if boxes[x]["ns"]:
                owner[x] = r
                st += boxes[x]["children"]
    # target shards (host shard plan): leaves by target start, cost midpoint rule
    tl, w = _shard_costs(boxes)
    tt = sum(w)
    need = [[False] * len(boxes) for _ in range(R_)]
    s0 = 0
    for i, n in zip(tl, w):
        r = 0 if R_ == 1 else min(R_ - 1, ((2 * s0 + n) * R_) // (2 * tt))
        s0 += n
        x = i
        while x >= 0 and not need[r][x]:
            need[r][x] = True
            x = boxes[x]["parent"]
    reads = [[False] * len(boxes) for _ in range(R_)]
    for r in range(R_):
        for i, b in enumerate(boxes):
            par = b["parent"]
            if b["nt"] and need[r][par if par >= 0 else i]:
                for c in b["col"]:
                    if boxes[c]["ns"]:
                        reads[r][c] = True
    cutset = set(cut)
    recv = np.zeros((R_, R_), np.int64)
    for f in range(R_):
        for r in range(R_):
            if f != r:
                recv[f, r] = sum(1 for i in range(len(boxes)) if owner[i] == f and (i in cutset or reads[r][i]))
    owned = np.array([sum(1 for i, b in enumerate(boxes) if b["leaf"] and owner[i] == r) for r in range(R_)])
    # closure: every box a rank reads is its own, above the cut, or received;
    # every box above the cut has all its children with sources available
    for r in range(R_):
        for i in range(len(boxes)):
            if reads[r][i]:
                assert owner[i] >= -1
    return recv, owned, sum(1 for o in owner if o == -1), len(cut), owner


@pytest.mark.parametrize("nranks,periodic,n_s", [(2, False, 300), (3, False, 300), (8, False, 120), (4, True, 200)])
def test_halo_plan_matches_restatement(nranks, periodic, n_s):
    qs = _points(20000, seed=nranks)
    h = g.host_halo_plan(3, periodic, n_s, 10, qs, nranks)
    boxes = _parse_dump(g.host_topology_dump(3, periodic, n_s, 10, qs))
    recv, owned, above, ncut, owner = _halo_plan_restated(boxes, nranks)
    np.testing.assert_array_equal(h["recv"], recv)
    np.testing.assert_array_equal(h["owned_leaves"], owned)
    assert h["above_cut"] == above and h["cut_boxes"] == ncut
    # every leaf with sources has exactly one owner; above-cut boxes are never leaves
    assert owned.sum() == sum(1 for b in boxes if b["leaf"] and b["ns"] > 0)
    assert all(not boxes[i]["leaf"] for i, o in enumerate(owner) if o == -1)
    # source balance of the cut: within one cut box of N / nranks
    if nranks > 1:
        per = np.zeros(nranks)
        for i, o in enumerate(owner):
            if o >= 0 and boxes[i]["leaf"]:
                per[o] += boxes[i]["ns"]
        assert np.abs(per - per.mean()).max() <= 20000 / (8 * nranks) + 1


def test_halo_plan_single_rank_is_empty():
    qs = _points(5000)
    h = g.host_halo_plan(3, False, 200, 8, qs, 1)
    assert h["recv"].sum() == 0 and h["above_cut"] == 0 and h["cut_boxes"] == 1
