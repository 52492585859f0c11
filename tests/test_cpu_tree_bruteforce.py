"""The product's host topology (csrc/host/tree.cpp, through
sdmk_host_topology_dump) against brute force, as the reference's
test_tree.cpp:56-99 does for its own tree: colleague / coarse / fine lists
equal the sets of touching boxes over all pairs and image shifts, colleague
lists hold at most 3^d entries including the box itself, and touching leaves
differ by at most one level (2:1 balance)."""
import itertools
import re

import numpy as np
import pytest

import paper_2509_21471_b200 as g
from oracle import restate as R

CELLS = 1 << 30


def parse(dump):
    lines = dump.strip().split("\n")
    head = dict(kv.split("=") for kv in lines[0].split()[1:])
    dim, periodic = int(head["dim"]), int(head["periodic"])
    boxes = []
    for ln in lines[1:]:
        m = re.match(r"(\d+) L(\d+) a=([\d,]+) (leaf|node) src=\[(\d+),(\d+)\) tgt=\[(\d+),(\d+)\)"
                     r" col=\{(.*?)\} crs=\{(.*?)\} fin=\{(.*?)\}", ln)
        assert m, ln
        def lst(s):
            out = set()
            for e in s.split():
                if "@" in e:
                    b, sh = e.split("@")
                    out.add((int(b),) + tuple(int(v) for v in sh.split(",")))
                else:
                    out.add((int(e), 0, 0, 0))
            return out
        boxes.append({"level": int(m.group(2)), "anchor": [int(v) for v in m.group(3).split(",")],
                      "leaf": m.group(4) == "leaf", "col": lst(m.group(9)), "crs": lst(m.group(10)),
                      "fin": lst(m.group(11))})
    # parents from geometry (the dump has no parent field): the level-(L-1) box containing the anchor
    return dim, periodic, boxes


def touch(b, c, sh, dim):
    sb, sc = CELLS >> b["level"], CELLS >> c["level"]
    for a in range(dim):
        l1, l2 = b["anchor"][a], c["anchor"][a] + sh[a] * CELLS
        if l1 > l2 + sc or l2 > l1 + sb:
            return False
    return True


def contains(p, c, dim):
    s = CELLS >> p["level"]
    return all(p["anchor"][a] <= c["anchor"][a] < p["anchor"][a] + s for a in range(dim))


def check(dump):
    dim, periodic, boxes = parse(dump)
    rng = [-1, 0, 1] if periodic else [0]
    shifts = [s + (0,) * (3 - dim) for s in itertools.product(rng, repeat=dim)]
    for bi, b in enumerate(boxes):
        col, crs, fin = set(), set(), set()
        for ci, c in enumerate(boxes):
            for s in shifts:
                if not touch(b, c, s, dim):
                    continue
                if c["level"] == b["level"]:
                    col.add((ci,) + s)
                if c["level"] == b["level"] - 1 and c["leaf"]:
                    crs.add((ci,) + s)
                if c["level"] == b["level"] + 1 and c["leaf"] and not (s == (0, 0, 0) and contains(b, c, dim)):
                    fin.add((ci,) + s)
        assert b["col"] == col, bi
        assert b["crs"] == crs, bi
        assert b["fin"] == fin, bi
        assert len(b["col"]) <= 3 ** dim and (bi, 0, 0, 0) in b["col"]
    leaves = [i for i, b in enumerate(boxes) if b["leaf"]]
    for i in leaves:
        for j in leaves:
            if j > i and any(touch(boxes[i], boxes[j], s, dim) for s in shifts):
                assert abs(boxes[i]["level"] - boxes[j]["level"]) <= 1


@pytest.mark.parametrize("dim,periodic,dist,n,n_s", [
    (3, False, "uniform", 3000, 40), (3, False, "cluster", 3000, 20), (3, True, "cluster", 2000, 20),
    (2, False, "cluster", 3000, 10), (2, True, "uniform", 2000, 15)])
def test_neighbour_lists_match_brute_force(dim, periodic, dist, n, n_s):
    rng = np.random.default_rng(n + dim)
    x = rng.uniform(-0.5, 0.5, (n, dim))
    if dist == "cluster":  # deep, unbalanced trees that need 2:1 repairs
        x[: n // 2] = np.clip(0.31 + 0.01 * rng.standard_normal((n // 2, dim)), -0.5, 0.5)
    q = R.quantize(x)
    dump = g.host_topology_dump(dim, periodic, n_s, 5, q[R.morton_order(q)])
    check(dump)
