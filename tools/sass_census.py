"""SASS instruction census of the dominant kernels (cuobjdump -sass on the
built objects): static counts of the instructions that show which hardware
paths a kernel uses -- DMMA (FP64 tensor core), DFMA/DMUL/DADD (FP64 pipe),
LDGSTS (cp.async), UBLKCP / UTMALDG (TMA bulk / tensor-map copies),
SYNCS (mbarrier), LDS/STS (shared memory), LDG/STG, SHFL, ATOM/RED.

usage: python tools/sass_census.py > profiles/round2/sass_census.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2509_21471_b200", "csrc", "build", "kernels")
KERNELS = [  # (object, kernel-name regex)
    ("residual.o", r"k_residual<0, 3, 6, 0>"),
    ("anterp_mma.o", r"k_anterp2<9, 3, 23, 0, 3, 12, 64>"),
    ("anterp_mma.o", r"k_interp_mma<3, 23, 3"),
    ("anterp_mma.o", r"k_basis<23>"),
    ("tree_kernels.o", r"k_refine"),
    ("tree_kernels.o", r"k_repair_scan"),
    ("tree_kernels.o", r"k_morton"),
    ("planewave.o", r"k_acc_group<0, 3, 1>"),
    ("planewave_mma.o", r"k_fwd_xy3<23, 33, 8>"),
    ("planewave_mma.o", r"k_zf3"),
    ("planewave_mma.o", r"k_zi3"),
    ("planewave_mma.o", r"k_inv_xy3<23, 33>"),
    ("tensor_mma.o", r"k_tensor_up<23>"),
    ("tensor_mma.o", r"k_tensor_down<23>"),
    ("ewald.o", r"k_ew_spread"),
    ("ewald.o", r"k_ew_gather"),
]
CLASSES = ["DMMA", "DFMA", "DMUL", "DADD", "LDGSTS", "UBLKCP", "UTMALDG", "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL", "REDG",
           "ATOM", "RED", "BAR", "MUFU"]


def kernels_in(obj):
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    funcs, cur, name = {}, [], None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
        elif name:
            cur.append(line)
    if name:
        funcs[name] = cur
    return funcs


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    print("# static SASS instruction counts (cuobjdump -sass, sm_100a), one line per kernel")
    print("# " + " ".join(f"{c:>7s}" for c in CLASSES) + "  kernel")
    cache = {}
    for obj, pat in KERNELS:
        if obj not in cache:
            f = kernels_in(obj)
            cache[obj] = (f, demangle(list(f)))
        funcs, dm = cache[obj]
        hit = [m for m in funcs if re.search(re.escape(pat).replace(r"\ ", " "), dm[m])]
        if not hit:
            print(f"# (not found: {pat})")
            continue
        body = funcs[hit[0]]
        cnt = collections.Counter()
        for line in body:
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+)", line)
            if m:
                cnt[m.group(1)] += 1
        print("  " + " ".join(f"{cnt[c]:7d}" for c in CLASSES) + "  " + dm[hit[0]][:90])


if __name__ == "__main__":
    sys.exit(main())
