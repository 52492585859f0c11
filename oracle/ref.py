"""TEST INFRASTRUCTURE ONLY: ctypes binding of the compiled reference.

oracle/_ref/libsdmk_ref.so is the UNMODIFIED reference core
(/root/reference/proj/core/src/*.cpp) plus oracle/ref_shim.cpp, built by
oracle/Makefile.  Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline legs may use it -- as the checker and the CPU
baseline, never as the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libsdmk_ref.so")
REF_SRC = "/root/reference/proj/core"


class ref_plan(C.Structure):
    _fields_ = [("kernel", C.c_int), ("dim", C.c_int), ("window", C.c_int), ("tol", C.c_double),
                ("c", C.c_double), ("sigma", C.c_double), ("p", C.c_int), ("N1", C.c_int), ("N_per", C.c_int),
                ("n_s", C.c_int), ("table_tol", C.c_double)]


class ref_report(C.Structure):
    _fields_ = [("num_boxes", C.c_int), ("max_level", C.c_int), ("num_sources", C.c_int),
                ("num_targets", C.c_int), ("t_tree", C.c_double), ("t_upward", C.c_double),
                ("t_root", C.c_double), ("t_downward", C.c_double), ("t_residual", C.c_double)]


def build(quiet=True) -> bool:
    """Compile the reference oracle if its sources are present here."""
    if os.path.exists(LIB):
        return True
    if not os.path.isdir(REF_SRC):
        return False
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return os.path.exists(LIB)


def available() -> bool:
    return os.path.exists(LIB) or build()


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError("reference oracle not built (oracle/_ref/libsdmk_ref.so)")
        L = C.CDLL(LIB)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_select_parameters.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int, C.POINTER(ref_plan)]
        L.ref_setup.argtypes = [C.POINTER(ref_plan), C.c_int, C.c_int64, dp, C.c_int64, dp, dp, C.c_int]
        L.ref_tree_info.argtypes = [ip]
        L.ref_tree_boxes.argtypes = [ip]
        L.ref_tree_perm.argtypes = [ip, ip]
        L.ref_tree_dump.argtypes = [C.c_char_p, C.c_int64]
        L.ref_tree_dump.restype = C.c_int64
        for n in ["ref_upward", "ref_target_far", "ref_residual", "ref_direct_sum", "ref_periodic_zero_mode"]:
            getattr(L, n).argtypes = [dp]
        L.ref_incoming.argtypes = [C.c_int, dp]
        L.ref_evaluate.argtypes = [dp, C.POINTER(ref_report)]
        L.ref_direct_residual_sum.argtypes = [C.c_double, dp]
        L.ref_ewald_reference.argtypes = [C.c_int, dp]
        L.ref_self_scaled.argtypes = [C.c_double, dp]
        L.ref_export_tables.argtypes = [C.c_char_p]
        L.ref_window.argtypes = [dp, dp, C.c_int]
        for n in ["ref_window_fourier", "ref_mollifier_fourier", "ref_window_eval", "ref_phi_tail"]:
            getattr(L, n).argtypes = [C.c_double]
            getattr(L, n).restype = C.c_double
        L.ref_truncated_biharmonic_fourier.argtypes = [C.c_double, C.c_double, C.c_int]
        L.ref_truncated_biharmonic_fourier.restype = C.c_double
        L.ref_mollifier_taylor.argtypes = [dp]
        L.ref_residual_apply.argtypes = [dp, C.c_double, dp, dp]
        L.ref_run_full.argtypes = [dp, dp, dp, C.POINTER(ref_report)]
        L.ref_proxy.argtypes = [C.c_int, C.POINTER(C.c_int64)]
        L.ref_proxy.restype = dp
        L.ref_release.argtypes = []
        L.ref_release.restype = None
        L.ref_time_tree.argtypes = []
        L.ref_time_tree.restype = C.c_double
        L.ref_count_pairs.argtypes = [C.POINTER(C.c_int64)]
        L.ref_set_window.argtypes = [C.c_double, C.c_double]
        _lib = L
    return _lib


def _dp(a):
    if a is None:
        return C.cast(None, C.POINTER(C.c_double))
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _chk(code):
    if code:
        msg = lib().ref_last_error().decode()
        if msg.startswith("invalid_argument"):
            raise ValueError(msg)
        if msg.startswith("domain_error"):
            raise ArithmeticError(msg)
        raise RuntimeError(msg)


def set_threads(n: int) -> int:
    return lib().ref_set_threads(int(n))


def select_parameters(kernel: int, eps: float, window: int, dim: int) -> dict:
    p = ref_plan()
    _chk(lib().ref_select_parameters(kernel, eps, window, dim, C.byref(p)))
    return {k: getattr(p, k) for k, _ in ref_plan._fields_}


class RefProblem:
    """One problem held by the reference shim (plan + system + tables + tree)."""

    def __init__(self, plan: dict, dim: int, sources, strengths, targets=None, periodic=False):
        self.plan = dict(plan)
        self.dim = dim
        src = np.ascontiguousarray(np.asarray(sources, np.float64).ravel())
        stw = np.ascontiguousarray(np.asarray(strengths, np.float64).ravel())
        tgt = None if targets is None or np.asarray(targets).size == 0 else \
            np.ascontiguousarray(np.asarray(targets, np.float64).ravel())
        self.ns = src.size // dim
        self.nt = tgt.size // dim if tgt is not None else self.ns
        rp = ref_plan(**{k: self.plan[k] for k, _ in ref_plan._fields_})
        _chk(lib().ref_setup(C.byref(rp), dim, self.ns, _dp(src), 0 if tgt is None else self.nt, _dp(tgt),
                             _dp(stw), int(periodic)))
        info = (C.c_int * 7)()
        lib().ref_tree_info(info)
        self.info = dict(zip(["num_boxes", "max_level", "n_src", "n_tgt", "alias", "depth_capped", "channels"],
                             list(info)))

    def tree_dump(self) -> str:
        n = lib().ref_tree_dump(None, 0)
        buf = C.create_string_buffer(int(n))
        lib().ref_tree_dump(buf, n)
        return buf.raw[:n].decode()

    def tree_boxes(self):
        nb = self.info["num_boxes"]
        out = np.zeros(nb * 11, np.int32)
        lib().ref_tree_boxes(out.ctypes.data_as(C.POINTER(C.c_int)))
        return out.reshape(nb, 11)

    def tree_perm(self):
        sp = np.zeros(self.info["n_src"], np.int32)
        tp = np.zeros(self.info["n_tgt"], np.int32)
        lib().ref_tree_perm(sp.ctypes.data_as(C.POINTER(C.c_int)), tp.ctypes.data_as(C.POINTER(C.c_int)))
        return sp, (None if self.info["alias"] else tp)

    def _nodes(self):
        return self.plan["p"] ** self.dim

    def upward(self):
        out = np.empty(self.info["num_boxes"] * self.info["channels"] * self._nodes())
        _chk(lib().ref_upward(_dp(out)))
        return out

    def incoming(self, stage=1):
        out = np.empty(self.info["num_boxes"] * self.dim * self._nodes())
        _chk(lib().ref_incoming(stage, _dp(out)))
        return out

    def target_far(self):
        out = np.empty(self.nt * self.dim)
        _chk(lib().ref_target_far(_dp(out)))
        return out

    def residual(self):
        out = np.empty(self.nt * self.dim)
        _chk(lib().ref_residual(_dp(out)))
        return out

    def evaluate(self):
        out = np.empty(self.nt * self.dim)
        rep = ref_report()
        _chk(lib().ref_evaluate(_dp(out), C.byref(rep)))
        return out, {k: getattr(rep, k) for k, _ in ref_report._fields_}

    def direct_sum(self):
        out = np.empty(self.nt * self.dim)
        _chk(lib().ref_direct_sum(_dp(out)))
        return out

    def direct_residual_sum(self, cutoff):
        out = np.empty(self.nt * self.dim)
        _chk(lib().ref_direct_residual_sum(cutoff, _dp(out)))
        return out

    def ewald_reference(self, periodic=True):
        out = np.empty(self.nt * self.dim)
        _chk(lib().ref_ewald_reference(1 if periodic else 0, _dp(out)))
        return out

    def self_scaled(self, nu):
        v = C.c_double()
        _chk(lib().ref_self_scaled(nu, C.byref(v)))
        return v.value

    def export_tables(self, path):
        _chk(lib().ref_export_tables(path.encode()))

    # ---- full-size parity (tools/parity_configs.py) ----
    def run_full(self):
        """The passes of evaluate_with_plan once (shim ref_run_full): returns
        far, residual, u (caller order) and the pass times; the proxies stay
        alive for proxy() until release()."""
        far, res, u = (np.empty(self.nt * self.dim) for _ in range(3))
        rep = ref_report()
        _chk(lib().ref_run_full(_dp(far), _dp(res), _dp(u), C.byref(rep)))
        return far, res, u, {k: getattr(rep, k) for k, _ in ref_report._fields_}

    def proxy(self, which: int):
        """Zero-copy view of the kept outgoing (0) / incoming (1) proxies."""
        n = C.c_int64()
        ptr = lib().ref_proxy(which, C.byref(n))
        if n.value == 0:
            return np.empty(0)
        return np.ctypeslib.as_array(ptr, shape=(n.value,))

    def release(self):
        lib().ref_release()

    def time_tree(self) -> float:
        return lib().ref_time_tree()

    def count_pairs(self):
        """(tested, in_support, coincident) pairs of the reference's residual loop."""
        out = (C.c_int64 * 3)()
        _chk(lib().ref_count_pairs(out))
        return tuple(int(v) for v in out)

    def set_window(self, c: float = 0.0, sigma: float = 0.0):
        """Rebuild the problem's split tables with another window (same kernel, dim, table_tol)."""
        _chk(lib().ref_set_window(float(c), float(sigma)))

