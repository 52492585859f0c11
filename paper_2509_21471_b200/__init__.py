"""B200-native DMK hot path (stokesdmk drop-in), Python mirror.

The product is ``libsdmk_b200.so`` (CUDA kernels for sm_100a + C++ host
engine) behind the C-ABI in ``include/sdmk.h``.  This module binds that ABI
with ctypes and mirrors the reference's public API names and argument meaning
(``/root/reference/proj/core/include/stokesdmk/dmk.hpp``):

    select_parameters(kernel, eps, window, dim)          dmk.hpp:50-51
    evaluate_with_plan(plan, sys, mode, report=None)      dmk.hpp:151-155
    evaluate(kernel, sys, eps, window, mode, report=None) dmk.hpp:159-161
    outgoing_channels(kernel, dim)                        dmk.hpp:59

Errors map back to the reference's exception types: ``ValueError`` for
std::invalid_argument, ``ArithmeticError`` (DomainError) for
std::domain_error, ``RuntimeError`` otherwise.  There is no CPU fallback: if
the library or a B200 is missing, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDMK_LIB") or os.path.join(_HERE, "libsdmk_b200.so")  # SDMK_LIB: A/B builds

STOKESLET, STRESSLET, ROTLET = 0, 1, 2
PROLATE, GAUSSIAN = 0, 1
FREE_SPACE, PERIODIC = 0, 1

KERNELS = {"stokeslet": STOKESLET, "stresslet": STRESSLET, "rotlet": ROTLET}
WINDOWS = {"prolate": PROLATE, "gaussian": GAUSSIAN}
MODES = {"free_space": FREE_SPACE, "free": FREE_SPACE, "periodic": PERIODIC}


class DomainError(ArithmeticError):
    """std::domain_error (coincident points)."""


class CudaError(RuntimeError):
    pass


class sdmk_plan(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("dim", C.c_int32), ("window", C.c_int32), ("tol", C.c_double),
                ("c", C.c_double), ("sigma", C.c_double), ("p", C.c_int32), ("N1", C.c_int32),
                ("N_per", C.c_int32), ("n_s", C.c_int32), ("table_tol", C.c_double)]


class sdmk_report(C.Structure):
    _fields_ = [("num_boxes", C.c_int32), ("max_level", C.c_int32), ("num_sources", C.c_int32),
                ("num_targets", C.c_int32), ("t_tree", C.c_double), ("t_upward", C.c_double),
                ("t_root", C.c_double), ("t_downward", C.c_double), ("t_residual", C.c_double),
                ("t_h2d", C.c_double), ("t_d2h", C.c_double), ("t_total", C.c_double),
                ("p2p_candidates", C.c_int64), ("p2p_in_support", C.c_int64), ("kernel_launches", C.c_int32),
                ("t_residual_kernel", C.c_double), ("t_planewave", C.c_double), ("t_exchange", C.c_double),
                ("halo_bytes_sent", C.c_int64), ("halo_bytes_recv", C.c_int64),
                ("t_interp_kernel", C.c_double), ("t_anterp_kernel", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libsdmk_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `make -C paper_2509_21471_b200/csrc` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        dp, ip = P(C.c_double), P(C.c_int32)
        sig = {
            "sdmk_last_error": ([], C.c_char_p),
            "sdmk_device_ok": ([C.c_int], C.c_int),
            "sdmk_create": ([C.c_int, P(C.c_void_p)], C.c_int),
            "sdmk_destroy": ([C.c_void_p], C.c_int),
            "sdmk_select_parameters": ([C.c_int, C.c_double, C.c_int, C.c_int, P(sdmk_plan)], C.c_int),
            "sdmk_outgoing_channels": ([C.c_int, C.c_int], C.c_int),
            "sdmk_strength_components": ([C.c_int, C.c_int], C.c_int),
            "sdmk_load_tables": ([C.c_void_p, C.c_char_p], C.c_int),
            "sdmk_save_tables": ([C.c_void_p, P(sdmk_plan), C.c_char_p], C.c_int),
            "sdmk_evaluate_with_plan": ([C.c_void_p, P(sdmk_plan), C.c_int, C.c_int64, dp, C.c_int64, dp, dp,
                                         C.c_int, dp, P(sdmk_report)], C.c_int),
            "sdmk_evaluate": ([C.c_void_p, C.c_int, C.c_int, C.c_int64, dp, C.c_int64, dp, dp, C.c_double,
                               C.c_int, C.c_int, dp, P(sdmk_report)], C.c_int),
            "sdmk_evaluate_device": ([C.c_void_p, P(sdmk_plan), C.c_int, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, P(sdmk_report)], C.c_int),
            "sdmk_setup": ([C.c_void_p, P(sdmk_plan), C.c_int, C.c_int64, dp, C.c_int64, dp, dp, C.c_int], C.c_int),
            "sdmk_tree_info": ([C.c_void_p, ip], C.c_int),
            "sdmk_tree_boxes": ([C.c_void_p, ip], C.c_int),
            "sdmk_tree_perm": ([C.c_void_p, ip, ip], C.c_int),
            "sdmk_tree_dump": ([C.c_void_p, C.c_char_p, C.c_int64], C.c_int64),
            "sdmk_upward_pass": ([C.c_void_p, dp], C.c_int),
            "sdmk_incoming": ([C.c_void_p, C.c_int, dp], C.c_int),
            "sdmk_target_far_fields": ([C.c_void_p, dp], C.c_int),
            "sdmk_residual_pass": ([C.c_void_p, dp], C.c_int),
            "sdmk_get_stream": ([C.c_void_p, P(C.c_void_p)], C.c_int),
            "sdmk_fp64_peak": ([C.c_void_p, P(C.c_double)], C.c_int),
            "sdmk_fp64_mma_peak": ([C.c_void_p, P(C.c_double)], C.c_int),
            "sdmk_set_guard": ([C.c_void_p, C.c_int], C.c_int),
            "sdmk_guard_check": ([C.c_void_p, C.c_char_p, C.c_int64], C.c_int64),
            "sdmk_guard_selftest": ([C.c_void_p], C.c_int),
            "sdmk_host_save_tables": ([P(sdmk_plan), C.c_char_p], C.c_int),
            "sdmk_host_symbol_table": ([P(sdmk_plan), C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, dp],
                                       C.c_int),
            "sdmk_host_topology_dump": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, ip, C.c_int64, ip,
                                         C.c_char_p, C.c_int64], C.c_int64),
            "sdmk_set_shard": ([C.c_void_p, C.c_int, C.c_int], C.c_int),
            "sdmk_comm_unique_id": ([C.c_char_p], C.c_int),
            "sdmk_comm_init": ([C.c_void_p, C.c_int, C.c_int, C.c_char_p], C.c_int),
            "sdmk_set_manual_exchange": ([C.c_void_p, C.c_int], C.c_int),
            "sdmk_evaluate_begin": ([C.c_void_p, P(sdmk_plan), C.c_int, C.c_int64, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int),
            "sdmk_halo_transfer": ([C.c_void_p, C.c_void_p], C.c_int),
            "sdmk_evaluate_end": ([C.c_void_p, C.c_void_p, P(sdmk_report)], C.c_int),
            "sdmk_direct_sum": ([C.c_void_p, C.c_int, C.c_int, C.c_int64, dp, C.c_int64, dp, dp, dp], C.c_int),
            "sdmk_direct_residual_sum": ([C.c_void_p, P(sdmk_plan), C.c_int, C.c_int64, dp, C.c_int64, dp, dp,
                                          C.c_double, C.c_int, dp], C.c_int),
            "sdmk_host_halo_plan": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, ip, C.c_int64, ip, C.c_int,
                                     P(C.c_int64)], C.c_int),
            "sdmk_ewald": ([C.c_void_p, P(sdmk_plan), C.c_int64, dp, C.c_int64, dp, dp, dp, C.c_int, dp], C.c_int),
            "sdmk_ewald_device": ([C.c_void_p, P(sdmk_plan), C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int, dp], C.c_int),
            "sdmk_host_build_tables": ([C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_char_p,
                                        C.c_int64], C.c_int64),
            "sdmk_host_build_window": ([C.c_int, C.c_double, C.c_double, dp, dp, C.c_int], C.c_int),
            "sdmk_host_window_eval": ([C.c_int, C.c_double, C.c_double, dp, C.c_int, dp, C.c_int, C.c_int64, dp, dp],
                                      C.c_int),
            "sdmk_host_shard_bounds": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, ip, C.c_int64, ip, C.c_int,
                                        P(C.c_int64)], C.c_int),
            "sdmk_host_shard_plan": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, ip, C.c_int64, ip, C.c_int,
                                      C.c_int, P(C.c_int64)], C.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _raise(code: int):
    if code == 0:
        return
    msg = lib().sdmk_last_error().decode()
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise DomainError(msg)
    if code == 4:
        raise CudaError(msg)
    if code == 5:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return C.cast(None, C.POINTER(C.c_double))
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a: Optional[np.ndarray]):
    if a is None:
        return C.cast(None, C.POINTER(C.c_int32))
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _enum(v, table):
    return table[v] if isinstance(v, str) else int(v)


@dataclass
class DmkPlan:
    """stokesdmk::DmkPlan (dmk.hpp:27-40)."""
    kernel: int = STOKESLET
    dim: int = 3
    window: int = PROLATE
    tol: float = 1e-6
    c: float = 0.0
    sigma: float = 0.0
    p: int = 0
    N1: int = 0
    N_per: int = 0
    n_s: int = 0
    table_tol: float = 0.0

    def to_c(self) -> sdmk_plan:
        return sdmk_plan(self.kernel, self.dim, self.window, self.tol, self.c, self.sigma, self.p, self.N1,
                         self.N_per, self.n_s, self.table_tol)

    @staticmethod
    def from_c(p: sdmk_plan) -> "DmkPlan":
        return DmkPlan(p.kernel, p.dim, p.window, p.tol, p.c, p.sigma, p.p, p.N1, p.N_per, p.n_s, p.table_tol)


@dataclass
class ParticleSystem:
    """stokesdmk::ParticleSystem (oracle.hpp:29-46): point-major arrays."""
    dim: int = 3
    sources: np.ndarray = field(default_factory=lambda: np.zeros(0))
    targets: np.ndarray = field(default_factory=lambda: np.zeros(0))
    strengths: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def num_sources(self) -> int:
        return int(np.asarray(self.sources).size // self.dim)

    def num_targets(self) -> int:
        t = np.asarray(self.targets)
        return self.num_sources() if t.size == 0 else int(t.size // self.dim)


def select_parameters(kernel, eps: float, window=PROLATE, dim: int = 3) -> DmkPlan:
    out = sdmk_plan()
    _raise(lib().sdmk_select_parameters(_enum(kernel, KERNELS), float(eps), _enum(window, WINDOWS), int(dim),
                                        C.byref(out)))
    return DmkPlan.from_c(out)


def outgoing_channels(kernel, dim: int) -> int:
    r = lib().sdmk_outgoing_channels(_enum(kernel, KERNELS), int(dim))
    if r < 0:
        _raise(1)
    return r


def strength_components(kernel, dim: int) -> int:
    return lib().sdmk_strength_components(_enum(kernel, KERNELS), int(dim))


def _arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())


def _check_lengths(kernel: int, d: int, src: np.ndarray, tgt: np.ndarray, stw: np.ndarray):
    """validate_system's length checks (oracle.cpp:103-118), before the C-ABI reads any array."""
    if kernel not in (STOKESLET, STRESSLET, ROTLET):
        raise ValueError("particle sums support the Stokeslet, stresslet, and rotlet kernels")
    if d not in (2, 3):
        raise ValueError("ParticleSystem: dim must be 2 or 3")
    if src.size == 0 or src.size % d:
        raise ValueError("ParticleSystem: bad source array length")
    if tgt.size % d:
        raise ValueError("ParticleSystem: bad target array length")
    if stw.size != (src.size // d) * strength_components(kernel, d):
        raise ValueError("ParticleSystem: bad strength array length")


class Context:
    """One GPU context (device, stream, buffers, table cache)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _raise(lib().sdmk_create(int(device), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().sdmk_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- full evaluation -------------------------------------------------
    def evaluate_with_plan(self, plan: DmkPlan, sys: ParticleSystem, mode=FREE_SPACE,
                           report: Optional[dict] = None) -> np.ndarray:
        src, tgt, stw = _arr(sys.sources), _arr(sys.targets), _arr(sys.strengths)
        d = int(sys.dim)
        if plan.dim != d:
            raise ValueError("evaluate: plan and system dimensions differ")
        _check_lengths(plan.kernel, d, src, tgt, stw)
        ns = src.size // d
        nt = tgt.size // d
        u = np.empty((nt if nt else ns) * d)
        rep = sdmk_report()
        cp = plan.to_c()
        _raise(lib().sdmk_evaluate_with_plan(self._h, C.byref(cp), d, ns, _dptr(src), nt,
                                             _dptr(tgt if nt else None), _dptr(stw), _enum(mode, MODES),
                                             _dptr(u), C.byref(rep)))
        if report is not None:
            report.update(rep.as_dict())
        return u

    def evaluate(self, kernel, sys: ParticleSystem, eps: float, window=PROLATE, mode=FREE_SPACE,
                 report: Optional[dict] = None) -> np.ndarray:
        plan = select_parameters(kernel, eps, window, sys.dim)
        return self.evaluate_with_plan(plan, sys, mode, report)

    def evaluate_device(self, plan: DmkPlan, dim: int, ns: int, d_src: int, nt: int, d_tgt: int, d_str: int,
                        mode, d_u: int, report: Optional[dict] = None):
        """Device-resident variant: integer device addresses (e.g. torch tensor.data_ptr())."""
        rep = sdmk_report()
        cp = plan.to_c()
        _raise(lib().sdmk_evaluate_device(self._h, C.byref(cp), int(dim), int(ns), C.c_void_p(d_src), int(nt),
                                          C.c_void_p(d_tgt if nt else None), C.c_void_p(d_str),
                                          _enum(mode, MODES), C.c_void_p(d_u), C.byref(rep)))
        if report is not None:
            report.update(rep.as_dict())

    # ---- pass-level API (dmk.hpp:84-131, tree.hpp:90-104) -----------------
    def setup(self, plan: DmkPlan, sys: ParticleSystem, mode=FREE_SPACE):
        src, tgt, stw = _arr(sys.sources), _arr(sys.targets), _arr(sys.strengths)
        d = int(sys.dim)
        if plan.dim != d:
            raise ValueError("evaluate: plan and system dimensions differ")
        _check_lengths(plan.kernel, d, src, tgt, stw)
        cp = plan.to_c()
        _raise(lib().sdmk_setup(self._h, C.byref(cp), d, src.size // d, _dptr(src), tgt.size // d,
                                _dptr(tgt if tgt.size else None), _dptr(stw), _enum(mode, MODES)))
        self._plan = plan
        self._dim = d

    def tree_info(self) -> dict:
        info = np.zeros(7, np.int32)
        _raise(lib().sdmk_tree_info(self._h, _iptr(info)))
        keys = ["num_boxes", "max_level", "n_src", "n_tgt", "alias", "depth_capped", "channels"]
        return dict(zip(keys, info.tolist()))

    def tree_boxes(self) -> np.ndarray:
        nb = self.tree_info()["num_boxes"]
        out = np.zeros(nb * 11, np.int32)
        _raise(lib().sdmk_tree_boxes(self._h, _iptr(out)))
        return out.reshape(nb, 11)

    def tree_perm(self):
        info = self.tree_info()
        sp = np.zeros(info["n_src"], np.int32)
        tp = np.zeros(info["n_tgt"], np.int32) if not info["alias"] else None
        _raise(lib().sdmk_tree_perm(self._h, _iptr(sp), _iptr(tp)))
        return sp, tp

    def tree_dump(self) -> str:
        n = lib().sdmk_tree_dump(self._h, None, 0)
        if n < 0:
            _raise(1)
        buf = C.create_string_buffer(int(n))
        lib().sdmk_tree_dump(self._h, buf, n)
        return buf.raw[:n].decode()

    def _nodes(self):
        p, d = self._plan.p, self._dim
        return p ** d

    def upward_pass(self) -> np.ndarray:
        info = self.tree_info()
        out = np.empty(info["num_boxes"] * info["channels"] * self._nodes())
        _raise(lib().sdmk_upward_pass(self._h, _dptr(out)))
        return out

    def incoming(self, stage: int = 1) -> np.ndarray:
        info = self.tree_info()
        out = np.empty(info["num_boxes"] * self._dim * self._nodes())
        _raise(lib().sdmk_incoming(self._h, int(stage), _dptr(out)))
        return out

    def target_far_fields(self) -> np.ndarray:
        out = np.empty(self.tree_info()["n_tgt"] * self._dim)
        _raise(lib().sdmk_target_far_fields(self._h, _dptr(out)))
        return out

    def residual_pass(self) -> np.ndarray:
        out = np.empty(self.tree_info()["n_tgt"] * self._dim)
        _raise(lib().sdmk_residual_pass(self._h, _dptr(out)))
        return out

    # ---- O(N*M) reference sums on the GPU (oracle.hpp:60-75) ---------------
    def direct_sum(self, kernel, sys: ParticleSystem) -> np.ndarray:
        """stokesdmk::direct_sum (oracle.cpp:143-179): exact kernels, Kahan per target."""
        src, tgt, stw = _arr(sys.sources), _arr(sys.targets), _arr(sys.strengths)
        d = int(sys.dim)
        _check_lengths(_enum(kernel, KERNELS), d, src, tgt, stw)
        ns, nt = src.size // d, tgt.size // d
        u = np.empty((nt if nt else ns) * d)
        _raise(lib().sdmk_direct_sum(self._h, _enum(kernel, KERNELS), d, ns, _dptr(src), nt,
                                     _dptr(tgt if nt else None), _dptr(stw), _dptr(u)))
        return u

    def direct_residual_sum(self, plan: DmkPlan, sys: ParticleSystem, cutoff: float,
                            periodic: bool = False) -> np.ndarray:
        """stokesdmk::direct_residual_sum (oracle.cpp:181-241) with the plan's split tables."""
        src, tgt, stw = _arr(sys.sources), _arr(sys.targets), _arr(sys.strengths)
        d = int(sys.dim)
        ns, nt = src.size // d, tgt.size // d
        u = np.empty((nt if nt else ns) * d)
        cp = plan.to_c()
        _raise(lib().sdmk_direct_residual_sum(self._h, C.byref(cp), d, ns, _dptr(src), nt,
                                              _dptr(tgt if nt else None), _dptr(stw), float(cutoff),
                                              1 if periodic else 0, _dptr(u)))
        return u

    def ewald(self, plan: DmkPlan, sys: ParticleSystem, level: int = -1, info: Optional[dict] = None) -> np.ndarray:
        """FFT Ewald for the periodic 3D Stokeslet (include/sdmk.h sdmk_ewald)."""
        src, tgt, stw = _arr(sys.sources), _arr(sys.targets), _arr(sys.strengths)
        if plan.dim != 3 or int(sys.dim) != 3:
            raise ValueError("ewald: the FFT Ewald path covers the 3D Stokeslet")
        _check_lengths(plan.kernel, 3, src, tgt, stw)
        ns, nt = src.size // 3, tgt.size // 3
        u = np.empty((nt if nt else ns) * 3)
        out = np.zeros(8)
        cp = plan.to_c()
        _raise(lib().sdmk_ewald(self._h, C.byref(cp), ns, _dptr(src), nt, _dptr(tgt if nt else None), _dptr(stw),
                                _dptr(u), int(level), _dptr(out)))
        if info is not None:
            info.update(dict(zip(["level", "grid", "width", "kappa_max", "t_sort_ms", "t_local_ms", "t_far_ms",
                                  "t_total_ms"], out.tolist())))
        return u

    def set_shard(self, rank: int, nranks: int):
        """Own a contiguous Morton run of target leaves (see include/sdmk.h)."""
        _raise(lib().sdmk_set_shard(self._h, int(rank), int(nranks)))

    def comm_init(self, rank: int, nranks: int, uid: bytes):
        """Attach an NCCL communicator (uid from comm_unique_id() on rank 0):
        evaluations exchange outgoing-expansion halos and return the full u
        on every rank (include/sdmk.h)."""
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        _raise(lib().sdmk_comm_init(self._h, int(rank), int(nranks), bytes(uid)))

    def set_manual_exchange(self, on: bool = True):
        """Two-phase evaluation without NCCL (tests, per-rank timing on one GPU)."""
        _raise(lib().sdmk_set_manual_exchange(self._h, 1 if on else 0))

    def evaluate_begin(self, plan: DmkPlan, sys: ParticleSystem, mode=FREE_SPACE):
        """First half of a manual-exchange evaluation (host arrays; they are
        copied before this returns)."""
        src, tgt, stw = _arr(sys.sources), _arr(sys.targets), _arr(sys.strengths)
        d = int(sys.dim)
        ns, nt = src.size // d, tgt.size // d
        self._pending = (d, ns, nt)
        cp = plan.to_c()
        _raise(lib().sdmk_evaluate_begin(self._h, C.byref(cp), d, ns, src.ctypes.data, nt,
                                         tgt.ctypes.data if nt else None, stw.ctypes.data, _enum(mode, MODES), 0))

    def evaluate_begin_device(self, plan: DmkPlan, dim: int, ns: int, d_src: int, nt: int, d_tgt: int,
                              d_str: int, mode=FREE_SPACE):
        """evaluate_begin with device addresses; finish with evaluate_end(d_u=...)."""
        self._pending = (int(dim), int(ns), int(nt))
        cp = plan.to_c()
        _raise(lib().sdmk_evaluate_begin(self._h, C.byref(cp), int(dim), int(ns), C.c_void_p(d_src), int(nt),
                                         C.c_void_p(d_tgt if nt else None), C.c_void_p(d_str), _enum(mode, MODES),
                                         1))

    def evaluate_end(self, report: Optional[dict] = None, d_u: Optional[int] = None):
        """Second half: returns u (host) or writes it to the device address d_u
        when the evaluation began with device pointers."""
        d, ns, nt = self._pending
        rep = sdmk_report()
        if d_u is not None:
            _raise(lib().sdmk_evaluate_end(self._h, C.c_void_p(d_u), C.byref(rep)))
            u = None
        else:
            u = np.empty((nt if nt else ns) * d)
            _raise(lib().sdmk_evaluate_end(self._h, u.ctypes.data, C.byref(rep)))
        if report is not None:
            report.update(rep.as_dict())
        return u

    def halo_transfer_to(self, other: "Context"):
        """Copy this rank's halo slab for `other` into other's receive slab."""
        _raise(lib().sdmk_halo_transfer(self._h, other._h))

    def stream_handle(self) -> int:
        """cudaStream_t of this context (for CUDA-event timing by the caller)."""
        s = C.c_void_p()
        _raise(lib().sdmk_get_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def fp64_peak_tflops(self) -> float:
        v = C.c_double()
        _raise(lib().sdmk_fp64_peak(self._h, C.byref(v)))
        return float(v.value)

    def set_guard(self, on: bool = True):
        """Guard mode (canaries around every device buffer, poisoned contents);
        call before the context's first setup or evaluation."""
        _raise(lib().sdmk_set_guard(self._h, 1 if on else 0))

    def guard_check(self) -> list:
        """Names of device buffers whose canaries were overwritten."""
        buf = C.create_string_buffer(1 << 16)
        n = lib().sdmk_guard_check(self._h, buf, len(buf))
        if n < 0:
            _raise(-1 if n == -1 else int(n))
        return [s for s in buf.value.decode().split("\n") if s]

    def guard_selftest(self) -> bool:
        """Store one byte past each end of a scratch buffer; True when the
        canary check caught both."""
        r = lib().sdmk_guard_selftest(self._h)
        if r < 0:
            _raise(r)
        return r == 1

    def fp64_mma_peak_tflops(self) -> float:
        v = C.c_double()
        _raise(lib().sdmk_fp64_mma_peak(self._h, C.byref(v)))
        return float(v.value)

    def save_tables(self, plan: DmkPlan, path: str):
        cp = plan.to_c()
        _raise(lib().sdmk_save_tables(self._h, C.byref(cp), path.encode()))

    def load_tables(self, path: str):
        _raise(lib().sdmk_load_tables(self._h, path.encode()))


_default_ctx: Optional[Context] = None


def comm_unique_id() -> bytes:
    """NCCL unique id for Context.comm_init (call on rank 0, share the bytes)."""
    buf = C.create_string_buffer(128)
    _raise(lib().sdmk_comm_unique_id(buf))
    return buf.raw


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def evaluate_with_plan(plan: DmkPlan, sys: ParticleSystem, mode=FREE_SPACE, report=None) -> np.ndarray:
    return default_context().evaluate_with_plan(plan, sys, mode, report)


def evaluate(kernel, sys: ParticleSystem, eps: float, window=PROLATE, mode=FREE_SPACE, report=None) -> np.ndarray:
    return default_context().evaluate(kernel, sys, eps, window, mode, report)


def direct_sum(kernel, sys: ParticleSystem) -> np.ndarray:
    return default_context().direct_sum(kernel, sys)


def direct_residual_sum(plan: DmkPlan, sys: ParticleSystem, cutoff: float, periodic: bool = False) -> np.ndarray:
    return default_context().direct_residual_sum(plan, sys, cutoff, periodic)


# ---- host-only helpers (CPU tests of the setup / topology code) ----------
def host_save_tables(plan: DmkPlan, path: str):
    cp = plan.to_c()
    _raise(lib().sdmk_host_save_tables(C.byref(cp), path.encode()))


def host_symbol_table(plan: DmkPlan, h: float, s2max: int, kind: int, r_coarse: float, r_fine: float):
    out = np.empty(s2max + 1)
    cp = plan.to_c()
    _raise(lib().sdmk_host_symbol_table(C.byref(cp), h, s2max, kind, r_coarse, r_fine, _dptr(out)))
    return out


def host_topology_dump(dim, periodic, n_s, p, q_src_sorted, q_tgt_sorted=None) -> str:
    qs = np.ascontiguousarray(np.asarray(q_src_sorted, np.int32).T.ravel())  # (n, d) -> SoA
    ns = np.asarray(q_src_sorted).shape[0]
    if q_tgt_sorted is not None and np.asarray(q_tgt_sorted).size:
        qt = np.ascontiguousarray(np.asarray(q_tgt_sorted, np.int32).T.ravel())
        nt = np.asarray(q_tgt_sorted).shape[0]
    else:
        qt, nt = None, 0
    n = lib().sdmk_host_topology_dump(dim, int(periodic), n_s, p, ns, _iptr(qs), nt, _iptr(qt), None, 0)
    if n < 0:
        _raise(1)
    buf = C.create_string_buffer(int(n))
    lib().sdmk_host_topology_dump(dim, int(periodic), n_s, p, ns, _iptr(qs), nt, _iptr(qt), buf, n)
    return buf.raw[:n].decode()


def host_shard_plan(dim, periodic, n_s, p, q_src_sorted, rank, nranks, q_tgt_sorted=None) -> dict:
    """The shard plan sdmk_set_shard applies (host topology, no GPU)."""
    qs = np.ascontiguousarray(np.asarray(q_src_sorted, np.int32).T.ravel())
    ns = np.asarray(q_src_sorted).shape[0]
    if q_tgt_sorted is not None and np.asarray(q_tgt_sorted).size:
        qt = np.ascontiguousarray(np.asarray(q_tgt_sorted, np.int32).T.ravel())
        nt = np.asarray(q_tgt_sorted).shape[0]
    else:
        qt, nt = None, 0
    out = (C.c_int64 * 5)()
    _raise(lib().sdmk_host_shard_plan(dim, int(periodic), n_s, p, ns, _iptr(qs), nt, _iptr(qt), int(rank),
                                      int(nranks), out))
    return {"t0": out[0], "t1": out[1], "owned_leaves": out[2], "needed_boxes": out[3], "target_leaves": out[4]}


def host_halo_plan(dim, periodic, n_s, p, q_src_sorted, nranks, q_tgt_sorted=None) -> dict:
    """The exchange plan of comm_init evaluations (host topology, no GPU):
    recv[f, r] = boxes rank r receives from rank f, owned leaves per rank,
    boxes above the cut, cut boxes."""
    qs = np.ascontiguousarray(np.asarray(q_src_sorted, np.int32).T.ravel())
    ns = np.asarray(q_src_sorted).shape[0]
    if q_tgt_sorted is not None and np.asarray(q_tgt_sorted).size:
        qt = np.ascontiguousarray(np.asarray(q_tgt_sorted, np.int32).T.ravel())
        nt = np.asarray(q_tgt_sorted).shape[0]
    else:
        qt, nt = None, 0
    R = int(nranks)
    out = (C.c_int64 * (R * R + R + 2))()
    _raise(lib().sdmk_host_halo_plan(dim, int(periodic), n_s, p, ns, _iptr(qs), nt, _iptr(qt), R, out))
    a = np.array(out[:], dtype=np.int64)
    return {"recv": a[:R * R].reshape(R, R), "owned_leaves": a[R * R:R * R + R], "above_cut": int(a[R * R + R]),
            "cut_boxes": int(a[R * R + R + 1])}


def host_build_tables(kernel, dim: int, window, c: float, sigma: float, tol: float) -> bytes:
    """build_split_kernel (split.cpp:319-396) on the host: the SDMKSPLT v1 image."""
    k, w = _enum(kernel, KERNELS), _enum(window, WINDOWS)
    n = lib().sdmk_host_build_tables(k, int(dim), w, float(c), float(sigma), float(tol), None, 0)
    if n < 0:
        _raise(1)
    buf = C.create_string_buffer(int(n))
    lib().sdmk_host_build_tables(k, int(dim), w, float(c), float(sigma), float(tol), buf, n)
    return buf.raw[:n]


def host_build_window(window, c: float = 0.0, sigma: float = 0.0) -> dict:
    """build_prolate / build_gaussian (windows.cpp): scalars and Legendre coefficients."""
    sc = np.zeros(5)
    w = _enum(window, WINDOWS)
    n = lib().sdmk_host_build_window(w, float(c), float(sigma), _dptr(sc), None, 0)
    if n < 0:
        _raise(1)
    co = np.zeros(max(n, 1))
    lib().sdmk_host_build_window(w, float(c), float(sigma), _dptr(sc), _dptr(co), n)
    return {"lambda0": sc[0], "norm_r": sc[1], "trunc_error": sc[2], "psi0": sc[3], "chi0": sc[4],
            "legendre_coeffs": co[:n]}


def host_shard_bounds(dim, periodic, n_s, p, q_src_sorted, nranks, q_tgt_sorted=None) -> np.ndarray:
    """Every rank's owned range of sorted targets (nranks + 1 bounds; host topology, no GPU)."""
    qs = np.ascontiguousarray(np.asarray(q_src_sorted, np.int32).T.ravel())
    ns = np.asarray(q_src_sorted).shape[0]
    if q_tgt_sorted is not None and np.asarray(q_tgt_sorted).size:
        qt = np.ascontiguousarray(np.asarray(q_tgt_sorted, np.int32).T.ravel())
        nt = np.asarray(q_tgt_sorted).shape[0]
    else:
        qt, nt = None, 0
    out = (C.c_int64 * (int(nranks) + 1))()
    _raise(lib().sdmk_host_shard_bounds(dim, int(periodic), n_s, p, ns, _iptr(qs), nt, _iptr(qt), int(nranks), out))
    return np.array(out[:], dtype=np.int64)

