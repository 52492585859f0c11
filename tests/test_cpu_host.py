"""CPU checks of the product's host side and its C-ABI (no GPU needed).

* libsdmk_b200.so loads and exports every entry point declared in include/sdmk.h
* plan selection, split tables (byte-identical SDMKSPLT files), symbol tables
  and the bit-exact box topology agree with the golden vectors of the reference
"""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_case, golden_index
from oracle import restate as R

import paper_2509_21471_b200 as g


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "sdmk.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(sdmk_[a-z0-9_]+)\(", txt, re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    assert os.path.exists(g.LIB_PATH), "run __graft_entry__.build() / make -C paper_2509_21471_b200/csrc"
    out = subprocess.run(["nm", "-D", "--defined-only", g.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sdmk_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    g.lib()  # ctypes binding resolves every symbol it declares


def test_cxx_dropin_header_compiles():
    """include/stokesdmk_b200/dmk.hpp compiles against the reference-style call sites."""
    src = os.path.join(ROOT, "tests", "dropin_example.cpp")
    out = "/tmp/_sdmk_dropin"
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    del out


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("eps", [1e-3, 3e-5, 1e-6, 1e-8, 1e-9, 1e-12])
@pytest.mark.parametrize("window", [0, 1])
def test_select_parameters_matches_restatement(kernel, dim, eps, window):
    a = g.select_parameters(kernel, eps, window, dim).__dict__
    b = R.select_parameters(kernel, eps, window, dim)
    assert a == b


def test_select_parameters_errors_map_to_value_error():
    for bad in [(0, 0.5, 0, 3), (0, 1e-14, 0, 3), (0, 1e-6, 0, 4), (3, 1e-6, 0, 3)]:
        with pytest.raises(ValueError):
            g.select_parameters(*bad)
    assert g.outgoing_channels(1, 3) == 6 and g.outgoing_channels(2, 2) == 1
    assert g.strength_components(1, 2) == 4


@pytest.mark.parametrize("name", [c["name"] for c in golden_index()])
def test_tables_byte_identical_to_reference(name, tmp_path):
    meta = next(c for c in golden_index() if c["name"] == name)
    path = str(tmp_path / "t.bin")
    g.host_save_tables(g.DmkPlan(**meta["plan"]), path)
    ours = open(path, "rb").read()
    ref = open(os.path.join(GOLDEN, f"{name}.tables.bin"), "rb").read()
    if ours != ref:  # 2D tables come from quadrature + libm Bessel: allow last-ulp drift
        A, B = R.load_tables(path), R.load_tables(os.path.join(GOLDEN, f"{name}.tables.bin"))
        for k in ("s_diag", "s_offd", "t_diag", "t_offd", "w_offd"):
            assert len(A[k][2]) == len(B[k][2])
            assert np.allclose(A[k][2], B[k][2], rtol=0, atol=1e-14)
        assert abs(A["self_const"] - B["self_const"]) <= 1e-14
        assert meta["dim"] == 2, "3D tables must be byte-identical"


@pytest.mark.parametrize("name", ["stokeslet3d_uniform", "stresslet3d_periodic", "rotlet2d", "stokeslet3d_gaussian"])
def test_symbol_tables_match_restatement(name):
    meta = next(c for c in golden_index() if c["name"] == name)
    plan = meta["plan"]
    tabs = R.load_tables(os.path.join(GOLDEN, f"{name}.tables.bin"))
    M = (plan["N1"] - 1) // 2
    for kind, h, rc, rf in [(0, np.pi / 3 / 0.25, 0.5, 0.25), (0, np.pi / 3 / 2 ** -6, 2 ** -5, 2 ** -6),
                            (1, np.pi / 3, 1.0, 1.0), (2, 2 * np.pi, 1.0, 1.0)]:
        ours = g.host_symbol_table(g.DmkPlan(**plan), h, 3 * M * M, kind, rc, rf)
        want = R.symbol_table(tabs, h, 3 * M * M, kind, rc, rf)
        scale = max(np.max(np.abs(want)), 1e-300)
        # the rotlet's Taylor branch uses a finite difference of phi_hat at h0 = 0.02
        # (dmk.cpp:270-273), which amplifies last-ulp differences of the Legendre
        # evaluation (numpy Clenshaw vs the reference's recurrence) by 1/h0^2
        tol = 1e-11 if meta["kernel"] == 2 else 1e-13
        assert np.max(np.abs(ours - want)) <= tol * scale


@pytest.mark.parametrize("name", [c["name"] for c in golden_index()])
def test_host_topology_bit_exact(name):
    meta, d, dump = golden_case(name)
    plan, dim, per = meta["plan"], meta["dim"], meta["periodic"]
    src = R.wrap_into_box(d["sources"]) if per else d["sources"]
    qs = R.quantize(src)
    sp = R.morton_order(qs)
    assert np.array_equal(sp, d["sperm"])
    qt = None
    if meta["ntgt"]:
        tgt = R.wrap_into_box(d["targets"]) if per else d["targets"]
        q = R.quantize(tgt)
        qt = q[R.morton_order(q)]
    assert g.host_topology_dump(dim, per, plan["n_s"], plan["p"], qs[sp], qt) == dump


def test_host_topology_degenerate_inputs():
    # one point; all points identical (depth cap); points exactly on +1/2 faces
    for pts in [np.zeros((1, 3)), np.full((5, 3), 0.125), np.array([[0.5, 0.5, 0.5], [-0.5, -0.5, -0.5],
                                                                     [0.5, -0.5, 0.0]])]:
        q = R.quantize(pts)
        sp = R.morton_order(q)
        T = R.build_tree(pts, None, 1, 3, False, 5)
        assert g.host_topology_dump(3, False, 1, 5, q[sp]) == R.dump_tree(T)


def test_cxx_dropin_pass_program_links():
    """tests/dropin_passes.cpp (the pass-level drop-in program the GPU tests run)
    compiles against the header and links with libsdmk_b200.so."""
    lib_dir = os.path.join(ROOT, "paper_2509_21471_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "dropin_passes.cpp"), "-o", "/tmp/_sdmk_dropin_link",
                        "-L" + lib_dir, "-lsdmk_b200", "-Wl,-rpath," + lib_dir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("kernel,dim,eps", [(0, 3, 1e-6), (1, 3, 1e-6), (2, 3, 1e-9), (0, 3, 1e-12)])
def test_host_build_tables_image_equals_reference_export(kernel, dim, eps, tmp_path):
    """build_split_kernel through the C-ABI (the drop-in's SplitKernel) is byte-identical
    to the reference's export_split_kernel of its own tables (3D)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    plan = ref.select_parameters(kernel, eps, 0, dim)
    x = np.random.default_rng(0).uniform(-0.5, 0.5, (50, dim))
    s = np.ones((50, g.strength_components(kernel, dim)))
    P = ref.RefProblem(plan, dim, x, s)
    path = str(tmp_path / "t.bin")
    P.export_tables(path)
    img = g.host_build_tables(kernel, dim, 0, plan["c"], 0.0, plan["table_tol"])
    assert open(path, "rb").read() == img
    # and a window other than the plan's (the SplitKernel override case)
    P.set_window(plan["c"] * 1.15)
    P.export_tables(path)
    assert open(path, "rb").read() == g.host_build_tables(kernel, dim, 0, plan["c"] * 1.15, 0.0, plan["table_tol"])


def test_host_build_window_matches_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    plan = ref.select_parameters(0, 1e-6, 0, 3)
    P = ref.RefProblem(plan, 3, np.zeros((1, 3)), np.ones((1, 3)))
    sc = np.zeros(8)
    co = np.zeros(256)
    n = ref.lib().ref_window(ref._dp(sc), ref._dp(co), 256)
    w = g.host_build_window(0, plan["c"])
    assert np.array_equal(w["legendre_coeffs"], co[:n])
    assert [w["lambda0"], w["norm_r"], w["trunc_error"], w["psi0"], w["chi0"]] == list(sc[3:8])
    del P
