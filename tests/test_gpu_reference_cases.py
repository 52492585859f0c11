"""The reference's own pass-level known-answer tests, restated against the
GPU path through the C-ABI:

  outgoing proxies reproduce a point placed at a proxy node   test_dmk.cpp:169-212 (<= 1e-10)
  upward merges conserve per-channel totals on ancestors       test_dmk.cpp:214-265 (<= 1e-11)
  single-leaf residual pass == residual-only direct sum        test_dmk.cpp:344-372 (<= 1e-12)
  periodic evaluation vs the slow Fourier (Ewald) reference    test_dmk.cpp:512-575 (<= 2e-6 .. 4e-6)

Systems are seeded uniform points (the reference's mixed_system helper is a
test fixture, not part of the path); the checkers are the compiled reference
(oracle/_ref) where a reference quantity is needed.
"""
import numpy as np
import pytest

import paper_2509_21471_b200 as g

pytestmark = pytest.mark.gpu


def _ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not present")
    return ref


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _system(kernel, dim, ns, nt, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5, 0.5, (ns, dim))
    sc = g.strength_components(kernel, dim)
    s = rng.standard_normal((ns, sc))
    if kernel == 1:
        nn = rng.standard_normal((ns, dim))
        s[:, dim:] = nn / np.linalg.norm(nn, axis=1, keepdims=True)
    t = rng.uniform(-0.5, 0.5, (nt, dim)) if nt else np.zeros(0)
    return x, s, t


def _cheb_nodes(p):
    i = np.arange(p)
    return np.cos((2 * i + 1) * np.pi / (2 * p))


@pytest.mark.parametrize("dim", [2, 3])
def test_proxy_node_source_reproduced(dim):
    ctx = g.Context(0)
    plan = g.select_parameters(0, 1e-6, g.PROLATE, dim)
    plan.n_s = 64
    p = plan.p
    rng = np.random.default_rng(7)
    dummies = rng.uniform(-0.5, 0.5, (2, dim))
    # the root box is [-1/2, 1/2]^d: node coordinate 0.5 * cos((2i + 1) pi / 2p), axis 0 fastest
    pick = (5, 2, 4) if dim == 3 else (3, 6)
    node = np.array([0.5 * _cheb_nodes(p)[k] for k in pick])
    strength = np.zeros(dim)
    strength[0], strength[dim - 1] = 0.7, -0.3
    x = np.vstack([node, dummies])
    s = np.vstack([strength, rng.standard_normal((2, dim))])
    ctx.setup(plan, g.ParticleSystem(dim, x, np.zeros(0), s))
    assert ctx.tree_info()["num_boxes"] == 1
    w = ctx.upward_pass()
    ctx.setup(plan, g.ParticleSystem(dim, dummies, np.zeros(0), s[1:]))
    w2 = ctx.upward_pass()
    nodes = p ** dim
    idx = pick[0] + p * (pick[1] + (p * pick[2] if dim == 3 else 0))
    want = np.zeros(dim * nodes)
    for ch in range(dim):
        want[ch * nodes + idx] = strength[ch]
    assert np.max(np.abs((w - w2)[: dim * nodes] - want)) < 1e-10


def _channels(kernel, dim, s):
    if kernel != 1:
        return s
    f, n = s[:, :dim], s[:, dim:]
    w = np.sum(f * n, axis=1)
    if dim == 3:
        return np.stack([2 * f[:, 0] * n[:, 0] + w, 2 * f[:, 1] * n[:, 1] + w, 2 * f[:, 2] * n[:, 2] + w,
                         f[:, 0] * n[:, 1] + f[:, 1] * n[:, 0], f[:, 0] * n[:, 2] + f[:, 2] * n[:, 0],
                         f[:, 1] * n[:, 2] + f[:, 2] * n[:, 1]], axis=1)
    return np.stack([2 * f[:, 0] * n[:, 0] + w, 2 * f[:, 1] * n[:, 1] + w, f[:, 0] * n[:, 1] + f[:, 1] * n[:, 0]],
                    axis=1)


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("dim", [2, 3])
def test_upward_merges_conserve_channel_totals(kernel, dim):
    ctx = g.Context(0)
    plan = g.select_parameters(kernel, 1e-3, g.PROLATE, dim)
    plan.n_s = 16
    x, s, _ = _system(kernel, dim, 300, 0, 11)
    ctx.setup(plan, g.ParticleSystem(dim, x, np.zeros(0), s))
    info = ctx.tree_info()
    assert info["max_level"] >= 2
    boxes = ctx.tree_boxes()
    sperm, _ = ctx.tree_perm()
    w = ctx.upward_pass()
    nch = g.outgoing_channels(kernel, dim)
    nodes = plan.p ** dim
    chv = _channels(kernel, dim, s)
    for b in (0, boxes[0, 2]):
        sb, se = boxes[b, 7], boxes[b, 8]
        want = chv[sperm[sb:se]].sum(axis=0)
        got = w[b * nch * nodes:(b + 1) * nch * nodes].reshape(nch, nodes).sum(axis=1)
        np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-11 * np.abs(want).max())


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("dim", [2, 3])
def test_single_leaf_residual_equals_direct_residual(kernel, dim):
    ref = _ref()
    ctx = g.Context(0)
    plan = g.select_parameters(kernel, 1e-6, g.PROLATE, dim)
    plan.n_s = 1000
    x, s, _ = _system(kernel, dim, 150, 0, 41)
    sysm = g.ParticleSystem(dim, x, np.zeros(0), s)
    ctx.setup(plan, sysm)
    assert ctx.tree_info()["max_level"] == 0
    got = ctx.residual_pass()
    R = ref.RefProblem(plan.__dict__, dim, x, s)
    want = R.direct_residual_sum(1.0)
    selfc = R.self_scaled(1.0)  # the leaf self coefficient belongs to the same scale
    if selfc != 0.0:
        got = got - selfc * s[:, :dim].ravel()
    assert _rel_l2(got, want) <= 1e-12


@pytest.mark.parametrize("dim,kernel,bound,n_s,ns,nt", [
    (3, 0, 2e-6, 40, 220, 60), (3, 1, 3e-6, 40, 220, 60), (3, 2, 2e-6, 40, 220, 60),
    (2, 0, 2e-6, 30, 180, 50), (2, 2, 4e-6, 30, 180, 50)])
def test_periodic_matches_slow_fourier_reference(dim, kernel, bound, n_s, ns, nt):
    ref = _ref()
    ctx = g.Context(0)
    plan = g.select_parameters(kernel, 1e-6, g.PROLATE, dim)
    plan.n_s = n_s
    x, s, t = _system(kernel, dim, ns, nt, 401 + kernel + 100 * dim)
    if kernel != 1:  # zero net force / torque, as the periodic sums require
        s = s - s.mean(axis=0)
    u = ctx.evaluate_with_plan(plan, g.ParticleSystem(dim, x, t, s), g.PERIODIC)
    R = ref.RefProblem(plan.__dict__, dim, x, s, targets=t, periodic=True)
    want = R.ewald_reference(True)
    # the reference's bounds were set on its own fixture; on this system the
    # reference DMK's own error is the yardstick where it is larger
    ref_err = _rel_l2(R.evaluate()[0], want)
    assert _rel_l2(u, want) <= max(bound, 1.001 * ref_err)


def _direct(kernel, dim, x, s, t=None):
    ref = _ref()
    plan = ref.select_parameters(kernel, 1e-6, 0, dim)
    return ref.RefProblem(plan, dim, x, s, targets=t).direct_sum()


def _yardstick(plan, dim, x, s, t, bound, exact):
    """max(bound, the reference DMK's own error on this system): the
    reference's bounds were set on its own fixture (mixed_system)."""
    ref = _ref()
    ur, _ = ref.RefProblem(plan.__dict__, dim, x, s, targets=t).evaluate()
    return max(bound, 1.001 * _rel_l2(ur, exact))


@pytest.mark.parametrize("sep", [0.4, 0.26, 0.13, 0.06, 0.031, 0.015, 0.008, 0.004, 0.0019, 0.0009])
def test_deep_trees_all_separation_classes(sep):  # test_dmk.cpp:393-413
    ctx = g.Context(0)
    plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    plan.n_s = 1
    x = np.array([[-0.271, 0.113, -0.041], [-0.271 + sep, 0.113 + 0.3 * sep, -0.041 - 0.2 * sep]])
    s = np.array([[0.8, -0.45, 0.3], [-0.6, 0.95, 0.21]])
    u = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, np.zeros(0), s))
    assert _rel_l2(u, _direct(0, 3, x, s)) <= 5e-6


@pytest.mark.parametrize("kernel,eps,bound", [(0, 1e-3, 1e-3), (0, 1e-6, 1e-6), (1, 1e-3, 1e-3), (1, 1e-6, 1e-6),
                                              (2, 1e-3, 2e-3), (2, 1e-6, 2e-6)])
def test_adaptive_accuracy_3d(kernel, eps, bound):  # test_dmk.cpp:415-458
    ctx = g.Context(0)
    plan = g.select_parameters(kernel, eps, g.PROLATE, 3)
    plan.n_s = 75
    x, s, t = _system(kernel, 3, 600, 150, 101 + kernel)
    rep = {}
    u = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, t, s), g.FREE_SPACE, rep)
    exact = _direct(kernel, 3, x, s, t)
    assert rep["max_level"] >= 2
    assert _rel_l2(u, exact) <= _yardstick(plan, 3, x, s, t, bound, exact)


@pytest.mark.parametrize("eps", [1e-9, 1e-12])
def test_tight_tolerances_shallow_tree(eps):
    ctx = g.Context(0)
    plan = g.select_parameters(0, eps, g.PROLATE, 3)
    plan.n_s = 150
    x, s, _ = _system(0, 3, 400, 0, 7)
    u = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, np.zeros(0), s))
    exact = _direct(0, 3, x, s)
    bound = 5e-12 if eps == 1e-12 else eps
    assert _rel_l2(u, exact) <= _yardstick(plan, 3, x, s, np.zeros(0), bound, exact)


@pytest.mark.parametrize("kernel,factor", [(0, 1.0), (1, 3.0), (2, 4.0)])
@pytest.mark.parametrize("eps", [1e-3, 1e-6])
def test_adaptive_accuracy_2d(kernel, factor, eps):  # test_dmk.cpp:460-492
    ctx = g.Context(0)
    plan = g.select_parameters(kernel, eps, g.PROLATE, 2)
    plan.n_s = 48
    x, s, t = _system(kernel, 2, 500, 120, 211 + kernel)
    u = ctx.evaluate_with_plan(plan, g.ParticleSystem(2, x, t, s))
    exact = _direct(kernel, 2, x, s, t)
    assert _rel_l2(u, exact) <= _yardstick(plan, 2, x, s, t, factor * eps, exact)


def test_gaussian_window_agrees_with_direct_and_prolate():  # test_dmk.cpp:494-510
    ctx = g.Context(0)
    gp = g.select_parameters(0, 1e-6, g.GAUSSIAN, 3)
    gp.n_s = 75
    x, s, t = _system(0, 3, 500, 100, 307)
    sysm = g.ParticleSystem(3, x, t, s)
    ug = ctx.evaluate_with_plan(gp, sysm)
    exact = _direct(0, 3, x, s, t)
    assert _rel_l2(ug, exact) <= _yardstick(gp, 3, x, s, t, 2e-6, exact)
    pp = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    pp.n_s = 75
    up = ctx.evaluate_with_plan(pp, sysm)
    assert _rel_l2(up, ug) <= 3e-6


def test_leaf_capacity_does_not_change_the_answer():  # test_dmk.cpp:625-634
    ctx = g.Context(0)
    plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    x, s, _ = _system(0, 3, 300, 0, 601)
    exact = _direct(0, 3, x, s)
    for n_s in (60, 200):
        plan.n_s = n_s
        u = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, np.zeros(0), s))
        assert _rel_l2(u, exact) <= 1e-6


def test_report_and_convenience_wrapper():  # test_dmk.cpp:645-666
    ctx = g.Context(0)
    x, s, t = _system(2, 3, 250, 80, 701)
    rep = {}
    u = ctx.evaluate(g.ROTLET, g.ParticleSystem(3, x, t, s), 1e-3, g.PROLATE, g.FREE_SPACE, rep)
    assert u.size == 80 * 3
    assert rep["num_sources"] == 250 and rep["num_targets"] == 80 and rep["num_boxes"] >= 1
    assert g.select_parameters(g.ROTLET, 1e-3, g.PROLATE, 3).p == 8
    assert rep["t_tree"] >= 0.0 and rep["t_residual"] >= 0.0
    assert _rel_l2(u, _direct(2, 3, x, s, t)) <= 1e-3
    uz = ctx.evaluate(g.ROTLET, g.ParticleSystem(3, x, t, np.zeros_like(s)), 1e-3, g.PROLATE, g.FREE_SPACE)
    assert np.all(uz == 0.0)
