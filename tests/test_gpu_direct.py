"""GPU reference sums against the compiled reference.

  sdmk_direct_sum           == stokesdmk::direct_sum           (oracle.cpp:143-179)
  sdmk_direct_residual_sum  == stokesdmk::direct_residual_sum  (oracle.cpp:181-241)

Same per-target order, Kahan accumulation and unfused arithmetic as the
reference, so the 3D results (and every kernel without a log) are compared
bit for bit; the 2D Stokeslet's log(r^2) / log(s) comes from CUDA's libdevice
(<= 1 ulp from glibc), so it is held to 1e-14 of the largest component.
Then the GPU direct sum serves as ground truth for the GPU DMK at sizes the
CPU reference cannot reach quickly (the reference's acceptance.cpp:451-474
accuracy check, at N = 1e5 instead of 5e3).
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


def _system(kernel, dim, ns, nt, seed, box=0.5):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-box, box, (ns, dim))
    sc = g.strength_components(kernel, dim)
    s = rng.standard_normal((ns, sc))
    if kernel == 1:
        nn = rng.standard_normal((ns, dim))
        s[:, dim:] = nn / np.linalg.norm(nn, axis=1, keepdims=True)
    t = rng.uniform(-box, box, (nt, dim)) if nt else np.zeros(0)
    return x, s, t


def _same(got, want, kernel, dim):
    if kernel == 0 and dim == 2:  # log from libdevice
        scale = float(np.max(np.abs(want)))
        assert float(np.max(np.abs(got - want))) <= 1e-14 * scale
    else:
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (bad.size, got[bad[:4]], want[bad[:4]])


CASES = [(k, d) for d in (3, 2) for k in (0, 1, 2)]


@pytest.mark.parametrize("kernel,dim", CASES)
@pytest.mark.parametrize("nt", [0, 700])
def test_direct_sum_matches_reference(kernel, dim, nt):
    ref = _ref()
    x, s, t = _system(kernel, dim, 1500, nt, 11 + kernel + 10 * dim + nt)
    got = g.Context(0).direct_sum(kernel, g.ParticleSystem(dim, x, t, s))
    plan = g.select_parameters(kernel, 1e-6, g.PROLATE, dim)
    want = ref.RefProblem(plan.__dict__, dim, x, s, targets=t if nt else None).direct_sum()
    _same(got, want, kernel, dim)


@pytest.mark.parametrize("kernel,dim", CASES)
@pytest.mark.parametrize("periodic,cutoff", [(False, 0.15), (True, 0.4)])
def test_direct_residual_sum_matches_reference(kernel, dim, periodic, cutoff):
    ref = _ref()
    box = 0.7 if periodic else 0.5  # periodic inputs outside the box are wrapped first
    x, s, t = _system(kernel, dim, 1200, 500, 71 + kernel + 10 * dim, box)
    plan = g.select_parameters(kernel, 1e-6, g.PROLATE, dim)
    got = g.Context(0).direct_residual_sum(plan, g.ParticleSystem(dim, x, t, s), cutoff, periodic)
    want = ref.RefProblem(plan.__dict__, dim, x, s, targets=t, periodic=periodic).direct_residual_sum(cutoff)
    _same(got, want, kernel, dim)


def test_direct_sum_alias_and_errors():
    ctx = g.Context(0)
    x = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.3], [-0.2, 0.0, 0.4]])
    s = np.ones((3, 3))
    with pytest.raises(g.DomainError, match="direct_sum: coincident points"):
        ctx.direct_sum(0, g.ParticleSystem(3, x, np.zeros(0), s))
    with pytest.raises(ValueError, match="outside the unit box"):
        ctx.direct_sum(0, g.ParticleSystem(3, x * 3.0, np.zeros(0), s))
    with pytest.raises(ValueError, match="non-finite strength"):
        ctx.direct_sum(0, g.ParticleSystem(3, x[1:], np.zeros(0), np.array([[1.0, np.nan, 0.0], [0, 0, 1.0]])))
    plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    ok = g.ParticleSystem(3, x[1:], np.zeros(0), s[1:])
    with pytest.raises(ValueError, match="cutoff must be positive"):
        ctx.direct_residual_sum(plan, ok, 0.0)
    with pytest.raises(ValueError, match="cutoff <= 1"):
        ctx.direct_residual_sum(plan, ok, 1.5, True)
    with pytest.raises(ValueError, match="dimension mismatch"):
        ctx.direct_residual_sum(g.select_parameters(0, 1e-6, g.PROLATE, 2), ok, 0.5)
    # a lone pair: u = K(x) f exactly as the kernel formula (oracle.cpp:36-42)
    u = ctx.direct_sum(0, ok)
    d = x[1] - x[2]
    r = np.linalg.norm(d)
    want = s[2] / (8 * np.pi * r) + d * (d @ s[2]) / (8 * np.pi * r ** 3)
    assert np.allclose(u[:3], want, rtol=1e-14, atol=0)


@pytest.mark.parametrize("kernel,eps,bound", [(0, 1e-6, 3e-6), (1, 1e-6, 5e-6), (0, 1e-9, 3e-9)])
def test_dmk_accuracy_vs_gpu_direct_sum(kernel, eps, bound):
    """acceptance.cpp:451-474 (DMK vs the exact sum) at N = 1e5 uniform points."""
    x, s, _ = _system(kernel, 3, 100_000, 0, 5 + kernel)
    sysm = g.ParticleSystem(3, x, np.zeros(0), s)
    ctx = g.Context(0)
    exact = ctx.direct_sum(kernel, sysm)
    u = ctx.evaluate(kernel, sysm, eps)
    err = float(np.linalg.norm(u - exact) / np.linalg.norm(exact))
    assert err <= bound, err
