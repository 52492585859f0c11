"""Host-buffer paths of evaluate_with_plan: pinned caller arrays above the
staging size send the strengths on a side stream that overlaps the tree
build (engine.cpp evaluate / build_problem).  The result must be bitwise the
pageable path's, and validation must keep the reference's precedence
(strengths before coordinates, oracle.cpp:116-127)."""
import numpy as np
import pytest
import torch

import paper_2509_21471_b200 as g

pytestmark = pytest.mark.gpu

N = 1_500_000  # 36 MB of strengths: above the 32 MB staging chunk


def _pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t, t.numpy()


@pytest.fixture(scope="module")
def system():
    rng = np.random.default_rng(3)
    return rng.uniform(-0.5, 0.5, (N, 3)), rng.standard_normal((N, 3))


def test_pinned_side_stream_matches_pageable(system):
    x, s = system
    ctx = g.Context(0)
    plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    u_page = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, np.zeros(0), s))
    keep = [_pinned(x), _pinned(s)]
    u_pin = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, keep[0][1], np.zeros(0), keep[1][1]))
    assert np.array_equal(u_page, u_pin)


def test_pinned_strength_errors_keep_reference_precedence(system):
    x, s = system
    ctx = g.Context(0)
    plan = g.select_parameters(0, 1e-6, g.PROLATE, 3)
    bad_s = s.copy()
    bad_s[N // 2, 1] = np.nan
    ts, hs = _pinned(bad_s)
    tx, hx = _pinned(x)
    with pytest.raises(ValueError, match="non-finite strength"):
        ctx.evaluate_with_plan(plan, g.ParticleSystem(3, hx, np.zeros(0), hs))
    bad_x = x.copy()
    bad_x[7, 0] = 0.75  # outside the unit box, and a non-finite strength: strengths are reported first
    tbx, hbx = _pinned(bad_x)
    with pytest.raises(ValueError, match="non-finite strength"):
        ctx.evaluate_with_plan(plan, g.ParticleSystem(3, hbx, np.zeros(0), hs))
    tg, hg = _pinned(s)
    with pytest.raises(ValueError, match="outside the unit box"):
        ctx.evaluate_with_plan(plan, g.ParticleSystem(3, hbx, np.zeros(0), hg))
    # the context is still usable after the failures
    ok = ctx.evaluate_with_plan(plan, g.ParticleSystem(3, hx, np.zeros(0), hg))
    assert np.all(np.isfinite(ok))


def test_array_length_errors_are_reported_before_any_read(gpu_ctx):
    """mismatched array lengths raise the reference's invalid_argument
    messages (oracle.cpp:108-115, dmk.cpp:1046-1047) instead of reading past an array."""
    rng = np.random.default_rng(5)
    x = rng.uniform(-0.5, 0.5, (100, 3))
    plan = g.select_parameters(1, 1e-6, g.PROLATE, 3)  # stresslet: 6 strength doubles per source
    cases = [
        (g.ParticleSystem(3, x, np.zeros(0), rng.standard_normal((100, 3))), "bad strength array length"),
        (g.ParticleSystem(3, x.ravel()[:-1], np.zeros(0), rng.standard_normal((100, 6))), "bad source array length"),
        (g.ParticleSystem(3, x, x.ravel()[:-2], rng.standard_normal((100, 6))), "bad target array length"),
        (g.ParticleSystem(2, x, np.zeros(0), rng.standard_normal((100, 6))), "plan and system dimensions differ"),
    ]
    for sys_, msg in cases:
        with pytest.raises(ValueError, match=msg):
            gpu_ctx.evaluate_with_plan(plan, sys_)
    with pytest.raises(ValueError, match="bad strength array length"):
        gpu_ctx.direct_sum(0, g.ParticleSystem(3, x, np.zeros(0), rng.standard_normal((99, 3))))
