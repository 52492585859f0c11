"""Guard-mode runs: a memcheck / initcheck stand-in (compute-sanitizer is
closed on the GPU pool, profiles/round2/sanitizer/).

A guarded context (include/sdmk.h sdmk_set_guard) allocates every device
buffer at exactly its requested size between two 64 KB canary regions and
fills it with all-ones bytes (NaN doubles, -1 integers) before first use.  So
  * a kernel storing past either end of a buffer overwrites a canary, which
    sdmk_guard_check reports by buffer name;
  * a kernel reading an element that no kernel wrote (the write-only incoming
    proxies, the never-zeroed outgoing of source-free boxes, padded tiles)
    pulls a NaN or a -1 index into the result, which the parity check against
    the compiled reference (or the unguarded run, bitwise) then fails.
The cases cover every kernel family on the metric path (k_anterp2, k_acc_group
TMA ring, k_fwd_xy3 TMA bulk stores, k_inv_xy3, the z stages, k_interp_mma,
k_residual's work queue and spill lists), the FFMA 2D / p > 32 kernels, the
periodic and separate-target paths, the sharded halo path and the FFT Ewald.
"""
import numpy as np
import pytest

from conftest import parity_ok
from test_gpu_parity import CASES, _make, _ref

import paper_2509_21471_b200 as g

pytestmark = pytest.mark.gpu


def _guarded():
    c = g.Context(0)
    c.set_guard(True)
    return c


@pytest.mark.parametrize("case", CASES)
def test_guarded_matches_reference(case):
    ref = _ref()
    kernel, dim, n, eps, per, dist, ntgt = case
    x, s, t = _make(kernel, dim, n, 11 + n, dist, ntgt)
    plan = ref.select_parameters(kernel, eps, 0, dim)
    ur, _ = ref.RefProblem(plan, dim, x, s, t, per).evaluate()
    ctx = _guarded()
    u = ctx.evaluate_with_plan(g.DmkPlan(**plan), g.ParticleSystem(dim, x, t if t is not None else np.zeros(0), s),
                               int(per))
    assert ctx.guard_check() == []
    assert np.isfinite(u).all()
    ok, err = parity_ok(u, ur, 1e-10)
    assert ok, err


@pytest.mark.parametrize("kernel,n", [(0, 400000), (1, 200000)])
def test_guarded_bitwise_at_depth(kernel, n):
    """Deeper trees (levels >= 4, full 320-target interpolation passes, the
    spill lists of the residual) than the reference can check in seconds:
    the guarded run equals the unguarded one bit for bit."""
    x, s, _ = _make(kernel, 3, n, 5)
    plan = g.select_parameters(kernel, 1e-6, 0, 3)
    sysm = g.ParticleSystem(3, x, np.zeros(0), s)
    plain = g.Context(0).evaluate_with_plan(plan, sysm, 0)
    ctx = _guarded()
    u = ctx.evaluate_with_plan(plan, sysm, 0)
    assert ctx.guard_check() == []
    assert np.array_equal(u, plain)
    # a second evaluation reuses the buffers (no fresh poison): still equal
    assert np.array_equal(ctx.evaluate_with_plan(plan, sysm, 0), plain)
    assert ctx.guard_check() == []


def test_guarded_halo_shards():
    x, s, _ = _make(0, 3, 60000, 37, "mixture")
    plan = g.select_parameters(0, 1e-6, 0, 3)
    sysm = g.ParticleSystem(3, x, np.zeros(0), s)
    full = g.Context(0).evaluate_with_plan(plan, sysm, 0)
    ctxs = [_guarded() for _ in range(3)]
    for r, c in enumerate(ctxs):
        c.set_shard(r, 3)
        c.set_manual_exchange(True)
        c.evaluate_begin(plan, sysm, 0)
    for a in ctxs:
        for b in ctxs:
            if a is not b:
                a.halo_transfer_to(b)
    acc = np.zeros_like(full)
    for c in ctxs:
        acc += c.evaluate_end()
        assert c.guard_check() == []
    assert np.array_equal(acc, full)


def test_guarded_ewald():
    x, s, _ = _make(0, 3, 50000, 3)
    plan = g.select_parameters(0, 1e-8, 0, 3)
    sysm = g.ParticleSystem(3, x, np.zeros(0), s)
    plain = g.Context(0).ewald(plan, sysm)
    ctx = _guarded()
    u = ctx.ewald(plan, sysm)
    assert ctx.guard_check() == []
    assert np.array_equal(u, plain)


def test_guard_refused_after_allocation():
    """Guard mode is fixed before the first allocation: switching it later is
    refused (buffers already handed out would lose their canaries)."""
    x, s, _ = _make(0, 3, 5000, 1)
    plan = g.select_parameters(0, 1e-6, 0, 3)
    ctx = _guarded()
    ctx.evaluate_with_plan(plan, g.ParticleSystem(3, x, np.zeros(0), s), 0)
    assert ctx.guard_check() == []
    with pytest.raises(ValueError):
        ctx.set_guard(False)


def test_guard_catches_overrun():
    """The detector itself: a one-byte store past either end of a buffer is
    reported by name (and an unguarded context reports nothing)."""
    ctx = _guarded()
    assert ctx.guard_selftest()
    assert ctx.guard_check() == []
    assert not g.Context(0).guard_selftest()
