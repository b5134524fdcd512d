"""GPU: BASELINE-size workloads, checked through size-independent properties
(the oracle is too slow at these sizes):

* exact-sum conservation: every sample deposits the same (f J)^2 on every
  axis, so each contribution row sums the same multiset -- rows agree to the
  rounding of their cells (<= n_bins ulp);
* determinism: repeated runs are bitwise identical;
* partition additivity: exchange words of disjoint cube slices (simulated
  GPUs) sum to the full words bit for bit, including across the 2^32 cube
  index boundary (8D at maxcalls 1e10: m = 2^32);
* statistics: the estimate is within 5 sigma of the analytic value;
* write accounting: writes = m * p * bin_axes.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_2202_01753_b200 as M
from conftest import bits, words_value

pytestmark = pytest.mark.gpu


def _setup(d, maxcalls):
    return M.setup(M.RunConfig(dims=d, maxcalls=maxcalls, lower=[0.0] * d, upper=[1.0] * d))


@pytest.mark.parametrize("fam,d,maxcalls", [(4, 8, 10 ** 9), (2, 8, 10 ** 8), (4, 6, 10 ** 9), (3, 10, 10 ** 8)])
def test_large_v_sample_properties(ctx, fam, d, maxcalls):
    sp = _setup(d, maxcalls)
    f = M.make_suite_integrand(fam, d)
    g = M.Grid(d, 50, [0.0] * d, [1.0] * d)
    a = M.v_sample(f, g, sp.m, sp.s, sp.p, 1, 1, ctx=ctx)
    b = M.v_sample(f, g, sp.m, sp.s, sp.p, 1, 1, ctx=ctx)
    assert bits(a.raw_estimate) == bits(b.raw_estimate) and bits(a.raw_variance) == bits(b.raw_variance)
    assert np.array_equal(a.contributions.values.view(np.uint64), b.contributions.values.view(np.uint64))
    assert a.contributions.writes() == sp.m * sp.p * d
    rows = [a.contributions.axis_row(j).sum() for j in range(d)]
    assert all(math.isclose(r, rows[0], rel_tol=60 * 2.3e-16) for r in rows)
    assert abs(a.raw_estimate - f.reference) < 5 * math.sqrt(a.raw_variance)


def _words(ctx, run, it, n0, n1, x):
    run.sample(it, n0, n1)
    run.reduce(it)
    return x.clone()


@pytest.mark.parametrize("d,maxcalls", [(8, 10 ** 10), (2, 10 ** 10)])
def test_partition_additivity_at_scale(ctx, d, maxcalls):
    cfg = M.RunConfig(dims=d, maxcalls=maxcalls, itmax=1, ita=1, tau_rel=1e-15, lower=[0.0] * d, upper=[1.0] * d)
    f = M.make_suite_integrand(4, d)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    try:
        with torch.cuda.stream(stream):
            run = M.Run(f, cfg, ctx)
            m = run.work_items
            assert m >= 2 ** 32
            x = torch.zeros(run.exchange_words(), dtype=torch.int64, device="cuda")
            run.set_exchange(x.data_ptr())
            full = _words(ctx, run, 1, 0, m, x)
            cuts = [0, m // 4, 2 ** 31 + 7, 2 ** 32 - 3 if m > 2 ** 32 else m - 5, m]
            cuts = sorted(set(c for c in cuts if 0 <= c <= m))
            acc = torch.zeros_like(x)
            for a, b in zip(cuts[:-1], cuts[1:]):
                acc += _words(ctx, run, 1, a, b, x)
            assert words_value(acc.cpu().numpy()) == words_value(full.cpu().numpy())
            x.copy_(full)
            run.finish(1)
            r = run.result()
            run.close()
        torch.cuda.synchronize()
    finally:
        ctx.set_stream(0)
    assert r.iterations_used == 1
    assert abs(r.estimate - f.reference) < 5 * r.sigma


def test_integrate_c3_6d_1e9(ctx):
    """BASELINE config 3 shape: 6D f4 at 1e9 evals/iteration, a short schedule."""
    d = 6
    cfg = M.RunConfig(dims=d, maxcalls=10 ** 9, itmax=3, ita=2, tau_rel=1e-12, lower=[0.0] * d, upper=[1.0] * d)
    f = M.make_suite_integrand(4, d)
    r = M.integrate(f, cfg, ctx=ctx)
    assert r.params.m == 28 ** 6 and r.iterations_used == 3
    assert abs(r.estimate - f.reference) < 5 * r.sigma
    assert r.sigma / r.estimate < 1e-4
