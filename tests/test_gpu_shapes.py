"""GPU: shapes beyond one CTA's shared-memory histogram, against the reference.

An adjusting K1 block holds bin_axes x (n_bins + 1) exact accumulators
(67 words each) in shared memory; shapes whose histograms exceed it -- 8D at
100 or 200 bins, 12D at 100 bins, 15+ axes at 50 bins -- are sampled in
several bin passes over the same keyed points (engine.cuh launch_k1).  The
reference accepts any n_bins >= 2 and any dims < 63 (driver.hpp:52-56,
grid.hpp:30-50); the B200 path compiles dims <= 20.  Estimate, variance, all
contribution cells and the device-counted writes must match the reference
bit for bit (f2: + - * / only), and whole integrate() runs its trajectory.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
import paper_2202_01753_b200 as M
from conftest import bits, same_bits

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

THREADS = os.cpu_count() or 1


def _grid(d, nb, seed):
    """A non-uniform grid (monotone random edges) on [0,1]^d."""
    rng = np.random.default_rng(seed)
    e = np.cumsum(rng.uniform(0.2, 1.0, size=(d, nb)), axis=1)
    e = e / e[:, -1:]
    e[:, -1] = 1.0
    return e.ravel()


@pytest.mark.parametrize("d,nb,maxcalls,mode", [
    (8, 100, 10 ** 6, "all"), (8, 200, 10 ** 6, "all"), (8, 200, 10 ** 6, "axis0"), (12, 100, 10 ** 6, "all"),
    (15, 50, 2 * 10 ** 5, "all"), (17, 50, 3 * 10 ** 5, "all"), (20, 50, 2_200_000, "all"), (20, 60, 2_200_000, "frozen"),
    (8, 100, 10 ** 8, "all"),  # row mode and two bin passes
])
def test_large_histograms_bitwise_vs_reference(ctx, d, nb, maxcalls, mode):
    sp = M.setup(M.RunConfig(dims=d, n_bins=nb, maxcalls=maxcalls, lower=[0.0] * d, upper=[1.0] * d))
    edges = _grid(d, nb, d * 1000 + nb)
    f = M.make_suite_integrand(2, d)
    g = M.Grid.from_edges(d, nb, [0.0] * d, [1.0] * d, edges)
    want = O.v_sample("ref", 2, None, d, nb, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 5, 2, mode, THREADS)
    if mode == "frozen":
        r = M.v_sample_no_adjust(f, g, sp.m, 1, sp.p, 5, 2, ctx=ctx)
        assert bits(r.raw_estimate) == bits(want["est"]) and bits(r.raw_variance) == bits(want["var"])
        return
    bu = M.BinUpdate.axis0_only if mode == "axis0" else M.BinUpdate.all_axes
    r = M.v_sample(f, g, sp.m, 1, sp.p, 5, 2, bu, ctx=ctx)
    assert bits(r.raw_estimate) == bits(want["est"]) and bits(r.raw_variance) == bits(want["var"])
    assert same_bits(r.contributions.values, want["contrib"])
    assert r.contributions.writes() == want["writes"] == sp.m * sp.p * (d if mode == "all" else 1)


@pytest.mark.parametrize("rng", ["philox", "philox_exact"])
@pytest.mark.parametrize("d,nb", [(8, 100), (12, 100), (18, 50)])
def test_large_histograms_philox_bitwise_vs_c_twin(ctx, d, nb, rng):
    maxcalls = 10 ** 6 if d < 18 else 600_000
    sp = M.setup(M.RunConfig(dims=d, n_bins=nb, maxcalls=maxcalls, lower=[0.0] * d, upper=[1.0] * d))
    edges = _grid(d, nb, 7 + d)
    g = M.Grid.from_edges(d, nb, [0.0] * d, [1.0] * d, edges)
    r = M.v_sample(M.make_suite_integrand(2, d), g, sp.m, 1, sp.p, 3, 4, rng="philox",
                   bins="exact" if rng == "philox_exact" else "r24", ctx=ctx)
    want = O.v_sample("orc", 2, None, d, nb, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 3, 4, "all", THREADS,
                      rng=rng)
    assert bits(r.raw_estimate) == bits(want["est"]) and bits(r.raw_variance) == bits(want["var"])
    assert same_bits(r.contributions.values, want["contrib"])
    assert r.contributions.writes() == want["writes"]


@pytest.mark.parametrize("d,nb", [(8, 100), (12, 100)])
def test_integrate_large_histograms_matches_reference(ctx, d, nb):
    """A whole adaptive run at n_bins 100: iteration 1 bitwise, the
    trajectory (device grid adaptation: libdevice pow/log) within 1e-11, the
    same iteration count and convergence decision."""
    cfg = M.RunConfig(dims=d, n_bins=nb, maxcalls=2 * 10 ** 6, itmax=6, ita=4, tau_rel=1e-15, seed=3,
                      lower=[0.0] * d, upper=[1.0] * d)
    r = M.integrate(M.make_suite_integrand(2, d), cfg, ctx=ctx)
    o = O.integrate("ref", 2, None, d, nb, cfg.maxcalls, cfg.itmax, cfg.ita, cfg.tau_rel, 1.5, 1.5, 3, 0,
                    [0.0] * d, [1.0] * d, workers=THREADS)
    assert r.iterations_used == o["iterations_used"] and r.converged == o["converged"]
    assert bits(r.history[0].estimate) == bits(o["hist_est"][0])
    np.testing.assert_allclose([h.estimate for h in r.history], o["hist_est"], rtol=1e-11)
    assert r.total_samples == o["total_samples"] and r.bin_writes == o["bin_writes"]
