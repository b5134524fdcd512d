"""GPU: statistical parity at the headline scale (BASELINE config 2's largest
8D shape, maxcalls 1e9: m = 12^8 sub-cubes per iteration), 16 seeds.

The north-star acceptance standard (BASELINE.json north_star): estimates
within 3 combined sigma of the reference's, the same convergence behaviour,
and agreement with the analytic value.  The compat stream IS the reference
(bitwise per iteration, tests/test_gpu_rowmode.py), so the Philox stream --
with 24-bit bin addends (the bench headline) and with exact bins -- is judged
against it on the same integrand, ncall and schedule:

* per-iteration pulls (I_i - truth) / sigma_i over iterations 2..6 of all
  seeds: mean and spread of a unit normal, like the compat stream's;
* final combined estimates within 3 combined sigma of compat's (>= 15 of 16)
  and of the analytic value;
* chi^2/dof of the combined estimate: the same distribution (means);
* time to tau_rel: the converged-iteration distribution matches compat's.

Reference call sites: tests/acceptance.cpp:48-99 (multi-seed acceptance
protocol), :236-261 (pull/chi^2 gates); driver.hpp:146-178.
"""
from __future__ import annotations

import math
import statistics

import pytest

import paper_2202_01753_b200 as M

pytestmark = pytest.mark.gpu

D, MAXCALLS, SEEDS = 8, 10 ** 9, range(100, 116)
STREAMS = {"compat": ("compat", ""), "philox_r24": ("philox", "r24"), "philox_exact": ("philox", "exact")}


def _chi2_dof(history):
    """chi^2/dof of a run of iterations about their weighted mean (driver.hpp:146-169)."""
    w = [1.0 / h.variance for h in history]
    mean = sum(wi * h.estimate for wi, h in zip(w, history)) / sum(w)
    return sum((h.estimate - mean) ** 2 / h.variance for h in history) / max(1, len(history) - 1)


def _runs(ctx, fam, itmax, ita, tau):
    f = M.make_suite_integrand(fam, D)
    out = {}
    for name, (rng, bins) in STREAMS.items():
        out[name] = [M.integrate(f, M.RunConfig(dims=D, maxcalls=MAXCALLS, itmax=itmax, ita=ita, tau_rel=tau,
                                                seed=s, lower=[0.0] * D, upper=[1.0] * D, rng=rng, bins=bins),
                                 ctx=ctx) for s in SEEDS]
    return f, out


@pytest.mark.parametrize("fam", [4, 5])
def test_pulls_and_combined_estimates_match_reference_stream(ctx, fam):
    f, runs = _runs(ctx, fam, itmax=6, ita=6, tau=1e-15)
    truth = f.reference
    stats = {}
    for name, rr in runs.items():
        # iterations 2..6: iteration 1 samples the uniform grid, where a peaked
        # integrand's variance estimate is unreliable on every stream
        pulls = [(h.estimate - truth) / math.sqrt(h.variance) for r in rr for h in r.history[1:]]
        stats[name] = (statistics.fmean(pulls), statistics.pstdev(pulls),
                       statistics.fmean(_chi2_dof(r.history[1:]) for r in rr))
        assert len(pulls) == 5 * len(SEEDS)
    for name, (mean, sd, chi2) in stats.items():
        assert abs(mean) < 0.45, stats  # 80 pulls: standard error 0.11
        assert 0.7 < sd < 1.35, stats
        assert 0.5 < chi2 < 1.6, stats  # 16 seeds x 4 dof: standard error of the mean 0.18
    for name, rr in runs.items():
        # the combined estimate against the analytic value
        assert sum(abs(r.estimate - truth) <= 3 * r.sigma for r in rr) >= 15, name
        # device-counted samples: every iteration sampled every cube p times
        assert all(r.total_samples == 6 * r.params.m * r.params.p for r in rr)
    for name in ("philox_r24", "philox_exact"):
        within = sum(abs(a.estimate - b.estimate) <= 3 * math.hypot(a.sigma, b.sigma)
                     for a, b in zip(runs[name], runs["compat"]))
        assert within >= 15, (name, within)
        # the same convergence behaviour: chi^2/dof and the estimate spread agree with the reference stream's
        assert abs(stats[name][2] - stats["compat"][2]) < 0.6, stats
        assert abs(stats[name][1] - stats["compat"][1]) < 0.4, stats


def test_time_to_tau_matches_reference_stream(ctx):
    """f5 at tau_rel 2e-5: the iteration at which each seed converges, per stream."""
    f, runs = _runs(ctx, 5, itmax=15, ita=10, tau=2e-5)
    its = {name: sorted(r.iterations_used for r in rr) for name, rr in runs.items()}
    conv = {name: sum(r.converged for r in rr) for name, rr in runs.items()}
    for name in ("philox_r24", "philox_exact"):
        assert abs(statistics.median(its[name]) - statistics.median(its["compat"])) <= 2, its
        assert abs(conv[name] - conv["compat"]) <= 4, conv
    for name, rr in runs.items():
        assert sum(abs(r.estimate - f.reference) <= 3 * r.sigma for r in rr if r.converged) >= conv[name] - 1, name
