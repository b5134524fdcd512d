"""The reference's acceptance criteria c2-c6 (proj/tests/acceptance.cpp:173-367),
run against the B200 path on either stream.

Each gate returns (pass, details) exactly as the reference's `report()` line
("criterion N: PASS|FAIL (...)").  The reference's own outcome on its CPU
library (proj/test_output.txt) is c2 FAIL (median sigma 99.49 > 2.0, the gate
is mis-set for fA at 2e6 calls) and c3..c6 PASS; the compat stream reproduces
those numbers bit for bit or to libm ulps, and the Philox stream must reach
the same outcomes.
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

from . import mcubes as M

REFERENCE_OUTCOME = {2: False, 3: True, 4: True, 5: True, 6: True}  # proj/test_output.txt


def _median(v):
    return float(np.median(np.asarray(v, dtype=float))) if len(v) else float("nan")


def accuracy_group(fid: str, dims: int, tau: float, maxcalls: int, variant, rng: str, ctx, seed0: int = 0) -> tuple:
    """run_accuracy_group (acceptance.cpp:60-103): 20 seeds, itmax 30, ita 10;
    converged runs need median |err| <= tau and >= 90% within 3 tau."""
    spec = M.make_integrand(fid, dims)
    truth = spec.reference
    errs, conv = [], 0
    for seed in range(seed0, seed0 + 20):
        cfg = M.RunConfig(dims=spec.dims, n_bins=50, maxcalls=maxcalls, itmax=30, ita=10, tau_rel=tau, seed=seed,
                          variant=variant, lower=spec.lower, upper=spec.upper, rng=rng)
        r = M.integrate(spec, cfg, ctx=ctx)
        if not r.converged:
            continue
        conv += 1
        errs.append(abs(r.estimate - truth) / abs(truth))
    label = f"{fid} d={spec.dims} tau={tau:.0e}{' 1d' if variant == M.Variant.mcubes1d else ''}: {conv}/20 conv"
    ok = False
    if errs:
        med = _median(errs)
        within = sum(e <= 3.0 * tau for e in errs) / len(errs)
        ok = med <= tau and within >= 0.9
        label += f" med {med:.2e} in3t {100 * within:.0f}%"
    return ok, label


def c2(rng: str, ctx):
    spec = M.make_fA()
    truth = -49.165073  # published benchmark value (acceptance.cpp:175)
    within, sigmas = 0, []
    for seed in range(20):
        cfg = M.RunConfig(dims=spec.dims, maxcalls=2000000, itmax=10, ita=10, tau_rel=1e-3, seed=seed,
                          lower=spec.lower, upper=spec.upper, rng=rng)
        r = M.integrate(spec, cfg, ctx=ctx)
        within += abs(r.estimate - truth) <= 3.0 * r.sigma
        sigmas.append(r.sigma)
    med = _median(sigmas)
    return within >= 18 and med <= 2.0, (f"{within}/20 runs within 3 sigma of {truth:.6f} (need >= 18), "
                                         f"median sigma {med:.4g} (gate 2.0)"), within, med


def c3(rng: str, ctx):
    spec = M.make_fB()
    good, sigmas = 0, []
    for seed in range(20):
        cfg = M.RunConfig(dims=spec.dims, maxcalls=2000000, itmax=15, ita=10, tau_rel=1e-3, seed=seed,
                          lower=spec.lower, upper=spec.upper, rng=rng)
        r = M.integrate(spec, cfg, ctx=ctx)
        good += (abs(r.estimate - 1.0) <= 3.0 * r.sigma) and r.sigma <= 1e-2
        sigmas.append(r.sigma)
    return good >= 18, (f"{good}/20 runs within 3 sigma of 1.0 at sigma <= 1e-2 (need >= 18), "
                        f"median sigma {_median(sigmas):.3g}")


def c4(rng: str, ctx, seed0: int = 0):
    cells = (("f2", 6, 1000000), ("f3", 3, 1000000), ("f4", 8, 2000000), ("f5", 8, 1000000))
    ok, labels = True, []
    for fid, d, mc in cells:
        for tau in (1e-3, 2e-4):
            p, lab = accuracy_group(fid, d, tau, mc, M.Variant.mcubes, rng, ctx, seed0)
            ok = ok and p
            labels.append(lab)
    return ok, "; ".join(labels)


def c5(rng: str, ctx):
    spec = M.make_suite_integrand(1, 6)
    nonconv = full = 0
    for seed in range(3):
        cfg = M.RunConfig(dims=6, maxcalls=200000, itmax=100, ita=10, tau_rel=2e-4, seed=seed, lower=spec.lower,
                          upper=spec.upper, rng=rng)
        r = M.integrate(spec, cfg, ctx=ctx)
        nonconv += not r.converged
        full += r.iterations_used == 100
    return nonconv == 3 and full == 3, (f"{nonconv}/3 seeds fail to converge at tau 2e-4 within 100 iterations "
                                        f"(expected: all)")


def c6(rng: str, ctx, seed0: int = 0):
    sym_ok, checks, writes_ok = True, 0, True
    for fam in (4, 5):
        spec = M.make_suite_integrand(fam, 8)
        base = dict(dims=8, maxcalls=100000, itmax=5, ita=3, tau_rel=1e-12, seed=0, lower=spec.lower,
                    upper=spec.upper, rng=rng)
        w_full, w_one = [], []
        full = M.integrate(spec, M.RunConfig(**base), observer=lambda v: w_full.append(v.bin_writes), ctx=ctx)

        def obs(v):
            nonlocal sym_ok, checks
            w_one.append(v.bin_writes)
            if not v.adjusting:
                return
            row0 = v.grid.edges(0).view(np.uint64)
            for j in range(v.grid.dims()):
                if not np.array_equal(v.grid.edges(j).view(np.uint64), row0):
                    sym_ok = False
                checks += 1

        one = M.integrate(spec, M.RunConfig(variant=M.Variant.mcubes1d, **base), observer=obs, ctx=ctx)
        if len(w_full) != len(w_one):
            writes_ok = False
        for i in range(min(len(w_full), len(w_one))):
            adjusting = i < base["ita"]
            if adjusting:
                writes_ok &= w_full[i] == 8 * w_one[i] and w_one[i] != 0
            else:
                writes_ok &= w_full[i] == 0 and w_one[i] == 0
        writes_ok &= full.bin_writes == 8 * one.bin_writes
    acc_ok, labels = True, []
    for tau in (1e-3, 2e-4):
        for fid in ("f4", "f5"):
            p, lab = accuracy_group(fid, 8, tau, 2000000 if fid == "f4" else 1000000, M.Variant.mcubes1d, rng, ctx,
                                    seed0)
            acc_ok = acc_ok and p
            labels.append(lab)
    head = (f"boundaries bitwise symmetric in {checks} axis checks: {'yes' if sym_ok else 'NO'}; bin writes 1/8 of "
            f"full variant: {'yes' if writes_ok else 'NO'}; ")
    return sym_ok and writes_ok and acc_ok, head + "; ".join(labels)


def run_all(rng: str = "compat", ctx: Optional[M.Context] = None, out=print) -> dict:
    ctx = ctx or M.default_context()
    res = {}
    p, d, *_ = c2(rng, ctx)
    res[2] = p
    out(f"[{rng}] criterion 2: {'PASS' if p else 'FAIL'} ({d})")
    for n, fn in ((3, c3), (4, c4), (5, c5), (6, c6)):
        p, d = fn(rng, ctx)
        res[n] = p
        out(f"[{rng}] criterion {n}: {'PASS' if p else 'FAIL'} ({d})")
    return res


def gate_pass_rates(rng: str, ctx=None, sets: int = 10) -> dict:
    """Pass rates of the statistical gates c4 and c6 over `sets` disjoint blocks
    of 20 seeds: the reference fixes seeds 0..19, and its gates are themselves
    random outcomes (c6's median over as few as 4 converged runs, say)."""
    ctx = ctx or M.default_context()
    out = {}
    for n, fn in ((4, c4), (6, c6)):
        out[n] = sum(fn(rng, ctx, 20 * k)[0] for k in range(sets)) / sets
    return out


if __name__ == "__main__":
    import sys

    args = sys.argv[1:]
    if args and args[0] == "rates":
        for stream in args[1:] or ["compat", "philox"]:
            print(f"[{stream}] pass rate over 10 seed blocks:", gate_pass_rates(stream))
    else:
        for stream in args or ["compat", "philox"]:
            run_all(stream)
