"""Generate the committed golden fixtures from the compiled reference.

Run here (where /root/reference exists):  python tests/golden/gen_golden.py

Every value comes from oracle/_ref/libmcubes_ref.so -- the UNMODIFIED
reference headers (/root/reference/proj/include/mcubes) compiled with the
reference's own -ffp-contract=off -- and is stored as hex bit patterns so the
tests can compare bit for bit.  The GPU box has no /root/reference; the tests
read only this JSON.
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402


def hx(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def hxa(a) -> list:
    return [hx(v) for v in np.asarray(a, dtype=np.float64).reshape(-1)]


def table_params(d: int, n: int, lower, upper, seed: int = 0):
    """Synthetic 'cosmology-style' tables: smooth positive bumps (BASELINE config 4)."""
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, n)
    tabs = []
    for j in range(d):
        c, w = rng.uniform(0.3, 0.7), rng.uniform(0.05, 0.2)
        tabs.append(0.2 + np.exp(-0.5 * ((t - c) / w) ** 2))
    tabs = np.array(tabs)
    inv_h = [float(n - 1) / (upper[j] - lower[j]) for j in range(d)]
    return np.concatenate([[float(n)], lower, inv_h, tabs.reshape(-1)])


def ref_adjust(d, nb, lower, upper, edges, contrib, alpha=1.5, symmetric=0):
    out = np.zeros(d * nb)
    rc = O.ref().ref_grid_adjust(d, nb, O.darr(lower), O.darr(upper), O.ptr(edges), O.ptr(contrib), alpha,
                                 symmetric, O.ptr(out))
    assert rc == 0, O.ref().ref_last_error()
    return out


def sample_case(name, fid, params, d, nb, lower, upper, edges, m, s, p, seed, it, mode="all"):
    r = O.v_sample("ref", fid, params, d, nb, lower, upper, edges, m, s, p, seed, it, mode=mode, threads=3)
    case = dict(name=name, integrand=fid, params=None if params is None else hxa(params), dims=d, n_bins=nb,
                lower=list(lower), upper=list(upper), edges=None if edges is None else hxa(edges), m=m, s=s, p=p,
                seed=seed, iteration=it, mode=mode, est=hx(r["est"]), var=hx(r["var"]), writes=r["writes"])
    if r["contrib"] is not None:
        case["contrib"] = hxa(r["contrib"])
    return case, r


def warm_grid(fid, params, d, nb, lower, upper, m, p, seed, rounds):
    """Grids adapted by the reference itself (test_oracle.cpp:91-96)."""
    edges = O.uniform_edges(d, nb, lower, upper)
    for it in range(rounds):
        r = O.v_sample("ref", fid, params, d, nb, lower, upper, edges, m, 4, p, seed, it, mode="all", threads=2)
        edges = ref_adjust(d, nb, lower, upper, edges, r["contrib"])
    return edges


def main():
    lib = O.ref()
    out = {"generator": "tests/golden/gen_golden.py (oracle/_ref: reference headers compiled in place)"}

    # ---- keyed RNG (rng.hpp:63-68)
    keys = [(0, 0, 0, 0, 0), (1, 1, 0, 0, 0), (42, 1, 12345, 1, 7), (7, 3, 2 ** 32, 1, 2),
            (2 ** 63 + 5, 17, 49999643235, 15, 9), (3, 1, 0, 1, 0)]
    out["uniform01"] = [dict(key=list(k), value=hx(lib.ref_uniform01(*k))) for k in keys]
    out["iteration_root"] = [dict(seed=s, it=i, value="%016x" % lib.ref_iteration_root(s, i))
                             for s, i in [(0, 1), (7, 3), (123456789, 10)]]

    # ---- exact sums (exact_sum.hpp): random mixed-magnitude streams
    rng = np.random.default_rng(2026)
    streams = []
    for n in (1, 2, 17, 1000):
        v = rng.standard_normal(n) * np.exp2(rng.integers(-300, 300, n))
        streams.append(dict(values=hxa(v), sum=hx(lib.ref_exact_sum(O.ptr(v), n))))
    sub = np.array([5e-324, 5e-324, -1e-320, 2.2250738585072014e-308, 1e-310])
    streams.append(dict(values=hxa(sub), sum=hx(lib.ref_exact_sum(O.ptr(sub), len(sub)))))
    out["exact_sum"] = streams

    # ---- setup shapes (driver.hpp:93-123)
    shapes = []
    for d, mc in [(2, 1000), (8, 10 ** 8), (1, 4), (2, 17), (5, 10 ** 6), (8, 10 ** 7), (6, 10 ** 9), (8, 10 ** 10),
                  (8, 10 ** 11), (2, 10 ** 11), (10, 10 ** 6), (10, 10 ** 11), (5, 10 ** 9), (6, 10 ** 11),
                  (3, 10 ** 5), (9, 10 ** 6)]:
        sp = (O._U64 * 4)()
        rc = lib.ref_setup(d, 50, mc, 15, 10, 1e-3, 1.5, 1.5, O.darr([0.0] * d), O.darr([1.0] * d), 1, sp)
        assert rc == 0
        shapes.append(dict(dims=d, maxcalls=mc, g=sp[0], m=sp[1], p=sp[2], s_workers1=sp[3]))
    out["setup"] = shapes

    # ---- v_sample cases
    cases = []
    add = lambda *a, **k: cases.append(sample_case(*a, **k)[0])  # noqa: E731
    add("golden_triple_x0", 32, None, 1, 4, [0.0], [1.0], None, 4, 1, 2, 1, 0)
    add("const7_pow2_grid", 33, [7.0], 2, 4, [0.0, 0.0], [2.0, 2.0], None, 4, 1, 4, 9, 1)
    add("const3_general", 33, [3.0], 2, 50, [0.0, -1.0], [1.5, 2.0], None, 9, 2, 3, 4, 1)
    add("zero", 37, None, 2, 8, [0.0] * 2, [1.0] * 2, None, 16, 3, 2, 1, 1, mode="frozen")
    add("x0sq_half_single_cube", 34, None, 1, 50, [0.0], [1.0], None, 1, 1, 8, 3, 1)
    for d, m, p in [(1, 16, 3), (2, 64, 2), (3, 125, 4), (4, 81, 2), (6, 64, 5)]:
        lo, hi = [0.0] * d, [1.0] * d
        e = warm_grid(4, None, d, 8, lo, hi, m, p, 5, 2)
        add(f"f4_adapted_d{d}", 4, None, d, 8, lo, hi, e, m, 4, p, 5, 2)
    add("f5_axis0", 5, None, 3, 6, [0.0] * 3, [1.0] * 3, None, 27, 2, 3, 9, 1, mode="axis0")
    add("f5_all", 5, None, 3, 10, [0.0] * 3, [1.0] * 3, None, 27, 4, 3, 77, 2)
    add("f5_frozen", 5, None, 3, 10, [0.0] * 3, [1.0] * 3, None, 27, 4, 3, 77, 2, mode="frozen")
    add("f2_2d", 2, None, 2, 16, [0.0] * 2, [1.0] * 2, None, 64, 64, 4, 5, 3)
    add("f2_3d_survey", 2, None, 3, 8, [0.0] * 3, [1.0] * 3, None, 1000, 7, 3, 5, 1)
    # the 8D suite on a uniform and on a reference-adapted grid (BASELINE config 2 shapes, small ncall)
    for fam in range(1, 7):
        d = 8
        lo, hi = [0.0] * d, [1.0] * d
        add(f"f{fam}_8d_uniform", fam, None, d, 50, lo, hi, None, 4 ** 8, 9, 3, 3, 1)
        e = warm_grid(fam, None, d, 50, lo, hi, 4 ** 8, 3, 3, 2)
        add(f"f{fam}_8d_adapted", fam, None, d, 50, lo, hi, e, 4 ** 8, 9, 3, 3, 3)
    add("f2_8d_1e7", 2, None, 8, 50, [0.0] * 8, [1.0] * 8, None, 6 ** 8, 1000, 5, 3, 1)
    add("fA_6d", 7, None, 6, 50, [0.0] * 6, [10.0] * 6, None, 8 ** 6, 50, 3, 1, 1)
    add("fB_9d", 8, None, 9, 50, [-1.0] * 9, [1.0] * 9, None, 3 ** 9, 50, 3, 1, 1)
    tp = table_params(6, 4096, [0.0] * 6, [1.0] * 6)
    add("table_6d", 9, tp, 6, 50, [0.0] * 6, [1.0] * 6, None, 6 ** 6, 50, 2, 2, 1)
    add("f4_1d_large_g", 4, None, 1, 50, [0.0], [1.0], None, 100003, 7, 2, 11, 4)
    out["v_sample"] = cases

    # ---- grid adaptation (grid.hpp:104-146): random contributions on random grids
    adj = []
    rng = np.random.default_rng(31)
    for case in range(12):
        d = int(rng.integers(1, 5))
        nb = int(rng.integers(2, 60))
        lower = list(rng.uniform(-3.0, 1.0, d))
        upper = [lo + rng.uniform(0.5, 6.0) for lo in lower]
        e = O.uniform_edges(d, nb, lower, upper)
        for _ in range(int(rng.integers(0, 3))):
            e = ref_adjust(d, nb, lower, upper, e, rng.uniform(0.0, 1.0, d * nb))
        c = rng.uniform(0.0, 1.0, d * nb) * np.exp2(rng.integers(-40, 40))
        if case % 4 == 1:
            c[: nb // 2] = 0.0  # zero runs exercise the imp == 0 skip in the walk
        if case % 4 == 2 and d > 1:
            c[nb: 2 * nb] = 0.0  # an all-zero axis is left untouched
        sym = 1 if case % 3 == 0 else 0
        if sym:
            upper = list(upper)
        adj.append(dict(dims=d, n_bins=nb, lower=hxa(lower), upper=hxa(upper), edges=hxa(e), contrib=hxa(c),
                        alpha=1.5, symmetric=sym, out=hxa(ref_adjust(d, nb, lower, upper, e, c, 1.5, sym))))
    out["adjust"] = adj

    # ---- weighted estimate (driver.hpp:146-169)
    we = []
    for hist in ([(1.0, 0.01)], [(1.0, 0.01), (1.2, 0.04)], [(1.0, 0.01)] * 3, [(3.0, 1.0), (2.0, 0.0), (5.0, 0.0)],
                 [(1.7e-6, 3e-20), (1.79e-6, 1.1e-20), (1.791e-6, 4e-21)]):
        e = np.array([h[0] for h in hist])
        v = np.array([h[1] for h in hist])
        o3 = np.zeros(3)
        assert lib.ref_weighted_estimate(len(hist), O.ptr(e), O.ptr(v), O.ptr(o3)) == 0
        we.append(dict(est=hxa(e), var=hxa(v), out=hxa(o3)))
    out["weighted_estimate"] = we

    # ---- full integrate runs (driver.hpp:215-258)
    runs = []
    for name, fid, params, d, mc, itmax, ita, tau, seed, variant, lo, hi in [
        ("C1_f4_5d_1e6", 4, None, 5, 10 ** 6, 10, 10, 1e-9, 0, 0, [0.0] * 5, [1.0] * 5),
        ("readme_f2_3d_1e5", 2, None, 3, 10 ** 5, 15, 10, 1e-3, 7, 0, [0.0] * 3, [1.0] * 3),
        ("f4_2d_repro", 4, None, 2, 2000, 4, 2, 1e-9, 42, 0, [0.0] * 2, [1.0] * 2),
        ("f4_3d_mcubes1d", 4, None, 3, 1000, 3, 3, 1e-12, 5, 1, [0.0] * 3, [1.0] * 3),
        ("f2_8d_1e6_frozen_tail", 2, None, 8, 10 ** 6, 6, 3, 1e-12, 2, 0, [0.0] * 8, [1.0] * 8),
        ("const7_3d_exact", 33, [7.0], 3, 128, 15, 10, 1e-3, 0, 0, [0.0] * 3, [1.0] * 3),
        ("f5_8d_1e6_tau", 5, None, 8, 10 ** 6, 30, 10, 1e-3, 1, 0, [0.0] * 8, [1.0] * 8),
    ]:
        nb = 4 if name.startswith("const7") else 50
        r = O.integrate("ref", fid, params, d, nb, mc, itmax, ita, tau, 1.5, 1.5, seed, variant, lo, hi, workers=2,
                        want_grids=True)
        runs.append(dict(name=name, integrand=fid, params=None if params is None else hxa(params), dims=d,
                         n_bins=nb, maxcalls=mc, itmax=itmax, ita=ita, tau_rel=tau, seed=seed, variant=variant,
                         lower=lo, upper=hi, estimate=hx(r["estimate"]), sigma=hx(r["sigma"]),
                         chi2_dof=hx(r["chi2_dof"]), iterations_used=r["iterations_used"],
                         converged=r["converged"], total_samples=r["total_samples"], bin_writes=r["bin_writes"],
                         hist_est=hxa(r["hist_est"]), hist_var=hxa(r["hist_var"]), grids=[hxa(g) for g in r["grids"]],
                         writes=r["writes"]))
    out["integrate"] = runs

    # ---- reference values (integrands.hpp:53-103, 181-215)
    out["reference_value"] = [dict(family=f, dims=d, value=hx(lib.ref_reference_value(f, d)))
                              for f in range(1, 7) for d in (1, 2, 3, 5, 8)] + \
                             [dict(family=7, dims=6, value=hx(lib.ref_reference_value(7, 6))),
                              dict(family=8, dims=9, value=hx(lib.ref_reference_value(8, 9)))]

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print(f"wrote {path} ({os.path.getsize(path)} bytes): {len(cases)} v_sample cases, {len(adj)} adjust cases, "
          f"{len(runs)} integrate runs")


if __name__ == "__main__":
    main()
