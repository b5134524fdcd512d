"""Randomised parity sweep (evidence, not a test): random shapes, bounds,
seeds, iterations and bin modes through the B200 path against the C oracle,
for both streams.  compat is compared with oracle/mcubes_oracle.c (the
reference's arithmetic); philox with its C twin (run_cube_philox).  +-*/
integrands (f2) must agree bit for bit; transcendental ones (libdevice vs
glibc exp/cos/pow) are reported as the fraction of bitwise-equal estimates
and the largest relative difference.

    python tools/parity_sweep.py [trials]
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2202_01753_b200 as M  # noqa: E402


def bits(x):
    return np.float64(x).tobytes()


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    ctx = M.Context(0)
    rng = np.random.default_rng(2026)
    stats = {}
    for t in range(trials):
        stream = ("compat", "philox", "philox_exact")[t % 3]
        mrng, mbins = ("philox", "exact") if stream == "philox_exact" else (stream, "")
        d = int(rng.integers(1, 11))
        g = int(rng.integers(1, max(2, int(200000 ** (1 / d))) + 1))
        m = g ** d
        p = int(rng.integers(2, 9))
        nb = int(rng.integers(2, min(80, 700 // d)))  # adjusting K1 holds d*(nb+1) cells in shared memory
        fam = [2, 1, 3, 4, 5, 6][int(rng.integers(0, 6))]
        lo = list(rng.uniform(-1.0, 0.5, d))
        hi = [v + float(rng.uniform(0.5, 2.0)) for v in lo]
        seed, it = int(rng.integers(0, 2 ** 62)), int(rng.integers(1, 40))
        mode = ["all", "axis0", "frozen"][int(rng.integers(0, 3))]
        want = O.v_sample("orc", fam, None, d, nb, lo, hi, None, m, 1, p, seed, it, mode=mode, rng=stream)
        f = M.IntegrandSpec("f", d, lo, hi, fam)
        grid = M.Grid(d, nb, lo, hi)
        if mode == "frozen":
            r = M.v_sample_no_adjust(f, grid, m, 1, p, seed, it, ctx=ctx, rng=mrng)
            est, var, contrib = r.raw_estimate, r.raw_variance, None
        else:
            r = M.v_sample(f, grid, m, 1, p, seed, it,
                           M.BinUpdate.axis0_only if mode == "axis0" else M.BinUpdate.all_axes, ctx=ctx, rng=mrng,
                           bins=mbins)
            est, var, contrib = r.raw_estimate, r.raw_variance, r.contributions.values
        same = bits(est) == bits(want["est"]) and bits(var) == bits(want["var"])
        if contrib is not None:
            same = same and np.array_equal(np.asarray(contrib).view(np.uint64), np.asarray(want["contrib"]).view(np.uint64))
            assert r.contributions.writes() == want["writes"], (stream, d, m, p, nb, mode)  # device-counted deposits
        rel = abs(est - want["est"]) / max(abs(want["est"]), 1e-300)
        key = (stream, "f%d" % fam)
        s = stats.setdefault(key, [0, 0, 0.0])
        s[0] += 1
        s[1] += int(same)
        s[2] = max(s[2], rel)
        if fam == 2 and not same:
            print("MISMATCH", stream, d, m, p, nb, seed, it, mode, flush=True)
    print("# tools/parity_sweep.py %d trials: B200 v_sample / v_sample_no_adjust vs the C oracle" % trials)
    print("# (compat: the reference's arithmetic; philox / philox_exact: its C twin, 24-bit / exact bins).")
    print("# f2 is +-*/ only: must be bitwise.  Device-counted writes equal the oracle's in every adjusting case.")
    print("%-8s %-4s %7s %9s %14s" % ("stream", "f", "trials", "bitwise", "max rel diff"))
    for (stream, fam), (n, same, rel) in sorted(stats.items()):
        print("%-8s %-4s %7d %9d %14.3e" % (stream, fam, n, same, rel))


if __name__ == "__main__":
    main()
