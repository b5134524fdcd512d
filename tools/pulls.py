"""Per-iteration pull distribution (estimate - truth) / sigma_iteration over
seeds, per stream (compat = the reference bit for bit, philox = 24-bit bins,
philox_exact): checks the Philox paths for bias beyond the reference's own
early-iteration bias.

    python tools/pulls.py FAMILY DIMS MAXCALLS SEEDS [compat,philox,philox_exact]
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_01753_b200 as M  # noqa: E402

fam = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mc = int(float(sys.argv[3])) if len(sys.argv) > 3 else 10 ** 7
nseed = int(sys.argv[4]) if len(sys.argv) > 4 else 40
its = 8
ctx = M.Context(0)
f = M.make_suite_integrand(fam, d)
truth = f.reference
streams = sys.argv[5].split(",") if len(sys.argv) > 5 else ["compat", "philox"]
for stream in streams:
    rng, bins = ("philox", "exact") if stream == "philox_exact" else (stream, "")
    P = np.zeros((nseed, its))
    for s in range(nseed):
        cfg = M.RunConfig(dims=d, maxcalls=mc, itmax=its, ita=its, tau_rel=1e-15, seed=s, lower=[0.0] * d,
                          upper=[1.0] * d, rng=rng, bins=bins)
        r = M.integrate(f, cfg, ctx=ctx)
        for i, h in enumerate(r.history):
            P[s, i] = (h.estimate - truth) / math.sqrt(h.variance)
    print(f"f{fam} {d}D {mc:.0e} {stream:12s} mean pull per iteration: " + " ".join(f"{x:6.2f}" for x in P.mean(0))
          + f"   ({nseed} seeds)")
    print(f"f{fam} {d}D {mc:.0e} {stream:12s}  std pull per iteration: " + " ".join(f"{x:6.2f}" for x in P.std(0)))
