"""integrate() wall time vs itmax at BASELINE C1 size: slope = per-iteration
cost, intercept = fixed per-call cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_01753_b200 as M  # noqa: E402

ctx = M.Context(0)
f = M.make_suite_integrand(4, 5)
for its in (1, 2, 5, 10, 20):
    cfg = M.RunConfig(dims=5, maxcalls=10**6, itmax=its, ita=its, tau_rel=1e-12, seed=1, lower=[0.0]*5,
                      upper=[1.0]*5, rng="philox")
    M.integrate(f, cfg, ctx=ctx)
    best = 1e9
    for _ in range(7):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M.integrate(f, cfg, ctx=ctx)
        best = min(best, time.perf_counter() - t0)
    print(its, round(best * 1e6, 1), "us")
