"""Small-ncall latency of integrate() (wall clock, best of N): BASELINE C1
(5D f4, 1e6 calls, 10 iterations) and the bench's time-to-epsrel case
(8D f5, 1e7 calls, tau 1e-3, itmax 30: converges at iteration 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_01753_b200 as M  # noqa: E402

ctx = M.Context(0)
cases = [("C1 5D f4 1e6 x10", 4, 5, 10 ** 6, 10, 10, 1e-12, 0),
         ("8D f5 1e7 tau1e-3", 5, 8, 10 ** 7, 30, 10, 1e-3, 1)]
for name, fam, d, mc, itmax, ita, tau, seed in cases:
    for rng in ("compat", "philox"):
        f = M.make_suite_integrand(fam, d)
        cfg = M.RunConfig(dims=d, maxcalls=mc, itmax=itmax, ita=ita, tau_rel=tau, seed=seed, lower=[0.0] * d,
                          upper=[1.0] * d, rng=rng)
        M.integrate(f, cfg, ctx=ctx)
        best = 1e30
        for _ in range(7):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = M.integrate(f, cfg, ctx=ctx)
            best = min(best, time.perf_counter() - t0)
        print(f"{name:22s} {rng:7s} {1e3 * best:8.3f} ms  iterations={r.iterations_used} converged={r.converged} "
              f"est={r.estimate!r}")
