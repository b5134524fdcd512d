"""One C1 integrate() (5D f4, 1e6 calls, 10 iterations) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_01753_b200 as M  # noqa: E402

rng = sys.argv[1] if len(sys.argv) > 1 else "philox"
ctx = M.Context(0)
cfg = M.RunConfig(dims=5, maxcalls=10**6, itmax=10, ita=10, tau_rel=1e-12, seed=1, lower=[0.0]*5, upper=[1.0]*5,
                  rng=rng)
f = M.make_suite_integrand(4, 5)
for _ in range(2):
    r = M.integrate(f, cfg, ctx=ctx)
print(r.estimate)
