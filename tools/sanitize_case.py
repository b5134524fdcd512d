"""Small-shape workload for compute-sanitizer (memcheck / racecheck /
synccheck): adjusting + frozen iterations on both streams, 2D..8D, the
integrate() loop with its finish kernel, and a non-finite sample."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_01753_b200 as M  # noqa: E402

ctx = M.Context(0)
for rng in ("compat", "philox"):
    for d, m, fam in ((2, 40 ** 2, 2), (5, 5 ** 5, 4), (8, 3 ** 8, 5)):
        g = M.Grid(d, 50, [0.0] * d, [1.0] * d)
        f = M.make_suite_integrand(fam, d)
        M.v_sample(f, g, m, 1, 2, 1, 1, rng=rng, ctx=ctx)
        M.v_sample_no_adjust(f, g, m, 1, 2, 1, 2, rng=rng, ctx=ctx)
    cfg = M.RunConfig(dims=4, maxcalls=20000, itmax=4, ita=2, tau_rel=1e-12, lower=[0.0] * 4, upper=[1.0] * 4, rng=rng)
    M.integrate(M.make_suite_integrand(4, 4), cfg, ctx=ctx)
try:
    M.v_sample(M.test_integrand("inf_if_x0_pos", 1), M.Grid(1, 4, [0.0], [1.0]), 4, 1, 2, 1, 1, ctx=ctx)
except M.NonFiniteSample:
    pass
print("sanitize case done")
