"""BASELINE config 4 throughput probe: 6D table integrand (device-resident
4096-point interpolation tables), integrate() at 1e8 and 1e9 calls."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_01753_b200 as M  # noqa: E402

ctx = M.Context(0)
d, n = 6, 4096
t = np.linspace(0, 1, n)
rng = np.random.default_rng(0)
tabs = np.array([0.2 + np.exp(-0.5 * ((t - rng.uniform(0.3, 0.7)) / rng.uniform(0.05, 0.2)) ** 2) for _ in range(d)])
f = M.make_table_integrand(tabs, [0.0] * d, [1.0] * d)
for mc in (10 ** 8, 10 ** 9):
    for r in ("compat", "philox"):
        cfg = M.RunConfig(dims=d, maxcalls=mc, itmax=3, ita=3, tau_rel=1e-15, seed=1, lower=[0.0] * d,
                          upper=[1.0] * d, rng=r)
        M.integrate(f, cfg, ctx=ctx)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = M.integrate(f, cfg, ctx=ctx)
        dt = time.perf_counter() - t0
        print(f"table6d {mc:.0e} {r}: {res.total_samples / dt:.3e} evals/s  est={res.estimate:.10g}")
