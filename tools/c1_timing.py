"""Whole-run wall time of integrate() for BASELINE config 1 (C1: 5D f4,
maxcalls 1e6, 10 iterations) and a few small/medium configs, GPU vs the
reference CPU library on the host cores."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2202_01753_b200 as M

ctx = M.Context(0)
rows = []
for fam, d, mc, itmax, ita in [(4, 5, 10**6, 10, 10), (4, 8, 10**7, 10, 10), (4, 8, 10**8, 5, 3), (5, 8, 10**7, 30, 10)]:
    cfg = M.RunConfig(dims=d, maxcalls=mc, itmax=itmax, ita=ita, tau_rel=1e-12 if fam == 4 else 1e-3, seed=1,
                      lower=[0.0] * d, upper=[1.0] * d)
    f = M.make_suite_integrand(fam, d)
    M.integrate(f, cfg, ctx=ctx)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = M.integrate(f, cfg, ctx=ctx); ts.append(time.perf_counter() - t0)
    gpu = min(ts)
    t0 = time.perf_counter()
    o = O.integrate("ref", fam, None, d, 50, mc, itmax, ita, cfg.tau_rel, 1.5, 1.5, 1, 0, [0.0] * d, [1.0] * d,
                    workers=os.cpu_count())
    cpu = time.perf_counter() - t0
    rows.append(dict(integrand=f"f{fam}", dims=d, maxcalls=mc, iterations=r.iterations_used,
                     evals=r.total_samples, gpu_ms=gpu * 1e3, cpu_ms=cpu * 1e3, cpu_threads=os.cpu_count(),
                     speedup=cpu / gpu, gpu_est=r.estimate, cpu_est=o["estimate"], same_iterations=r.iterations_used == o["iterations_used"]))
    print(json.dumps(rows[-1]), flush=True)
