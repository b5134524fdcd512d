"""Quick GPU-vs-oracle check used while bringing up the kernels."""
import struct, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2202_01753_b200 as M
import oracle as O

def bits(x): return hex(struct.unpack('<Q', struct.pack('<d', x))[0])

# golden triple (test_oracle.cpp:62-78)
g = M.Grid(1, 4, [0.0], [1.0])
r = M.v_sample(M.test_integrand('x0', 1), g, 4, 1, 2, 1, 0)
print('triple', bits(r.raw_estimate), bits(r.raw_variance), [bits(v) for v in r.contributions.values], r.contributions.writes())

for fam, d, maxcalls in [(2, 3, 100000), (4, 5, 1000000), (2, 8, 10**7), (4, 8, 10**7), (1, 6, 10**6), (5, 8, 10**6), (6, 4, 10**6), (3, 6, 10**6)]:
    cfg = M.RunConfig(dims=d, maxcalls=maxcalls, lower=[0.0]*d, upper=[1.0]*d)
    sp = M.setup(cfg)
    f = M.make_suite_integrand(fam, d)
    grid = M.Grid(d, 50, [0.0]*d, [1.0]*d)
    t = time.time()
    gr = M.v_sample(f, grid, sp.m, sp.s, sp.p, 3, 1)
    tg = time.time() - t
    t = time.time()
    orc = O.v_sample('orc', fam, None, d, 50, [0.0]*d, [1.0]*d, None, sp.m, 1, sp.p, 3, 1)
    to = time.time() - t
    ce = np.array_equal(gr.contributions.values, orc['contrib'])
    print(f"f{fam} d={d} m={sp.m} p={sp.p}: est {bits(gr.raw_estimate)} vs {bits(orc['est'])} eq={gr.raw_estimate==orc['est']} var eq={gr.raw_variance==orc['var']} contrib eq={ce} maxrel={np.max(np.abs(gr.contributions.values-orc['contrib'])/np.maximum(orc['contrib'],1e-300)):.2e} writes {gr.contributions.writes()}=={orc['writes']} gpu {tg:.3f}s orc {to:.2f}s")

# full integrate C1
cfg = M.RunConfig(dims=5, maxcalls=10**6, itmax=10, ita=10, tau_rel=1e-9, lower=[0.0]*5, upper=[1.0]*5)
t = time.time(); r = M.integrate(M.make_suite_integrand(4, 5), cfg); tg = time.time() - t
o = O.integrate('orc', 4, None, 5, 50, 10**6, 10, 10, 1e-9, 1.5, 1.5, 0, 0, [0]*5, [1]*5)
print('C1 gpu', repr(r.estimate), repr(r.sigma), repr(r.chi2_dof), r.iterations_used, f'{tg:.3f}s')
print('C1 orc', repr(o['estimate']), repr(o['sigma']), repr(o['chi2_dof']), o['iterations_used'])
print('hist eq', [a.estimate == b for a, b in zip(r.history, o['hist_est'])])
# README row
cfg = M.RunConfig(dims=3, maxcalls=100000, seed=7, lower=[0.0]*3, upper=[1.0]*3)
r = M.integrate(M.make_suite_integrand(2, 3), cfg)
print('README', repr(r.estimate), repr(r.sigma), repr(r.chi2_dof), r.iterations_used, r.total_samples, r.converged)
print('launches', M.default_context().launches)
