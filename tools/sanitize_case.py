"""Small-shape workload for compute-sanitizer (memcheck / racecheck /
synccheck): adjusting + frozen iterations on both streams, 2D..8D, the
integrate() loop with its finish kernel, the peer-memory exchange (two
virtual ranks), and a non-finite sample."""
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
    # runtime n_bins (grid-table copies chosen at launch) and bin passes
    # (8D at 200 bins: the histograms of all axes exceed one CTA)
    for d, nb, m in ((3, 100, 12 ** 3), (8, 200, 2 ** 8)):
        g = M.Grid(d, nb, [0.0] * d, [1.0] * d)
        M.v_sample(M.make_suite_integrand(4, d), g, m, 1, 3, 1, 1, rng=rng, ctx=ctx)
# Philox with exact bins
g = M.Grid(5, 50, [0.0] * 5, [1.0] * 5)
M.v_sample(M.make_suite_integrand(4, 5), g, 5 ** 5, 1, 2, 1, 1, rng="philox", bins="exact", ctx=ctx)
# the peer-memory exchange (two virtual ranks on this GPU, phases separated by device syncs)
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2202_01753_b200 import _lib as L  # noqa: E402
from paper_2202_01753_b200 import dist as mdist  # noqa: E402

lib = L.lib()
cfg = M.RunConfig(dims=3, maxcalls=20000, itmax=3, ita=2, tau_rel=1e-12, lower=[0.0] * 3, upper=[1.0] * 3, rng="philox")
ctxs = [M.Context(0), M.Context(0)]
runs = [M.Run(M.make_suite_integrand(4, 3), cfg, c) for c in ctxs]


def _alloc(n):
    out = C.c_void_p()
    assert lib.mcb_dev_alloc(ctxs[0].ptr, n, C.byref(out)) == 0
    return out.value


nw = runs[0].exchange_words()
odd, even, flags, cnt = [_alloc(8 * nw) for _ in range(2)], [_alloc(8 * nw) for _ in range(2)], \
    [_alloc(16) for _ in range(2)], [_alloc(4) for _ in range(2)]
for r in range(2):
    runs[r].set_peers(r, 2, odd, even, flags, cnt[r])
torch.cuda.synchronize()
for it in range(1, cfg.itmax + 1):
    for r in range(2):
        runs[r].sample(it, *mdist.partition(runs[r].work_items, 2, r))
    torch.cuda.synchronize()
    for r in range(2):
        runs[r].finish(it)
    torch.cuda.synchronize()
assert runs[0].result().estimate == runs[1].result().estimate
for run in runs:
    run.close()
for ptr in odd + even + flags + cnt:
    lib.mcb_dev_free(ctxs[0].ptr, C.c_void_p(ptr))
try:
    M.v_sample(M.test_integrand("inf_if_x0_pos", 1), M.Grid(1, 4, [0.0], [1.0]), 4, 1, 2, 1, 1, ctx=ctx)
except M.NonFiniteSample:
    pass
print("sanitize case done")
