"""GPU: the real multi-rank path (paper_2202_01753_b200.dist.integrate) with
two processes.  The round's GPU boxes have one GPU, so both ranks share
cuda:0 and the exchange buffer (a CUDA int64 tensor) is all-reduced over
gloo; on an 8xB200 box the same code runs over NCCL.  Every rank must hold
the same result, bitwise equal to the single-process run."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

D, MAXCALLS = 6, 2 * 10 ** 6


def _cfg(M, early=False):
    if early is True:  # converges at iteration 2 of 12: the ranks must leave the loop together
        return M.RunConfig(dims=D, maxcalls=MAXCALLS, itmax=12, ita=6, tau_rel=2e-2, seed=13, lower=[0.0] * D,
                           upper=[1.0] * D, rng="philox")
    return M.RunConfig(dims=D, maxcalls=MAXCALLS, itmax=6, ita=4, tau_rel=1e-15, seed=13, lower=[0.0] * D,
                       upper=[1.0] * D)


FAMILY = {False: 4, True: 5, "resume": 4}


def _checkpoint(M, k):
    """Grid and history after k iterations of the uninterrupted single-process run."""
    grids = []
    cfg = _cfg(M)
    part = M.integrate(M.make_suite_integrand(4, D), M.RunConfig(**{**cfg.__dict__, "itmax": k, "ita": min(k, cfg.ita)}),
                       observer=lambda v: grids.append(v.grid))
    return M.Checkpoint(grids[-1], part.history)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q, early):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2202_01753_b200 as M
        from paper_2202_01753_b200 import dist as mdist

        torch.cuda.set_device(0)
        resume = _checkpoint(M, 3) if early == "resume" else None
        r = mdist.integrate(M.make_suite_integrand(FAMILY[early], D), _cfg(M, early), resume=resume)
        q.put((rank, r.estimate, r.sigma, r.chi2_dof, [h.estimate for h in r.history],
               [h.variance for h in r.history], r.converged, r.iterations_used))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,early", [(2, False), (3, False), (2, True), (2, "resume")])
def test_multi_rank_integrate_matches_single(world, early, ctx):
    import paper_2202_01753_b200 as M

    want = M.integrate(M.make_suite_integrand(FAMILY[early], D), _cfg(M, early), ctx=ctx)
    if early is True:
        assert want.converged and want.iterations_used < 12
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_rank, args=(r, world, port, q, early)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, est, sigma, chi2, he, hv, conv, used in res:
        assert conv == want.converged and used == want.iterations_used
        assert est == want.estimate and sigma == want.sigma and chi2 == want.chi2_dof
        assert he == [h.estimate for h in want.history] and hv == [h.variance for h in want.history]


def _nf_cfg(M):
    # 2D, g = 70: inf_near_origin(0.014) fails only inside corner cube 0, which
    # lies in rank 0's slice (n = 0 maps to cube 0); the other ranks see no failure
    return M.RunConfig(dims=2, maxcalls=10 ** 4, itmax=4, ita=2, tau_rel=1e-15, seed=5, lower=[0.0] * 2,
                       upper=[1.0] * 2)


def _nf_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2202_01753_b200 as M
        from paper_2202_01753_b200 import dist as mdist

        torch.cuda.set_device(0)
        try:
            mdist.integrate(M.test_integrand("inf_near_origin", 2, 0.014), _nf_cfg(M))
            q.put((rank, None, None))
        except M.NonFiniteSample as e:
            q.put((rank, e.point(), e.value()))
    finally:
        dist.destroy_process_group()


def test_nonfinite_in_one_rank_stops_every_rank(ctx):
    """A non-finite sample in one rank's slice: every rank stops at the same
    iteration (the failure count travels with the exchange words) and raises
    the same NonFiniteSample as the single-process run (the first failing
    sample in serial order, min-reduced over the ranks)."""
    import paper_2202_01753_b200 as M

    with pytest.raises(M.NonFiniteSample) as ei:
        M.integrate(M.test_integrand("inf_near_origin", 2, 0.014), _nf_cfg(M), ctx=ctx)
    want = (ei.value.point(), ei.value.value())
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    world = 2
    procs = [mpc.Process(target=_nf_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, point, value in res:
        assert (point, value) == want


def test_peer_exchange_virtual_ranks_match_single(ctx):
    """The peer-memory exchange's device path (system-scope reductions into
    every rank's buffer, release/acquire flags, odd/even buffers) with two
    ranks in one process on one GPU: each rank's K1 writes both ranks'
    buffers, each finish waits for both flags.  The kernels of the two ranks
    are separated by device synchronisations (on one GPU a spinning finish
    must not hold SMs the other rank's K1 needs)."""
    import ctypes as C

    import paper_2202_01753_b200 as M
    from paper_2202_01753_b200 import _lib as L
    from paper_2202_01753_b200 import dist as mdist

    for early in (False, True):
        cfg = _cfg(M, early)
        f = M.make_suite_integrand(FAMILY[early], D)
        want = M.integrate(f, cfg, ctx=ctx)
        lib = L.lib()
        ctxs = [M.Context(0), M.Context(0)]
        runs = [M.Run(f, cfg, c) for c in ctxs]
        words = runs[0].exchange_words()

        def alloc(n):
            out = C.c_void_p()
            assert lib.mcb_dev_alloc(ctxs[0].ptr, n, C.byref(out)) == 0
            return out.value

        odd, even, flags, counters = [alloc(8 * words) for _ in range(2)], [alloc(8 * words) for _ in range(2)], \
            [alloc(16) for _ in range(2)], [alloc(4) for _ in range(2)]
        for r in range(2):
            runs[r].set_peers(r, 2, odd, even, flags, counters[r])
        m = runs[0].work_items
        torch.cuda.synchronize()
        for it in range(1, cfg.itmax + 1):
            for r in range(2):
                runs[r].sample(it, *mdist.partition(m, 2, r))
            torch.cuda.synchronize()
            for r in range(2):
                runs[r].finish(it)
            torch.cuda.synchronize()
        got = [run.result() for run in runs]
        for run in runs:
            run.close()
        for p in odd + even + flags + counters:
            lib.mcb_dev_free(ctxs[0].ptr, C.c_void_p(p))
        for g in got:
            assert g.iterations_used == want.iterations_used and g.converged == want.converged
            assert g.estimate == want.estimate and g.sigma == want.sigma and g.chi2_dof == want.chi2_dof
            assert [h.estimate for h in g.history] == [h.estimate for h in want.history]


def _peer_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2202_01753_b200 as M
        from paper_2202_01753_b200 import dist as mdist

        torch.cuda.set_device(0)
        r = mdist.integrate(M.make_suite_integrand(FAMILY[False], D), _cfg(M, False), transport="peer")
        q.put((rank, r.estimate, r.sigma, r.chi2_dof, [h.estimate for h in r.history], r.iterations_used))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_two_processes(ctx):
    """dist.integrate(transport="peer"): two processes share their exchange
    buffers and flags through CUDA IPC (here both on cuda:0, time-sliced;
    on an NVLink box each on its own GPU) and agree bitwise with the
    single-process run, with no collective inside the iteration loop."""
    import paper_2202_01753_b200 as M

    want = M.integrate(M.make_suite_integrand(FAMILY[False], D), _cfg(M, False), ctx=ctx)
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_peer_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, est, sigma, chi2, he, used in res:
        assert used == want.iterations_used
        assert est == want.estimate and sigma == want.sigma and chi2 == want.chi2_dof
        assert he == [h.estimate for h in want.history]
