"""Multi-GPU m-Cubes over torch.distributed (NCCL over NVLink).

One process per GPU.  Every rank runs the same device-resident iteration
loop; rank r samples the contiguous slice ``partition(m, world, r)`` of the
linear work index, then the exchange buffer -- est+/est-/var and the
d x n_bins contribution superaccumulators as unnormalised uint64 digit sums
(include/mcubes_b200.h, MCB_XWORDS words each) -- is all-reduced with a plain
integer SUM.  Integer sums are associative, so the all-reduce is exact and
every rank rounds, adapts the grid and updates the weighted estimate on
device to bit-identical values: results are independent of the GPU count and
equal to the single-GPU (and reference) result.  This replaces the
reference's in-process exact merge of per-worker partials
(sampler.hpp:272-276).
"""
from __future__ import annotations

from typing import Optional

from . import mcubes as M


def partition(m: int, world: int, rank: int):
    """Contiguous slice [n0, n1) of the linear work index for `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("partition: need 0 <= rank < world")
    return rank * m // world, (rank + 1) * m // world


def integrate(f: M.IntegrandSpec, cfg: M.RunConfig, group=None, ctx: Optional[M.Context] = None,
              observer=None, resume: Optional[M.Checkpoint] = None) -> M.IntegrationResult:
    """integrate() across the ranks of `group` (default: WORLD).  Every rank
    returns the same IntegrationResult.  `resume` continues from a checkpoint
    (every rank passes the same one)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    if stream.cuda_stream == 0:  # keep the library, NCCL and torch on one explicit stream
        stream = torch.cuda.Stream(dev)
    ctx = ctx or M.Context(dev.index)
    ctx.set_stream(stream.cuda_stream)
    # Bounded lookahead (as the single-GPU integrate): at most `ahead`
    # iterations in flight; stop enqueuing once the device reports the run
    # stopped through host-mapped progress flags.  The flags are identical on
    # every rank (the state is), so all ranks leave the loop together.
    ahead = 2
    flags = torch.zeros(cfg.itmax, dtype=torch.int32).pin_memory()
    events = [torch.cuda.Event() for _ in range(ahead + 1)]
    with torch.cuda.stream(stream):
        run = M.Run(f, cfg, ctx)
        run.set_progress(flags.data_ptr())
        n0, n1 = partition(run.work_items, world, rank)
        xbuf = torch.zeros(run.exchange_words(), dtype=torch.int64, device=dev)
        run.set_exchange(xbuf.data_ptr())
        first = run.resume(resume) if resume is not None else 1
        if first > 1 and run.result().converged:
            res = run.result()
            run.close()
            return res
        for it in range(first, cfg.itmax + 1):
            if observer is None and it >= first + ahead:
                events[(it - ahead) % (ahead + 1)].synchronize()
                if int(flags[it - ahead - 1]) != 1:
                    break
            run.sample(it, n0, n1)
            run.reduce(it)
            # exact integer sum across ranks, of the words this iteration uses
            # (frozen iterations: the count word and est+/est-/var only)
            dist.all_reduce(xbuf[:run.exchange_words(it)], group=group)
            run.finish(it)
            events[it % (ahead + 1)].record(stream)
            if observer is not None:
                r = run.result()
                if r.iterations_used < it:
                    break
                observer(it, r, run.grid())
        # A non-finite sample in any rank's slice stops every rank at the same
        # iteration (its count is exchanged with the words); report the first
        # one in serial order over all slices, as a single process would.
        failed, key = run.failure_key()
        if failed:
            k = torch.tensor([key - (1 << 63)], dtype=torch.int64, device=dev)  # u64 order in int64
            dist.all_reduce(k, op=dist.ReduceOp.MIN, group=group)
            run.set_failure_key(int(k.item()) + (1 << 63))
        try:
            res = run.result()
        finally:
            run.close()
    return res
