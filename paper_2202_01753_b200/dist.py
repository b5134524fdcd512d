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

transport="compact" is SURVEY.md section 8(e)'s exchange: every rank rounds
its own slice to d x n_bins + 2 doubles (plus the counts), the ranks
all-gather them (3.2 KB per rank at 8D instead of 216 KB), and every rank
sums them in rank order on the device and runs the epilogue: identical state
on every rank, last bits dependent on the GPU count (one rank is bitwise the
exact path).

transport="peer" replaces the all-reduce by the sampling kernel itself:
its blocks add their words into every rank's buffer over peer memory (CUDA
IPC mappings, system-scope reductions) and release a per-iteration flag that
every rank's finish kernel acquires (PeerExchange below).
"""
from __future__ import annotations

from typing import Optional

from . import mcubes as M


def all_gather_rank_major(every, mine, group=None):
    """every[r * len(mine):(r + 1) * len(mine)] = rank r's `mine` (NCCL: one
    all_gather_into_tensor; gloo, which lacks it: the list form)."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(every, mine, group=group)
    else:
        dist.all_gather(list(every.view(-1, mine.numel()).unbind(0)), mine, group=group)


def partition(m: int, world: int, rank: int):
    """Contiguous slice [n0, n1) of the linear work index for `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("partition: need 0 <= rank < world")
    return rank * m // world, (rank + 1) * m // world


class _CudaPeerMemory:
    """Device allocation and CUDA IPC through the library (mcb_dev_alloc,
    mcb_ipc_handle / mcb_ipc_open / mcb_ipc_close, mcb_dev_free)."""

    def __init__(self, ctx: M.Context):
        from . import _lib as L

        self._lib, self.ctx = L.lib(), ctx

    def alloc(self, nbytes: int) -> int:
        import ctypes as C

        out = C.c_void_p()
        M._raise(self._lib.mcb_dev_alloc(self.ctx.ptr, nbytes, C.byref(out)), self.ctx.ptr)
        return out.value

    def handle(self, ptr: int) -> bytes:
        import ctypes as C

        h = C.create_string_buffer(64)
        M._raise(self._lib.mcb_ipc_handle(self.ctx.ptr, C.c_void_p(ptr), h), self.ctx.ptr)
        return h.raw

    def open(self, handle: bytes) -> int:
        import ctypes as C

        out = C.c_void_p()
        M._raise(self._lib.mcb_ipc_open(self.ctx.ptr, handle, C.byref(out)), self.ctx.ptr)
        return out.value

    def close(self, ptr: int):
        import ctypes as C

        self._lib.mcb_ipc_close(self.ctx.ptr, C.c_void_p(ptr))

    def free(self, ptr: int):
        import ctypes as C

        self._lib.mcb_dev_free(self.ctx.ptr, C.c_void_p(ptr))


class PeerExchange:
    """The peer-memory exchange's buffers for one run on this rank: two
    exchange buffers (odd / even iterations), a flag array and a block
    counter, allocated zeroed and shared with every rank of the group through
    IPC handles (all_gather_object).  Every rank ends up with every rank's
    pointers, indexed by rank: its own directly, the others' mapped (over
    NVLink on an HGX box).  `memory` supplies alloc/handle/open/close/free
    (the CUDA library by default; the CPU tests inject a stand-in)."""

    def __init__(self, ctx: Optional[M.Context], words: int, group=None, memory=None):
        import torch.distributed as dist

        self.mem = memory if memory is not None else _CudaPeerMemory(ctx)
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        if self.world > 8:
            raise ValueError("peer-memory exchange: at most 8 ranks")
        self.group = group
        # odd buffer, even buffer, flag array (one u64 slot per rank), block counter
        self.own = [self.mem.alloc(8 * words), self.mem.alloc(8 * words), self.mem.alloc(8 * self.world),
                    self.mem.alloc(4)]
        every = [None] * self.world
        dist.all_gather_object(every, [self.mem.handle(p) for p in self.own[:3]], group=group)
        self.opened = []
        table = []
        for q, hs in enumerate(every):
            if q == self.rank:
                table.append(self.own[:3])
                continue
            row = [self.mem.open(h) for h in hs]
            self.opened += row
            table.append(row)
        self.bufs_odd = [r[0] for r in table]
        self.bufs_even = [r[1] for r in table]
        self.flags = [r[2] for r in table]
        self.counter = self.own[3]

    def attach(self, run: M.Run):
        run.set_peers(self.rank, self.world, self.bufs_odd, self.bufs_even, self.flags, self.counter)

    def close(self):
        """Collective: unmap the peers' buffers, then free ours once every
        rank has unmapped them."""
        import torch.distributed as dist

        for p in self.opened:
            self.mem.close(p)
        self.opened = []
        dist.barrier(group=self.group)
        for p in self.own:
            self.mem.free(p)
        self.own = []


def integrate(f: M.IntegrandSpec, cfg: M.RunConfig, group=None, ctx: Optional[M.Context] = None,
              observer=None, resume: Optional[M.Checkpoint] = None, transport: str = "collective") -> M.IntegrationResult:
    """integrate() across the ranks of `group` (default: WORLD).  Every rank
    returns the same IntegrationResult.  `resume` continues from a checkpoint
    (every rank passes the same one).  transport="collective" all-reduces the
    exchange buffer through the process group (NCCL over NVLink);
    transport="peer" has K1 write every rank's buffer directly over peer
    memory (CUDA IPC, system-scope reductions and flags), with no collective
    inside the iteration loop."""
    if transport not in ("collective", "peer", "compact"):
        raise ValueError("transport must be 'collective', 'peer' or 'compact'")
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
        peers = None
        try:
            run.set_progress(flags.data_ptr())
            n0, n1 = partition(run.work_items, world, rank)
            if transport == "peer":
                torch.cuda.current_stream(dev).synchronize()
                peers = PeerExchange(ctx, run.exchange_words(), group)
                peers.attach(run)
            else:
                xbuf = torch.zeros(run.exchange_words(), dtype=torch.int64, device=dev)
                run.set_exchange(xbuf.data_ptr())
            if transport == "compact":
                mine = torch.zeros(run.compact_len(), dtype=torch.float64, device=dev)
                every = torch.zeros(world * run.compact_len(), dtype=torch.float64, device=dev)
            first = run.resume(resume) if resume is not None else 1
            if first > 1 and run.result().converged:
                return run.result()
            for it in range(first, cfg.itmax + 1):
                if observer is None and it >= first + ahead:
                    events[(it - ahead) % (ahead + 1)].synchronize()
                    if int(flags[it - ahead - 1]) != 1:
                        break
                run.sample(it, n0, n1)
                run.reduce(it)
                if transport == "compact":
                    run.round_local(it, mine.data_ptr())
                    all_gather_rank_major(every, mine, group)
                    run.combine(it, every.data_ptr(), world)
                    run.finish_rounded(it)
                else:
                    if peers is None:
                        # exact integer sum across ranks, of the words this iteration uses
                        # (frozen iterations: the count words and est+/est-/var only)
                        dist.all_reduce(xbuf[:run.exchange_words(it)], group=group)
                    run.finish(it)
                events[it % (ahead + 1)].record(stream)
                if observer is not None:
                    # a failed iteration stops here, before result() (which raises): the
                    # failure key is min-reduced over the ranks below first, as the C++
                    # loop does (`if (st.failed) break`)
                    if run.failure_key()[0]:
                        break
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
            return run.result()
        finally:
            run.close()
            if peers is not None:
                torch.cuda.current_stream(dev).synchronize()
                peers.close()
