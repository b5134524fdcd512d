"""CPU, world_size 2 over gloo: the multi-GPU exchange semantics.

Each rank samples its slice of the linear work index (dist.partition, the
product's partition), produces the exchange buffer in the GPU format (uint64
radix-2^32 digit sums, MCB_XWORDS per accumulator), the buffers are
all-reduced with an integer SUM (what NCCL does between GPUs), and every rank
rounds and adapts independently.  The oracle stands in for the per-rank
kernel; the test checks that the decomposition is exact: identical results on
every rank and bitwise equal to the single-process run, for a full
multi-iteration integrate trajectory.
"""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2202_01753_b200.dist import partition

        d, nb, fam, p, seed = 4, 20, 4, 3, 17
        g = 5
        m = g ** d
        lo, hi = [0.0] * d, [1.0] * d
        W = O.XWORDS
        edges = O.uniform_edges(d, nb, lo, hi)
        hist_e, hist_v, grids = [], [], []
        n0, n1 = partition(m, world, rank)
        for it in range(1, 5):
            nacc = 3 + d * nb
            words = np.zeros(nacc * W, dtype=np.uint64)
            # rank's slice in cube-index space: contiguous cubes [n0, n1) (exactness makes the split free)
            rc = O.orc().orc_sample_partial(fam, None, 0, d, nb, O.darr(lo), O.darr(hi), O.ptr(edges), m, p, seed, it,
                                            0, 1, n0, n1, words.ctypes.data_as(C.POINTER(C.c_uint64)), None, None,
                                            None)
            assert rc == 0
            t = torch.from_numpy(words.view(np.int64).copy())
            dist.all_reduce(t)  # exact integer sum across ranks
            words = t.numpy().view(np.uint64).copy()
            est, var = C.c_double(), C.c_double()
            contrib = np.zeros(d * nb)
            O.orc().orc_round_partial(words.ctypes.data_as(C.POINTER(C.c_uint64)), d, nb, m, 0, 1, C.byref(est),
                                      C.byref(var), O.ptr(contrib))
            out = np.zeros(d * nb)
            assert O.orc().orc_grid_adjust(d, nb, O.darr(lo), O.darr(hi), O.ptr(edges), O.ptr(contrib), 1.5, 0,
                                           O.ptr(out)) == 0
            edges = out
            hist_e.append(est.value)
            hist_v.append(var.value)
            grids.append(edges.copy())
        q.put((rank, hist_e, hist_v, [g_.tobytes() for g_ in grids]))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_is_exact():
    import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    res.sort()
    (_, e0, v0, g0), (_, e1, v1, g1) = res
    assert e0 == e1 and v0 == v1 and g0 == g1  # every rank holds identical state

    # single-process reference trajectory (same integrand, grid schedule)
    d, nb = 4, 20
    r = O.integrate("orc", 4, None, d, nb, 1900, 4, 4, 1e-15, 1.5, 1.5, 17, 0, [0.0] * d, [1.0] * d,
                    want_grids=True)
    assert r["m"] == 5 ** 4 and r["p"] == 3
    assert list(r["hist_est"]) == e0 and list(r["hist_var"]) == v0
    assert [g.tobytes() for g in r["grids"]] == g0


class _FakePeerMemory:
    """Stand-in for the CUDA allocation / IPC calls of dist.PeerExchange: a
    'pointer' is 1000 * (rank + 1) + index and its 'handle' encodes the same
    number, so every rank can check the table it assembles."""

    def __init__(self, rank):
        self.rank, self.n, self.log = rank, 0, []

    def alloc(self, nbytes):
        self.n += 1
        p = 1000 * (self.rank + 1) + self.n
        self.log.append(("alloc", p, nbytes))
        return p

    def handle(self, ptr):
        return ptr.to_bytes(8, "little") + bytes(56)

    def open(self, handle):
        assert len(handle) == 64
        p = int.from_bytes(handle[:8], "little")
        self.log.append(("open", p))
        return p

    def close(self, ptr):
        self.log.append(("close", ptr))

    def free(self, ptr):
        self.log.append(("free", ptr))


def _peer_table_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_01753_b200.dist import PeerExchange

        mem = _FakePeerMemory(rank)
        px = PeerExchange(None, words=1 + 67 * 3, group=None, memory=mem)
        tables = (px.bufs_odd, px.bufs_even, px.flags, px.counter, px.rank, px.world)
        px.close()
        q.put((rank, tables, mem.log))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_host_tables():
    """dist.PeerExchange (the transport='peer' setup) over gloo with world
    size 3: every rank assembles the same per-rank pointer tables (its own
    allocations in its own slot, the others' opened from their handles),
    sized buffers, and on close unmaps what it opened and frees what it
    allocated."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_table_rank, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    want_odd = [1000 * (r + 1) + 1 for r in range(world)]
    want_even = [1000 * (r + 1) + 2 for r in range(world)]
    want_flags = [1000 * (r + 1) + 3 for r in range(world)]
    for rank, (odd, even, flags, counter, rk, w), log in res:
        assert rk == rank and w == world
        assert odd == want_odd and even == want_even and flags == want_flags
        assert counter == 1000 * (rank + 1) + 4
        allocs = [e for e in log if e[0] == "alloc"]
        assert [a[2] for a in allocs] == [8 * (1 + 67 * 3), 8 * (1 + 67 * 3), 8 * world, 4]
        opened = sorted(e[1] for e in log if e[0] == "open")
        closed = sorted(e[1] for e in log if e[0] == "close")
        assert opened == closed and len(opened) == 3 * (world - 1)
        assert all(p // 1000 != rank + 1 for p in opened)
        assert sorted(e[1] for e in log if e[0] == "free") == sorted(a[1] for a in allocs)


def _compact_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2202_01753_b200.dist import all_gather_rank_major, partition

        # each rank's rounded slice in the compact layout (est, var, 4 counts, contributions)
        d, nb, fam, p, seed, g = 3, 10, 2, 3, 5, 7
        m = g ** d
        lo, hi = [0.0] * d, [1.0] * d
        edges = O.uniform_edges(d, nb, lo, hi)
        n0, n1 = partition(m, world, rank)
        words = np.zeros((3 + d * nb) * O.XWORDS, dtype=np.uint64)
        assert O.orc().orc_sample_partial(fam, None, 0, d, nb, O.darr(lo), O.darr(hi), O.ptr(edges), m, p, seed, 1,
                                          0, 1, n0, n1, words.ctypes.data_as(C.POINTER(C.c_uint64)), None, None,
                                          None) == 0
        est, var = C.c_double(), C.c_double()
        contrib = np.zeros(d * nb)
        O.orc().orc_round_partial(words.ctypes.data_as(C.POINTER(C.c_uint64)), d, nb, m, 0, 1, C.byref(est),
                                  C.byref(var), O.ptr(contrib))
        counts = np.array([(n1 - n0) * p, (n1 - n0) * p * d, 0, 0], dtype=np.uint64).view(np.float64)
        mine = torch.from_numpy(np.concatenate([[est.value, var.value], counts, contrib]))
        every = torch.zeros(world * mine.numel(), dtype=torch.float64)
        all_gather_rank_major(every, mine)
        q.put((rank, mine.numpy().tobytes(), every.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_compact_exchange_gathers_rank_major():
    """dist.all_gather_rank_major (transport='compact') over gloo, world 3:
    every rank receives every rank's rounded slice at offset rank * len, and
    the combine that Run.combine performs on the device -- the per-rank values
    added in rank order -- gives one result on every rank, within the partial
    sums' rounding of the single-process iteration."""
    import oracle as O

    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_compact_rank, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    mines = [np.frombuffer(r[1], dtype=np.float64) for r in res]
    for _, _, ev in res:
        assert np.array_equal(np.frombuffer(ev, dtype=np.float64).view(np.uint64),
                              np.concatenate(mines).view(np.uint64))
    est = mines[0][0]
    for r in range(1, world):
        est = est + mines[r][0]
    d, nb = 3, 10
    want = O.v_sample("orc", 2, None, d, nb, [0.0] * d, [1.0] * d, None, 7 ** d, 1, 3, 5, 1)
    assert abs(est - want["est"]) <= 1e-14 * abs(want["est"])
    assert sum(int(m_[2:6].view(np.uint64)[0]) for m_ in mines) == want["writes"] // d
