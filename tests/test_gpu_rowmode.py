"""GPU: K1's row-mode work mapping and the 64-bit cube-index regime against
the reference, bit for bit.

K1 walks whole rows along axis 0 once there are >= 2^20 rows (m / g); every
shape of >= 1e8 calls at 8D -- including the bench headline, 8D at maxcalls
1e9 (m = 12^8) -- runs that mapping, and maxcalls 1e10 at 8D (m = 16^8 = 2^32)
crosses the 32-bit cube index.  These tests compare those shapes with:

* the UNMODIFIED reference (oracle/_ref, v_sample on all host threads) on the
  compat stream: estimate, variance, all d x n_bins contribution cells and
  the device-counted write count, bitwise (f2 uses + - * / only), on a grid
  the reference itself adapted;
* the C twin of the Philox path (oracle/mcubes_oracle.c run_cube_philox,
  threaded over contiguous cube ranges) on row-mode shapes at 3D..8D.

Reference call sites: sampler.hpp:312-333 (v_sample), sampler.hpp:339-349
(v_sample_no_adjust), sampler.hpp:116-119 (the write count), the reference's
own invariance test tests/test_oracle.cpp:80-112.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
import paper_2202_01753_b200 as M
from conftest import bits, same_bits

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

THREADS = os.cpu_count() or 1
ROW_MIN = 1 << 20  # engine.cuh row_mode(): m / g >= 2^20


def _shape(d, maxcalls):
    sp = M.setup(M.RunConfig(dims=d, maxcalls=maxcalls, lower=[0.0] * d, upper=[1.0] * d))
    assert sp.m // sp.g >= ROW_MIN, "not a row-mode shape"
    return sp


def _ref_grid(fam, d, its=3):
    """A grid adapted by the reference itself (integrate at 1e6 calls)."""
    o = O.integrate("ref", fam, None, d, 50, 10 ** 6, its, its, 1e-15, 1.5, 1.5, 3, 0, [0.0] * d, [1.0] * d,
                    workers=THREADS, want_grids=True)
    return o["grids"][-1]


def _gpu(ctx, fam, d, edges, sp, seed, it, mode="all", rng="compat"):
    """rng: compat | philox (24-bit bin addends) | philox_exact (exact bins)."""
    f = M.make_suite_integrand(fam, d)
    g = M.Grid.from_edges(d, 50, [0.0] * d, [1.0] * d, edges)
    stream, bins = ("philox", "exact") if rng == "philox_exact" else (rng, "")
    if mode == "frozen":
        r = M.v_sample_no_adjust(f, g, sp.m, 1, sp.p, seed, it, rng=stream, ctx=ctx)
        return r.raw_estimate, r.raw_variance, None, None
    bu = M.BinUpdate.axis0_only if mode == "axis0" else M.BinUpdate.all_axes
    r = M.v_sample(f, g, sp.m, 1, sp.p, seed, it, bu, rng=stream, bins=bins, ctx=ctx)
    return r.raw_estimate, r.raw_variance, r.contributions.values, r.contributions.writes()


def _check(got, want, d, sp, mode="all"):
    est, var, contrib, writes = got
    assert bits(est) == bits(want["est"]), (est, want["est"])
    assert bits(var) == bits(want["var"]), (var, want["var"])
    if mode != "frozen":
        assert same_bits(contrib, want["contrib"])
        # device-counted deposits: every cube visited exactly once, p samples each
        assert writes == want["writes"] == sp.m * sp.p * (d if mode == "all" else 1)


@pytest.mark.parametrize("maxcalls", [10 ** 8, 10 ** 9])
def test_row_mode_compat_8d_bitwise_vs_reference(ctx, maxcalls):
    d = 8
    sp = _shape(d, maxcalls)  # 1e8: m = 9^8; 1e9: m = 12^8 (the bench headline's shape)
    edges = _ref_grid(2, d)
    got = _gpu(ctx, 2, d, edges, sp, 5, 4)
    want = O.v_sample("ref", 2, None, d, 50, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 5, 4, "all", THREADS)
    _check(got, want, d, sp)


def test_row_mode_compat_8d_2pow32_cubes_bitwise_vs_reference(ctx):
    """maxcalls 1e10 at 8D: m = 16^8 = 2^32 cubes -- cube indices past 32 bits
    (8.6e9 reference evaluations, ~50 s on the host cores)."""
    d = 8
    sp = _shape(d, 10 ** 10)
    assert sp.m == 1 << 32
    edges = _ref_grid(2, d)
    got = _gpu(ctx, 2, d, edges, sp, 11, 2)
    want = O.v_sample("ref", 2, None, d, 50, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 11, 2, "all", THREADS)
    _check(got, want, d, sp)


@pytest.mark.parametrize("d,maxcalls,mode", [(4, 3 * 10 ** 8, "axis0"), (4, 3 * 10 ** 8, "frozen"),
                                             (3, 2_200_000_000, "all"), (5, 8 * 10 ** 7, "all")])
def test_row_mode_compat_modes_bitwise_vs_reference(ctx, d, maxcalls, mode):
    sp = _shape(d, maxcalls)  # 4D: g = 110; 3D: g = 1032 (rows = g^2 >= 2^20); 5D: g = 33
    edges = _ref_grid(2, d)
    got = _gpu(ctx, 2, d, edges, sp, 3, 7, mode)
    want = O.v_sample("ref", 2, None, d, 50, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 3, 7, mode, THREADS)
    _check(got, want, d, sp, mode)


@pytest.mark.parametrize("rng", ["philox", "philox_exact"])
@pytest.mark.parametrize("d,maxcalls", [(8, 10 ** 8), (5, 8 * 10 ** 7), (4, 3 * 10 ** 8), (6, 2 * 10 ** 8)])
def test_row_mode_philox_bitwise_vs_c_twin(ctx, d, maxcalls, rng):
    """The north-star Philox path in row mode against its threaded C twin,
    with 24-bit and with exact bin addends."""
    sp = _shape(d, maxcalls)
    edges = _ref_grid(2, d)
    got = _gpu(ctx, 2, d, edges, sp, 9, 3, rng=rng)
    want = O.v_sample("orc", 2, None, d, 50, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 9, 3, "all", THREADS,
                      rng=rng)
    _check(got, want, d, sp)


def test_row_mode_transcendental_close_to_reference(ctx):
    """f4 (libdevice exp vs glibc) in row mode at the headline shape: within
    the stated ulp tolerance of the reference (tests/test_gpu_sampler.py)."""
    d = 8
    sp = _shape(d, 10 ** 9)
    edges = _ref_grid(4, d)
    est, var, contrib, writes = _gpu(ctx, 4, d, edges, sp, 1, 2)
    want = O.v_sample("ref", 4, None, d, 50, [0.0] * d, [1.0] * d, edges, sp.m, sp.s, sp.p, 1, 2, "all", THREADS)
    assert abs(est - want["est"]) <= 1e-12 * abs(want["est"]) + 1e-9 * np.sqrt(want["var"])
    assert abs(var - want["var"]) <= 1e-10 * want["var"]
    np.testing.assert_allclose(contrib, want["contrib"], rtol=1e-13, atol=0)
    assert writes == want["writes"] == sp.m * sp.p * d
