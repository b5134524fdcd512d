"""GPU: device grid adaptation (Grid::adjusted / adjusted_symmetric,
grid.hpp:104-146, 232-297) against the reference, plus the reference's own
grid tests (tests/test_grid.cpp:180-300).  The device uses libdevice pow/log
where the reference uses glibc, so edges agree to 1e-13 relative (typically
bitwise); structural properties are exact."""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2202_01753_b200 as M
from conftest import h2a, same_bits

pytestmark = pytest.mark.gpu


def uniform(d, nb, lo, hi):
    return M.Grid(d, nb, [lo] * d, [hi] * d)


def test_golden_adjust(golden, ctx):
    nbit = ntot = 0
    for c in golden["adjust"]:
        d, nb = c["dims"], c["n_bins"]
        g = M.Grid.from_edges(d, nb, list(h2a(c["lower"])), list(h2a(c["upper"])), h2a(c["edges"]))
        contrib = h2a(c["contrib"])
        out = g.adjusted_symmetric(contrib[:nb], c["alpha"], ctx=ctx) if c["symmetric"] else \
            g.adjusted(contrib, c["alpha"], ctx=ctx)
        want = h2a(c["out"])
        np.testing.assert_allclose(out.raw_edges, want, rtol=1e-13, atol=1e-15)
        nbit += int(np.sum(out.raw_edges.view(np.uint64) == want.view(np.uint64)))
        ntot += want.size
        for j in range(d):  # invariants hold exactly
            e = out.edges(j)
            assert np.all(np.diff(np.concatenate([[out.lower(j)], e])) > 0) and e[-1] == out.upper(j)
    assert nbit / ntot > 0.5  # most edges are bit-identical


def test_fixed_point_and_shrink(ctx):
    g = uniform(2, 8, 0.0, 2.0)
    a = g.adjusted(np.full(16, 3.25), 1.5, ctx=ctx)
    np.testing.assert_allclose(a.raw_edges, g.raw_edges, atol=1e-12)
    g = uniform(1, 4, 0.0, 1.0)
    a = g.adjusted(np.array([1.0, 0, 0, 0]), 1.5, ctx=ctx)
    assert a.edges(0)[0] < 0.25 and a.edges(0)[3] == 1.0
    g = uniform(1, 2, 0.0, 1.0)
    a = g.adjusted(np.array([1.0, 0.0]), 1.5, ctx=ctx)
    assert abs(a.edges(0)[0] - 0.5) < 1e-12


def test_zero_axis_untouched_and_alpha0(ctx):
    g = uniform(2, 4, 0.0, 1.0)
    c = np.zeros(8)
    c[7] = 2.0
    a = g.adjusted(c, 1.5, ctx=ctx)
    assert same_bits(a.edges(0), g.edges(0)) and a.edges(1)[2] > g.edges(1)[2]
    g = uniform(1, 6, 0.0, 1.0)
    a = g.adjusted(np.arange(1.0, 7.0), 0.0, ctx=ctx)
    np.testing.assert_allclose(a.raw_edges, g.raw_edges, atol=1e-12)


def test_invalid_contributions(ctx):
    g = uniform(1, 4, 0.0, 1.0)
    with pytest.raises(ValueError):
        g.adjusted(M.BinAccumulator(1, 5), 1.5, ctx=ctx)
    with pytest.raises(ValueError):
        g.adjusted(np.array([0.0, -1.0, 0.0, 0.0]), 1.5, ctx=ctx)
    with pytest.raises(ValueError):
        g.adjusted(np.array([0.0, np.nan, 0.0, 0.0]), 1.5, ctx=ctx)
    with pytest.raises(ValueError):
        g.adjusted(np.zeros(4), -1.0, ctx=ctx)


def test_repeated_adjustment_invariants(ctx):
    rng = np.random.default_rng(17)
    g = uniform(3, 10, -2.0, 3.0)
    for _ in range(20):
        g = g.adjusted(rng.uniform(0.0, 5.0, 30), 1.5, ctx=ctx)
        for j in range(3):
            e = np.concatenate([[g.lower(j)], g.edges(j)])
            assert np.all(np.diff(e) > 0) and g.edges(j)[-1] == 3.0
            assert math.isclose(np.sum(np.diff(e)), 5.0, rel_tol=1e-12)


def test_symmetric(ctx):
    g = uniform(3, 8, 0.0, 1.0)
    contrib = [5.0, 3.0, 1.0, 0.5, 0.25, 0.5, 3.0, 7.0]
    a = g.adjusted_symmetric(contrib, 1.5, ctx=ctx)
    for j in (1, 2):
        assert same_bits(a.edges(j), a.edges(0))
    b = g.adjusted(np.tile(contrib, 3), 1.5, ctx=ctx)
    assert same_bits(a.raw_edges, b.raw_edges)
    g = M.Grid(2, 6, [0.0, -2.0], [1.0, 4.0])
    a = g.adjusted_symmetric([4.0, 2.0, 1.0, 1.0, 2.0, 4.0], 1.5, ctx=ctx)
    np.testing.assert_allclose((a.edges(1) + 2.0) / 6.0, a.edges(0), rtol=1e-12)
    assert a.edges(1)[5] == 4.0
