"""CPU: the C ABI surface and the host-side logic of the product (no kernel
launches): every symbol include/mcubes_b200.h declares is exported, and the
host utilities match the reference's hand-worked examples
(tests/test_driver.cpp, tests/test_grid.cpp, tests/test_integrands.cpp)."""
from __future__ import annotations

import math
import os
import re

import numpy as np
import pytest

import paper_2202_01753_b200 as M
from paper_2202_01753_b200 import _lib
from conftest import ROOT, bits, h2a, h2f, same_bits


def unit_cfg(d, maxcalls, **kw):
    return M.RunConfig(dims=d, maxcalls=maxcalls, lower=[0.0] * d, upper=[1.0] * d, workers=1, **kw)


def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "mcubes_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|uint64_t|void\s*\*|const char\s*\*)\s*(mcb_\w+)\s*\(", header, re.M))
    assert len(declared) >= 25
    lib = _lib.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    assert lib.mcb_abi_version() == 2


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null | head -5").read()
    assert "sm_100a" in out


def test_setup_examples():
    # test_driver.cpp:47-76
    assert M.setup(unit_cfg(2, 1000))[:3] == (22, 484, 2)
    assert M.setup(unit_cfg(2, 1000)).s == M.set_batch_size(484, 1)
    assert M.setup(unit_cfg(8, 10 ** 8))[:3] == (9, 43046721, 2)
    assert M.setup(unit_cfg(1, 4)) == (2, 2, 2, 1)
    assert M.setup(unit_cfg(2, 17))[:3] == (2, 4, 4)


def test_setup_matches_golden(golden):
    for e in golden["setup"]:
        sp = M.setup(unit_cfg(e["dims"], e["maxcalls"]))
        assert (sp.g, sp.m, sp.p, sp.s) == (e["g"], e["m"], e["p"], e["s_workers1"])


def test_setup_maximal_property():
    # test_driver.cpp:78-98
    rng = np.random.default_rng(31)
    for _ in range(200):
        d = int(1 + rng.integers(0, 8))
        floor_calls = 2 << d
        maxcalls = int(floor_calls + rng.integers(0, 10_000_000 - floor_calls))
        sp = M.setup(unit_cfg(d, maxcalls))
        assert sp.m == sp.g ** d and sp.p >= 2 and sp.m * sp.p <= maxcalls
        assert 2 * (sp.g + 1) ** d > maxcalls


def test_batch_size():
    # test_driver.cpp:100-108
    assert M.set_batch_size(484, 8) == 2
    assert M.set_batch_size(1, 64) == 1
    assert M.set_batch_size(43046721, 16) == 84076
    assert M.set_batch_size(32, 1) == 1 and M.set_batch_size(33, 1) == 2
    with pytest.raises(ValueError):
        M.set_batch_size(0, 4)
    with pytest.raises(ValueError):
        M.set_batch_size(10, 0)


@pytest.mark.parametrize("field,value", [
    ("dims", 0), ("n_bins", 1), ("maxcalls", 7), ("tau_rel", 0.0), ("tau_rel", 1.0), ("itmax", 0),
    ("ita", 16), ("alpha", -0.5), ("alpha", float("inf")), ("chi2_dof_max", 0.0)])
def test_validate_rejects(field, value):
    # test_driver.cpp:110-163
    cfg = unit_cfg(2, 1000)
    cfg.validate()
    setattr(cfg, field, value)
    with pytest.raises(ValueError):
        cfg.validate()
    with pytest.raises(ValueError):
        M.setup(cfg)


def test_validate_bounds():
    cfg = unit_cfg(2, 1000)
    cfg.lower = [0.0]
    with pytest.raises(ValueError):
        cfg.validate()
    cfg = unit_cfg(2, 1000)
    cfg.upper = [1.0, float("nan")]
    with pytest.raises(ValueError):
        cfg.validate()
    cfg = unit_cfg(2, 1000)
    cfg.upper = [1.0, 0.0]
    with pytest.raises(ValueError):
        cfg.validate()


def test_variant_names():
    assert M.variant_name(M.Variant.mcubes) == "mcubes" and M.variant_name(M.Variant.mcubes1d) == "mcubes1d"
    assert M.parse_variant("mcubes1d") == M.Variant.mcubes1d and M.parse_variant("vegas") is None


def test_weighted_estimate_examples():
    # test_driver.cpp:174-209
    c = M.weighted_estimate([(1.0, 0.01, 1)])
    assert math.isclose(c.estimate, 1.0) and math.isclose(c.sigma, 0.1) and c.chi2_dof == 0.0
    c = M.weighted_estimate([(1.0, 0.01, 1), (1.2, 0.04, 2)])
    assert math.isclose(c.estimate, 1.04, rel_tol=1e-12) and math.isclose(c.sigma, 1 / math.sqrt(125), rel_tol=1e-12)
    assert math.isclose(c.chi2_dof, 0.8, rel_tol=1e-12)
    c = M.weighted_estimate([(1.0, 0.01, 1)] * 3)
    assert math.isclose(c.sigma, 0.1 / math.sqrt(3.0), rel_tol=1e-12) and abs(c.chi2_dof) < 1e-15
    c = M.weighted_estimate([(3.0, 1.0, 1), (2.0, 0.0, 2), (5.0, 0.0, 3)])
    assert (c.estimate, c.sigma, c.chi2_dof) == (2.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        M.weighted_estimate([])
    with pytest.raises(ValueError):
        M.weighted_estimate([(1.0, -0.5, 1)])


def test_weighted_estimate_bitwise_golden(golden):
    for c in golden["weighted_estimate"]:
        e, v = h2a(c["est"]), h2a(c["var"])
        got = M.weighted_estimate([(a, b, i + 1) for i, (a, b) in enumerate(zip(e, v))])
        assert same_bits(list(got), h2a(c["out"]))


def test_check_convergence():
    # test_driver.cpp:211-224
    cfg = unit_cfg(1, 100)
    assert M.check_convergence((10.0, 0.009, 1.0), cfg)
    assert not M.check_convergence((10.0, 0.011, 1.0), cfg)
    assert not M.check_convergence((10.0, 0.009, 1.6), cfg)
    assert M.check_convergence((-10.0, 0.009, 1.0), cfg)
    assert M.check_convergence((0.0, 9e-4, 1.0), cfg)
    assert not M.check_convergence((0.0, 2e-3, 1.0), cfg)


def test_grid_uniform_and_text_roundtrip():
    # test_grid.cpp:66-93, 302-319
    g = M.Grid(2, 4, [0.0, -1.0], [2.0, 1.0])
    assert np.array_equal(g.edges(0), [0.5, 1.0, 1.5, 2.0]) and np.array_equal(g.edges(1), [-0.5, 0.0, 0.5, 1.0])
    assert M.Grid.read(g.write()) == g
    with pytest.raises(ValueError):
        M.Grid(0, 4, [], [])
    with pytest.raises(ValueError):
        M.Grid(1, 1, [0.0], [1.0])
    with pytest.raises(ValueError):
        M.Grid(1, 4, [1.0], [0.0])
    with pytest.raises(ValueError):
        M.Grid.read("1 2\n0 1 0.5 0.9\n")  # last edge != upper
    with pytest.raises(ValueError):
        M.Grid.read("1 2\n0 1 0.5\n")


def test_grid_transform_hand_worked():
    # test_grid.cpp:95-131
    g = M.Grid.read("1 2\n0 1 0.2 1.0\n")
    jac, x = g.transform([0.25])
    assert math.isclose(x[0], 0.1, rel_tol=1e-15) and math.isclose(jac, 0.4, rel_tol=1e-15)
    jac, x = g.transform([0.75])
    assert math.isclose(x[0], 0.6, rel_tol=1e-14) and math.isclose(jac, 1.6, rel_tol=1e-14)
    g = M.Grid(1, 4, [0.0], [1.0])
    jac, x = g.transform([float.fromhex("0x1.fffffffffffffp-1")])
    assert 0.75 < x[0] < 1.0
    assert g.bin_index(1.0) == 3 and g.bin_index(0.0) == 0 and g.bin_index(0.3) == 1


def test_integrands_and_reference_values(golden):
    for e in golden["reference_value"]:
        fam, d = e["family"], e["dims"]
        spec = M.make_fA() if fam == 7 else (M.make_fB() if fam == 8 else M.make_suite_integrand(fam, d))
        assert math.isclose(spec.reference, h2f(e["value"]), rel_tol=1e-13, abs_tol=1e-300)
    assert M.make_integrand("f4", 8).id == 4 and M.make_integrand("fA", 0).dims == 6
    for bad in [("f7", 3), ("f4", 0), ("fA", 5), ("zz", 2)]:
        with pytest.raises(ValueError):
            M.make_integrand(*bad)
    assert math.isclose(M.make_fA().reference, -49.165073, rel_tol=1e-7)
    assert math.isclose(M.make_fB().reference, 1.0, rel_tol=1e-12)


def test_table_integrand_reference_value():
    tabs = np.array([[1.0, 3.0, 2.0], [0.5, 0.5, 1.5]])
    f = M.make_table_integrand(tabs, [0.0, -1.0], [2.0, 1.0])
    # trapezoid: axis0 h=1: 1*(6 - 1.5)=4.5 ; axis1 h=1: (2.5 - 1.0)=1.5
    assert math.isclose(f.reference, 4.5 * 1.5)
    assert f.params[0] == 3 and len(f.params) == 1 + 2 * 2 + 6


def test_partition_covers_range():
    from paper_2202_01753_b200.dist import partition
    for m in (1, 7, 43046721, 2 ** 32):
        for world in (1, 2, 3, 8):
            cuts = [partition(m, world, r) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))


def test_checkpoint_text_round_trip():
    import paper_2202_01753_b200 as M

    g = M.Grid(3, 5, [0.0, -1.0, 2.0], [1.0, 1.0, 4.5])
    hist = [M.IterationResult(0.1 + i / 3.0, 1e-7 * (i + 1) / 7.0, i + 1) for i in range(4)]
    cp = M.Checkpoint(g, hist)
    back = M.Checkpoint.read(cp.write())
    assert np.array_equal(back.grid.raw_edges.view(np.uint64), g.raw_edges.view(np.uint64))
    assert back.grid.lowers == g.lowers and back.grid.uppers == g.uppers
    assert [(h.estimate, h.variance, h.index) for h in back.history] == [(h.estimate, h.variance, h.index) for h in hist]
