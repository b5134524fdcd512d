"""CPU: pin the oracle (oracle/mcubes_oracle.c, the C restatement) to the
reference's own golden vectors and to the committed fixtures generated from
the compiled reference.  When oracle/_ref is built (this container), also
cross-check the restatement against the compiled reference directly."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle as O
from conftest import bits, h2a, h2f, same_bits

# reference-owned goldens (file:line under /root/reference/proj/)
TRIPLE = dict(est=0x3fe0bc4a50c32562, var=0x3f4a33dfda24e234,  # tests/test_oracle.cpp:62-78
              cells=[0x3fb06e6686d8c889, 0x3fcefebb1d601ea6, 0x3fef06ef329df87c, 0x3ff9ffd017aba70c])
# tests/test_exact_sum.cpp:31-56 (frozen stream, exact rational sum)
KSTREAM = [float.fromhex(v) for v in (
    "-0x1.5585300363cb9p-87", "-0x1.371a72b324890p-8", "-0x1.a975ce938fd5ep+34", "0x1.9ec48898db44bp-38",
    "0x1.3ffeea53e0af4p-312", "0x1.b3ac8d0889acap-207", "-0x1.b530da23339a3p+120", "0x1.c0acc5be64458p+297",
    "-0x1.77a3397d71e64p+102", "0x1.7954bed57438ap-103", "0x1.0726a1c74a7e4p-296", "0x1.eb0b7efc847cap+153",
    "-0x1.4c5d7d508cd1cp-288", "-0x1.f8988032c0a00p-84", "-0x1.1e737bef31d50p+154", "-0x1.d53edfa73edc3p-116",
    "0x1.c738881873644p-286", "0x1.a166784096461p-253", "0x1.112ac83f0104ap+28", "-0x1.da4132ee21677p+84",
    "0x1.bc8d409c5c571p-241", "0x1.82d480c797d1ap-128", "0x1.047405b78cc2cp-169", "-0x1.4763bc677fcdbp-223",
    "0x1.4d96dc0e2bc0ap+240", "0x1.35331756e4234p+149", "0x1.7cbdbdaa6de82p-129", "-0x1.506449b71c618p+7",
    "0x1.d257dbb346952p-205", "0x1.f21f1a3348915p-87", "0x1.fe6057754b40dp-304", "-0x1.a518812c4010ap+163",
    "-0x1.6df1a34c6ab1cp-27", "-0x1.2ef719a72a638p+202", "0x1.dddf7756c8691p-6", "-0x1.478711ba5db78p+70",
    "-0x1.f582333562d98p+63", "0x1.5cb55ad8b50c2p-146", "0x1.3de4d46246daep-106", "-0x1.9f4f4606e2a0ap-202",
    "0x1.0760170f7eb4cp-37", "-0x1.06b93d09ceca1p+191", "0x1.b0e2e1e788aa4p+174", "0x1.30487a1a3808ap-120",
    "-0x1.e7ba06f71a9d3p+133", "-0x1.8e4b9f47919b7p-57", "-0x1.12b5376d545c2p+125", "0x1.af3a7e2460616p+231",
    "-0x1.4ad70429c2d6ap+272", "0x1.608df75c44c0bp+82", "-0x1.4a11eed03fcddp-103", "0x1.127b557091b00p+113",
    "-0x1.2feb45521b9bep-173", "0x1.625e7d40e7474p-28", "-0x1.38d03633d876ap-265", "0x1.1a5216e039d5cp-170",
    "-0x1.0122c81909f71p-265", "-0x1.c8eeedae3826cp+151", "-0x1.bd241ea40af96p+241", "0x1.d9541fe50be0ep+236",
    "0x1.df661e726ad71p+284", "-0x1.f120fd2a1ea2dp-149", "0x1.63232cb16c88fp-200", "0x1.63a874ceb7585p-109",
)]


def test_reference_golden_triple():
    r = O.v_sample("orc", 32, None, 1, 4, [0.0], [1.0], None, 4, 1, 2, 1, 0)
    assert bits(r["est"]) == TRIPLE["est"] and bits(r["var"]) == TRIPLE["var"]
    assert [bits(c) for c in r["contrib"]] == TRIPLE["cells"]
    assert r["writes"] == 8


def test_reference_exact_sum_stream():
    v = np.array(KSTREAM)
    assert bits(O.orc().orc_exact_sum(O.ptr(v), len(v))) == bits(float.fromhex("0x1.c0bbc049ec56cp+297"))
    # permutation / partition invariance (test_exact_sum.cpp:58-79)
    rng = np.random.default_rng(7)
    for _ in range(20):
        w = rng.permutation(v)
        assert bits(O.orc().orc_exact_sum(O.ptr(w), len(w))) == bits(float.fromhex("0x1.c0bbc049ec56cp+297"))


def test_reference_exact_sum_edges():
    s = lambda *vals: O.orc().orc_exact_sum(O.darr(vals), len(vals))  # noqa: E731
    assert s(1e100, 1.0, -1e100) == 1.0  # classic cancellation (test_exact_sum.cpp:81-102)
    assert s(1.0, 2 ** -53) == 1.0  # tie to even (test_exact_sum.cpp:104-119)
    assert s(1.0, 2 ** -53, 2 ** -105) == 1.0 + 2 ** -52
    assert s(5e-324, 5e-324) == 1e-323  # subnormals exact (test_exact_sum.cpp:121-129)


def test_reference_readme_row():
    # proj/README.md:99-102: f2 3D maxcalls 1e5 seed 7
    r = O.integrate("orc", 2, None, 3, 50, 100000, 15, 10, 1e-3, 1.5, 1.5, 7, 0, [0.0] * 3, [1.0] * 3)
    assert repr(float(r["estimate"])) == "3590570.5674877567"
    assert r["sigma"] == 2559.8737453845001 and r["chi2_dof"] == 0.061055568029569747
    assert r["converged"] and r["iterations_used"] == 2 and r["total_samples"] == 186624


def test_reference_setup_examples():
    # tests/test_driver.cpp:47-76
    for d, mc, g, m, p in [(2, 1000, 22, 484, 2), (8, 10 ** 8, 9, 43046721, 2), (1, 4, 2, 2, 2), (2, 17, 2, 4, 4)]:
        sp = (O._U64 * 4)()
        assert O.orc().orc_setup(d, 50, mc, 15, 10, 1e-3, 1.5, 1.5, O.darr([0.0] * d), O.darr([1.0] * d), 1, sp) == 0
        assert (sp[0], sp[1], sp[2]) == (g, m, p)


def test_golden_uniform01(golden):
    for e in golden["uniform01"]:
        assert bits(O.orc().orc_uniform01(*e["key"])) == int(e["value"], 16)
    for e in golden["iteration_root"]:
        assert O.orc().orc_iteration_root(e["seed"], e["it"]) == int(e["value"], 16)


def test_golden_exact_sum(golden):
    for e in golden["exact_sum"]:
        v = h2a(e["values"])
        assert bits(O.orc().orc_exact_sum(O.ptr(v), len(v))) == int(e["sum"], 16)


def test_golden_setup(golden):
    for e in golden["setup"]:
        d = e["dims"]
        sp = (O._U64 * 4)()
        assert O.orc().orc_setup(d, 50, e["maxcalls"], 15, 10, 1e-3, 1.5, 1.5, O.darr([0.0] * d), O.darr([1.0] * d),
                                 1, sp) == 0
        assert (sp[0], sp[1], sp[2], sp[3]) == (e["g"], e["m"], e["p"], e["s_workers1"])


def _case_args(c):
    params = h2a(c["params"]) if c["params"] else None
    edges = h2a(c["edges"]) if c["edges"] else None
    return params, edges


def test_golden_v_sample(golden):
    for c in golden["v_sample"]:
        params, edges = _case_args(c)
        r = O.v_sample("orc", c["integrand"], params, c["dims"], c["n_bins"], c["lower"], c["upper"], edges, c["m"],
                       c["s"], c["p"], c["seed"], c["iteration"], mode=c["mode"])
        assert bits(r["est"]) == int(c["est"], 16), c["name"]
        assert bits(r["var"]) == int(c["var"], 16), c["name"]
        if "contrib" in c:
            assert same_bits(r["contrib"], h2a(c["contrib"])), c["name"]
            assert r["writes"] == c["writes"], c["name"]


def test_golden_adjust(golden):
    for c in golden["adjust"]:
        d, nb = c["dims"], c["n_bins"]
        out = np.zeros(d * nb)
        rc = O.orc().orc_grid_adjust(d, nb, O.ptr(h2a(c["lower"])), O.ptr(h2a(c["upper"])), O.ptr(h2a(c["edges"])),
                                     O.ptr(h2a(c["contrib"])), c["alpha"], c["symmetric"], O.ptr(out))
        assert rc == 0
        assert same_bits(out, h2a(c["out"]))


def test_golden_weighted(golden):
    for c in golden["weighted_estimate"]:
        e, v = h2a(c["est"]), h2a(c["var"])
        o3 = np.zeros(3)
        assert O.orc().orc_weighted_estimate(len(e), O.ptr(e), O.ptr(v), O.ptr(o3)) == 0
        assert same_bits(o3, h2a(c["out"]))


def test_golden_integrate(golden):
    for c in golden["integrate"]:
        params = h2a(c["params"]) if c["params"] else None
        r = O.integrate("orc", c["integrand"], params, c["dims"], c["n_bins"], c["maxcalls"], c["itmax"], c["ita"],
                        c["tau_rel"], 1.5, 1.5, c["seed"], c["variant"], c["lower"], c["upper"], want_grids=True)
        assert r["iterations_used"] == c["iterations_used"], c["name"]
        assert r["converged"] == c["converged"] and r["total_samples"] == c["total_samples"]
        assert r["bin_writes"] == c["bin_writes"], c["name"]
        assert same_bits(r["hist_est"], h2a(c["hist_est"])) and same_bits(r["hist_var"], h2a(c["hist_var"]))
        assert bits(r["estimate"]) == int(c["estimate"], 16) and bits(r["sigma"]) == int(c["sigma"], 16)
        assert bits(r["chi2_dof"]) == int(c["chi2_dof"], 16)
        for g, want in zip(r["grids"], c["grids"]):
            assert same_bits(g, h2a(want)), c["name"]


def test_partials_compose_exactly():
    """Splitting the cube range and summing exchange words reproduces the
    single-range result bit for bit (what the multi-GPU all-reduce relies on)."""
    d, nb, m, p = 3, 12, 6 ** 3, 3
    W = O.XWORDS
    nacc = 3 + d * nb
    full = np.zeros(nacc * W, dtype=np.uint64)
    args = (5, None, 0, d, nb, O.darr([0.0] * d), O.darr([1.0] * d))
    edges = O.uniform_edges(d, nb, [0.0] * d, [1.0] * d)

    def part(c0, c1):
        w = np.zeros(nacc * W, dtype=np.uint64)
        rc = O.orc().orc_sample_partial(5, None, 0, d, nb, O.darr([0.0] * d), O.darr([1.0] * d), O.ptr(edges), m, p,
                                        9, 2, 0, 1, c0, c1, w.ctypes.data_as(C.POINTER(C.c_uint64)), None, None, None)
        assert rc == 0
        return w

    full = part(0, m)
    for cuts in ([0, 1, m], [0, 100, 101, m], [0, 50, 100, 150, m]):
        acc = np.zeros_like(full)
        for a, b in zip(cuts[:-1], cuts[1:]):
            acc += part(a, b)
        assert np.array_equal(acc, full)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference here)")
def test_restatement_matches_compiled_reference_random():
    """Randomised shapes, integrands and modes: C restatement == reference."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        d = int(rng.integers(1, 6))
        g = int(rng.integers(1, 7))
        m = g ** d
        p = int(rng.integers(2, 6))
        nb = int(rng.integers(2, 20))
        fam = int(rng.integers(1, 7))
        mode = ["all", "axis0", "frozen"][trial % 3]
        lo = list(rng.uniform(-1.0, 0.5, d)) if fam in (1, 2, 4, 5) and trial % 2 else [0.0] * d
        hi = [v + 1.0 for v in lo]
        seed, it = int(rng.integers(0, 2 ** 40)), int(rng.integers(0, 50))
        a = O.v_sample("orc", fam, None, d, nb, lo, hi, None, m, 1, p, seed, it, mode=mode)
        b = O.v_sample("ref", fam, None, d, nb, lo, hi, None, m, 3, p, seed, it, mode=mode, threads=3)
        assert bits(a["est"]) == bits(b["est"]) and bits(a["var"]) == bits(b["var"])
        if mode != "frozen":
            assert same_bits(a["contrib"], b["contrib"]) and a["writes"] == b["writes"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference here)")
def test_restatement_nonfinite_point_matches_reference():
    with pytest.raises(O.OracleError) as ea:
        O.v_sample("orc", 35, None, 2, 4, [0.0] * 2, [1.0] * 2, None, 4, 4, 2, 1, 1)
    with pytest.raises(O.OracleError) as eb:
        O.v_sample("ref", 35, None, 2, 4, [0.0] * 2, [1.0] * 2, None, 4, 4, 2, 1, 1, mode="serial")
    assert ea.value.code == -2 and eb.value.code == -2
    assert same_bits(ea.value.x, eb.value.x) and np.isinf(ea.value.fx)
