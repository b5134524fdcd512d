"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and the ``--impl reference`` arm) may import this
package; the product (``paper_2202_01753_b200``) never does.

Two libraries live here:

* ``liboracle.so``  -- ``mcubes_oracle.c``, a plain-C restatement of the
  reference algorithm (each function cites the reference file:line it
  follows).  Single-threaded.
* ``_ref/libmcubes_ref.so`` -- the UNMODIFIED reference headers from
  ``/root/reference/proj/include`` compiled behind a C shim
  (``ref_harness.cpp``).  Multi-threaded exactly as the reference is
  (``sampler.hpp:213-278``).  Built here by ``oracle/Makefile``; it travels to
  the GPU box as a prebuilt file (``/root/reference`` does not exist there).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
XWORDS = 67  # words per exact accumulator (mcubes_oracle.c XW == MCB_XWORDS)
# sample stream codes (include/mcubes_b200.h mcb_rng; orc_set_rng)
RNG_CODES = {"compat": 0, "philox": 1, "philox_exact": 2}

_D = C.c_double
_U32 = C.c_uint32
_U64 = C.c_uint64
_I = C.c_int
_PD = C.POINTER(C.c_double)
_PU32 = C.POINTER(C.c_uint32)
_PU64 = C.POINTER(C.c_uint64)


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
    return C.CDLL(path)


_orc = None
_ref = None


def orc():
    """The C restatement (liboracle.so)."""
    global _orc
    if _orc is None:
        lib = _load(os.path.join(HERE, "liboracle.so"))
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_uniform01.restype = _D
        lib.orc_uniform01.argtypes = [_U64] * 5
        lib.orc_iteration_root.restype = _U64
        lib.orc_iteration_root.argtypes = [_U64, _U64]
        lib.orc_exact_sum.restype = _D
        lib.orc_exact_sum.argtypes = [_PD, _U64]
        lib.orc_words_value.restype = _D
        lib.orc_words_value.argtypes = [_PU64, _PU64]
        lib.orc_eval.argtypes = [_I, _PD, _U32, _U32, _PD, _PD]
        lib.orc_transform.argtypes = [_U32, _U32, _PD, _PD, _PD, _PD, _PD, _PU32, _PD]
        lib.orc_grid_uniform.argtypes = [_U32, _U32, _PD, _PD, _PD]
        lib.orc_grid_uniform.restype = None
        lib.orc_grid_adjust.argtypes = [_U32, _U32, _PD, _PD, _PD, _PD, _D, _I, _PD]
        lib.orc_sample_partial.argtypes = [_I, _PD, _U32, _U32, _U32, _PD, _PD, _PD, _U64, _U64,
                                           _U64, _U64, _I, _I, _U64, _U64, _PU64, _PU64, _PD, _PD]
        lib.orc_round_partial.argtypes = [_PU64, _U32, _U32, _U64, _I, _I, _PD, _PD, _PD]
        lib.orc_v_sample.argtypes = [_I, _PD, _U32, _U32, _U32, _PD, _PD, _PD, _U64, _U64, _U64,
                                     _U64, _U64, _I, _I, _PD, _PD, _PD, _PU64, _PD, _PD]
        lib.orc_setup.argtypes = [_U32, _U32, _U64, _U32, _U32, _D, _D, _D, _PD, _PD, C.c_uint, _PU64]
        lib.orc_weighted_estimate.argtypes = [_U32, _PD, _PD, _PD]
        lib.orc_check_convergence.argtypes = [_D, _D, _D, _D, _D]
        lib.orc_integrate.argtypes = [_I, _PD, _U32, _U32, _U32, _U64, _U32, _U32, _D, _D, _D, _U64,
                                      _I, _PD, _PD, _PD, _PU64, _PD, _PD, _U32, _PD, _PU64, _PD, _PD]
        lib.orc_set_rng.argtypes = [_I]
        lib.orc_set_rng.restype = None
        lib.orc_set_threads.argtypes = [_I]
        lib.orc_set_threads.restype = None
        lib.orc_xwords.restype = _U32
        assert lib.orc_xwords() == XWORDS
        _orc = lib
    return _orc


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libmcubes_ref.so"))


def ref():
    """The compiled reference (oracle/_ref/libmcubes_ref.so)."""
    global _ref
    if _ref is None:
        lib = _load(os.path.join(HERE, "_ref", "libmcubes_ref.so"))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_uniform01.restype = _D
        lib.ref_uniform01.argtypes = [_U64] * 5
        lib.ref_iteration_root.restype = _U64
        lib.ref_iteration_root.argtypes = [_U64, _U64]
        lib.ref_exact_sum.restype = _D
        lib.ref_exact_sum.argtypes = [_PD, _U64]
        lib.ref_reference_value.restype = _D
        lib.ref_reference_value.argtypes = [_I, _U32]
        lib.ref_eval.argtypes = [_I, _PD, _U32, _U32, _PD, _PD]
        lib.ref_transform.argtypes = [_U32, _U32, _PD, _PD, _PD, _PD, _PD, _PU32, _PD]
        lib.ref_v_sample.argtypes = [_I, _PD, _U32, _U32, _U32, _PD, _PD, _PD, _U64, _U64, _U64,
                                     _U64, _U64, _I, C.c_uint, _PD, _PD, _PD, _PU64, _PD, _PD]
        lib.ref_grid_adjust.argtypes = [_U32, _U32, _PD, _PD, _PD, _PD, _D, _I, _PD]
        lib.ref_setup.argtypes = [_U32, _U32, _U64, _U32, _U32, _D, _D, _D, _PD, _PD, C.c_uint, _PU64]
        lib.ref_set_batch_size.argtypes = [_U64, C.c_uint, _PU64]
        lib.ref_weighted_estimate.argtypes = [_U32, _PD, _PD, _PD]
        lib.ref_check_convergence.argtypes = [_D, _D, _D, _D, _D]
        lib.ref_integrate.argtypes = [_I, _PD, _U32, _U32, _U32, _U64, _U32, _U32, _D, _D, _D, _U64,
                                      _I, _PD, _PD, C.c_uint, _PD, _PU64, _PD, _PD, _U32, _PD, _PU64,
                                      _PD, _PD]
        _ref = lib
    return _ref


# ---------------------------------------------------------------- helpers
def darr(vals):
    vals = list(vals)
    return (C.c_double * max(1, len(vals)))(*vals)


def _np():
    import numpy as np
    return np


def ptr(a):
    """ctypes double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_PD)


def uniform_edges(d, nb, lower, upper):
    np = _np()
    e = np.zeros(d * nb)
    orc().orc_grid_uniform(d, nb, darr(lower), darr(upper), ptr(e))
    return e


class OracleError(RuntimeError):
    def __init__(self, code, msg, x=None, fx=None):
        super().__init__(msg)
        self.code, self.x, self.fx = code, x, fx


def v_sample(lib_kind, integrand, params, d, nb, lower, upper, edges, m, s, p, seed, iteration,
             mode="all", threads=0, rng="compat"):
    """Run one iteration through the oracle ('orc') or compiled reference ('ref').

    mode: 'all' | 'axis0' | 'frozen' | 'serial' (ref only: vegas_serial_iteration).
    rng: 'compat' (the reference stream) or 'philox' (orc only: the C twin of
    the B200 Philox path, which the reference does not have).
    Returns dict(est, var, contrib(np, d*nb) or None, writes).
    """
    np = _np()
    params = np.ascontiguousarray(params if params is not None else [], dtype=np.float64)
    est, var = C.c_double(), C.c_double()
    writes = C.c_uint64(0)
    contrib = np.zeros(d * nb)
    ex = np.zeros(max(d, 1))
    efx = C.c_double()
    lo, hi = darr(lower), darr(upper)
    ep = ptr(np.ascontiguousarray(edges, dtype=np.float64)) if edges is not None else None
    if lib_kind == "ref":
        lib = ref()
        code = {"all": 0, "axis0": 1, "frozen": 2, "serial": 3, "serial_axis0": 4}[mode]
        rc = lib.ref_v_sample(integrand, ptr(params), len(params), d, nb, lo, hi, ep, m, s, p, seed,
                              iteration, code, threads, C.byref(est), C.byref(var), ptr(contrib),
                              C.byref(writes), ptr(ex), C.byref(efx))
        err = lib.ref_last_error
    else:
        lib = orc()
        if ep is None:
            e = uniform_edges(d, nb, lower, upper)
            ep = ptr(e)
        bin_mode = 1 if mode in ("axis0", "serial_axis0") else 0
        kbins = 0 if mode == "frozen" else 1
        lib.orc_set_rng(RNG_CODES[rng])
        lib.orc_set_threads(threads if threads else 1)
        try:
            rc = lib.orc_v_sample(integrand, ptr(params), len(params), d, nb, lo, hi, ep, m, s, p, seed,
                                  iteration, bin_mode, kbins, C.byref(est), C.byref(var), ptr(contrib),
                                  C.byref(writes), ptr(ex), C.byref(efx))
        finally:
            lib.orc_set_rng(0)
            lib.orc_set_threads(1)
        err = lib.orc_last_error
    if rc != 0:
        raise OracleError(rc, err().decode(), ex[:d].copy(), efx.value)
    return dict(est=est.value, var=var.value, contrib=None if mode == "frozen" else contrib,
                writes=writes.value)


def integrate(lib_kind, integrand, params, d, nb, maxcalls, itmax, ita, tau, alpha, chi2max, seed,
              variant, lower, upper, workers=0, want_grids=False, rng="compat"):
    np = _np()
    params = np.ascontiguousarray(params if params is not None else [], dtype=np.float64)
    res = np.zeros(8)
    sp = (C.c_uint64 * 4)()
    he = np.zeros(itmax)
    hv = np.zeros(itmax)
    grids = np.zeros(itmax * d * nb) if want_grids else None
    wr = (C.c_uint64 * itmax)()
    ex = np.zeros(d)
    efx = C.c_double()
    if lib_kind == "ref":
        lib = ref()
        rc = lib.ref_integrate(integrand, ptr(params), len(params), d, nb, maxcalls, itmax, ita, tau,
                               alpha, chi2max, seed, variant, darr(lower), darr(upper), workers,
                               ptr(res), sp, ptr(he), ptr(hv), itmax, ptr(grids), wr, ptr(ex),
                               C.byref(efx))
        err = lib.ref_last_error
    else:
        lib = orc()
        lib.orc_set_rng(RNG_CODES[rng])
        try:
            rc = lib.orc_integrate(integrand, ptr(params), len(params), d, nb, maxcalls, itmax, ita, tau,
                                   alpha, chi2max, seed, variant, darr(lower), darr(upper), ptr(res), sp,
                                   ptr(he), ptr(hv), itmax, ptr(grids), wr, ptr(ex), C.byref(efx))
        finally:
            lib.orc_set_rng(0)
        err = lib.orc_last_error
    if rc != 0:
        raise OracleError(rc, err().decode(), ex.copy(), efx.value)
    n = int(res[3])
    out = dict(estimate=res[0], sigma=res[1], chi2_dof=res[2], iterations_used=n,
               converged=bool(res[4]), total_samples=int(res[5]), bin_writes=int(res[6]),
               g=sp[0], m=sp[1], p=sp[2], s=sp[3], hist_est=he[:n].copy(), hist_var=hv[:n].copy(),
               writes=[wr[i] for i in range(n)])
    if want_grids:
        out["grids"] = grids.reshape(itmax, d * nb)[:n].copy()
    return out


def grid_adjust(lib_kind, d, nb, lower, upper, edges, contrib, alpha=1.5, symmetric=False):
    """Grid::adjusted / adjusted_symmetric (grid.hpp:104-146) through the
    oracle ('orc') or the compiled reference ('ref'); returns the new edges."""
    np = _np()
    out = np.zeros(d * nb)
    e = np.ascontiguousarray(edges, dtype=np.float64)
    c = np.ascontiguousarray(contrib, dtype=np.float64)
    if lib_kind == "ref":
        lib, err = ref(), ref().ref_last_error
        rc = lib.ref_grid_adjust(d, nb, darr(lower), darr(upper), ptr(e), ptr(c), alpha, int(symmetric), ptr(out))
    else:
        lib, err = orc(), orc().orc_last_error
        rc = lib.orc_grid_adjust(d, nb, darr(lower), darr(upper), ptr(e), ptr(c), alpha, int(symmetric), ptr(out))
    if rc != 0:
        raise OracleError(rc, err().decode())
    return out


def weighted_estimate(est, var):
    """The reference's weighted_estimate (driver.hpp:146-169): (I, sigma, chi2/dof)."""
    np = _np()
    e = np.ascontiguousarray(est, dtype=np.float64)
    v = np.ascontiguousarray(var, dtype=np.float64)
    out = np.zeros(3)
    rc = ref().ref_weighted_estimate(len(e), ptr(e), ptr(v), ptr(out))
    if rc != 0:
        raise OracleError(rc, ref().ref_last_error().decode())
    return float(out[0]), float(out[1]), float(out[2])
