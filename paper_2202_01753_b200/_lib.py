"""ctypes binding of the C ABI in ``include/mcubes_b200.h`` (libmcubes_b200.so).

This is the product's only native entry point.  There is no CPU fallback: if
the shared library is missing the import fails loudly, and every compute call
goes to the sm_100a kernels behind the ABI.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmcubes_b200.so")

MCB_OK, MCB_EINVAL, MCB_ENONFINITE, MCB_ECUDA, MCB_EINTERNAL = 0, -1, -2, -3, -9
MCB_XWORDS = 67

_D, _U32, _U64, _I32 = C.c_double, C.c_uint32, C.c_uint64, C.c_int32
_PD = C.POINTER(C.c_double)
_PU64 = C.POINTER(C.c_uint64)
_VP = C.c_void_p


class mcb_integrand(C.Structure):
    _fields_ = [("id", C.c_int32), ("n_params", C.c_uint32), ("params", _PD)]


class mcb_config(C.Structure):
    _fields_ = [
        ("dims", _U32), ("n_bins", _U32), ("maxcalls", _U64), ("itmax", _U32), ("ita", _U32),
        ("tau_rel", _D), ("alpha", _D), ("chi2_dof_max", _D), ("seed", _U64), ("variant", _I32),
        ("workers", _U32), ("lower", _PD), ("upper", _PD), ("rng", _I32), ("reserved", _I32),
    ]


class mcb_result(C.Structure):
    _fields_ = [
        ("estimate", _D), ("sigma", _D), ("chi2_dof", _D), ("iterations_used", _U32),
        ("converged", _I32), ("total_samples", _U64), ("bin_writes", _U64),
        ("g", _U64), ("m", _U64), ("p", _U64), ("s", _U64),
    ]


class mcb_iteration(C.Structure):
    _fields_ = [("estimate", _D), ("variance", _D), ("index", _U32), ("pad", _U32)]


class mcb_iteration_view(C.Structure):
    _fields_ = [
        ("iteration", _U32), ("adjusting", _I32), ("result", mcb_iteration),
        ("running_estimate", _D), ("running_sigma", _D), ("running_chi2_dof", _D),
        ("grid_edges", _PD), ("bin_writes", _U64),
    ]


OBSERVER = C.CFUNCTYPE(None, C.POINTER(mcb_iteration_view), _VP)

# every symbol include/mcubes_b200.h declares, with its ctypes signature
SIGNATURES = {
    "mcb_abi_version": (C.c_int, []),
    "mcb_ctx_create": (C.c_int, [C.c_int, C.POINTER(_VP)]),
    "mcb_ctx_destroy": (C.c_int, [_VP]),
    "mcb_ctx_set_stream": (C.c_int, [_VP, _VP]),
    "mcb_ctx_synchronize": (C.c_int, [_VP]),
    "mcb_ctx_launches": (_U64, [_VP]),
    "mcb_last_error": (C.c_char_p, [_VP]),
    "mcb_last_nonfinite": (C.c_int, [_VP, _PD, _U32, _PD]),
    "mcb_v_sample": (C.c_int, [_VP, C.POINTER(mcb_integrand), _U32, _U32, _PD, _PD, _PD, _U64, _U64,
                               _U64, _U64, _U64, _I32, _PD, _PD, _PD, _PU64]),
    "mcb_v_sample_no_adjust": (C.c_int, [_VP, C.POINTER(mcb_integrand), _U32, _U32, _PD, _PD, _PD,
                                         _U64, _U64, _U64, _U64, _U64, _PD, _PD]),
    "mcb_v_sample_philox": (C.c_int, [_VP, C.POINTER(mcb_integrand), _U32, _U32, _PD, _PD, _PD, _U64,
                                      _U64, _U64, _U64, _U64, _I32, _PD, _PD, _PD, _PU64]),
    "mcb_v_sample_rng": (C.c_int, [_VP, C.POINTER(mcb_integrand), _I32, _U32, _U32, _PD, _PD, _PD, _U64,
                                   _U64, _U64, _U64, _U64, _I32, _PD, _PD, _PD, _PU64]),
    "mcb_grid_adjust": (C.c_int, [_VP, _U32, _U32, _PD, _PD, _PD, _PD, _D, _I32, _PD]),
    "mcb_setup": (C.c_int, [C.POINTER(mcb_config), _PU64, _PU64, _PU64, _PU64]),
    "mcb_set_batch_size": (C.c_int, [_U64, _U32, _PU64]),
    "mcb_weighted_estimate": (C.c_int, [_U32, _PD, _PD, _PD, _PD, _PD]),
    "mcb_check_convergence": (C.c_int, [_D, _D, _D, _D, _D]),
    "mcb_grid_uniform": (C.c_int, [_U32, _U32, _PD, _PD, _PD]),
    "mcb_integrate": (C.c_int, [_VP, C.POINTER(mcb_integrand), C.POINTER(mcb_config),
                                C.POINTER(mcb_result), C.POINTER(mcb_iteration), _U32, OBSERVER, _VP]),
    "mcb_integrate_resume": (C.c_int, [_VP, C.POINTER(mcb_integrand), C.POINTER(mcb_config), _PD,
                                       C.POINTER(mcb_iteration), _U32, C.POINTER(mcb_result),
                                       C.POINTER(mcb_iteration), _U32, OBSERVER, _VP]),
    "mcb_run_create": (C.c_int, [_VP, C.POINTER(mcb_integrand), C.POINTER(mcb_config), C.POINTER(_VP)]),
    "mcb_run_destroy": (C.c_int, [_VP]),
    "mcb_run_exchange_words": (_U64, [_VP, _U32]),
    "mcb_run_set_exchange": (C.c_int, [_VP, _VP]),
    "mcb_run_set_progress": (C.c_int, [_VP, _VP]),
    "mcb_run_failure_key": (C.c_int, [_VP, C.POINTER(C.c_int), C.POINTER(_U64)]),
    "mcb_run_set_failure_key": (C.c_int, [_VP, _U64]),
    "mcb_run_set_peers": (C.c_int, [_VP, C.c_int, C.c_int, C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP), _VP]),
    "mcb_dev_alloc": (C.c_int, [_VP, _U64, C.POINTER(_VP)]),
    "mcb_dev_free": (C.c_int, [_VP, _VP]),
    "mcb_ipc_handle": (C.c_int, [_VP, _VP, C.c_char_p]),
    "mcb_ipc_open": (C.c_int, [_VP, C.c_char_p, C.POINTER(_VP)]),
    "mcb_ipc_close": (C.c_int, [_VP, _VP]),
    "mcb_run_resume": (C.c_int, [_VP, _PD, C.POINTER(mcb_iteration), _U32, C.POINTER(_U32)]),
    "mcb_run_exchange_ptr": (_VP, [_VP]),
    "mcb_run_work_items": (_U64, [_VP]),
    "mcb_run_sample": (C.c_int, [_VP, _U32, _U64, _U64]),
    "mcb_run_reduce": (C.c_int, [_VP, _U32]),
    "mcb_run_finish": (C.c_int, [_VP, _U32]),
    "mcb_run_compact_len": (_U64, [_VP]),
    "mcb_run_round_local": (C.c_int, [_VP, _U32, _VP]),
    "mcb_run_combine": (C.c_int, [_VP, _U32, _VP, C.c_int]),
    "mcb_run_finish_rounded": (C.c_int, [_VP, _U32]),
    "mcb_run_result": (C.c_int, [_VP, C.POINTER(mcb_result), C.POINTER(mcb_iteration), _U32]),
    "mcb_run_set_grid": (C.c_int, [_VP, _PD]),
    "mcb_run_grid": (C.c_int, [_VP, _PD]),
}

_lib = None


def lib():
    """Load libmcubes_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2202_01753_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
