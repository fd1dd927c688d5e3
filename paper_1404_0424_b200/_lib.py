"""ctypes binding of libcgmimo_b200.so (the C ABI in include/cgmimo_b200.h).

There is no fallback: if the library is missing or no sm_100 device is
present, the calls raise.  ``symbols()`` lists every exported entry point the
header declares (checked by tests/test_abi.py without a GPU).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcgmimo_b200.so")

CGM_OK, CGM_EINVAL, CGM_EBREAKDOWN, CGM_ECUDA, CGM_ENCCL, CGM_ENOMEM = range(6)
CGM_TRACKER_EXACT, CGM_TRACKER_APPROX = 0, 1
CGM_DEVICE_POINTERS = 0x1
CGM_HD_UPLINK_LAYOUT = 0x2
# sim::Method order (sim.hpp:34)
METHODS = {"chol": 0, "cholesky": 0, "explicit": 0, "cg": 1, "cgls": 2, "neumann": 3}

_vp = C.c_void_p
_int = C.c_int
_long = C.c_long
_dbl = C.c_double
_u64 = C.c_uint64

# name -> (restype, argtypes); mirrors include/cgmimo_b200.h
SIGNATURES = {
    "cgm_ctx_create": (_int, [_int, C.POINTER(_vp)]),
    "cgm_ctx_destroy": (_int, [_vp]),
    "cgm_ctx_set_stream": (_int, [_vp, _vp]),
    "cgm_synchronize": (_int, [_vp]),
    "cgm_ctx_set_kernel_policy": (_int, [_vp, _int]),
    "cgm_ctx_set_profiling": (_int, [_vp, _int]),
    "cgm_ctx_kernel_times": (_int, [_vp, C.POINTER(_dbl), C.POINTER(_dbl), C.POINTER(_long)]),
    "cgm_ctx_kernel_times_kinds": (_int, [_vp, C.POINTER(_dbl), C.POINTER(_long)]),
    "cgm_ctx_kernel_timeline": (_int, [_vp, C.POINTER(_int), C.POINTER(_dbl), C.POINTER(_dbl),
                                       _long, C.POINTER(_long)]),
    "cgm_ctx_kernel_times_ex": (_int, [_vp, C.POINTER(_dbl), C.POINTER(_dbl), C.POINTER(_dbl),
                                       C.POINTER(_long)]),
    "cgm_last_error": (C.c_char_p, [_vp]),
    "cgm_kernel_launches": (_long, [_vp]),
    "cgm_version": (C.c_char_p, []),
    "cgm_detect_cg": (_int, [_vp, _int, _int, _long, _int, _vp, _vp, _dbl, _dbl, _dbl, _int, _int,
                             _int, _vp, _vp, _vp, _vp, _vp, C.c_uint]),
    "cgm_precode_cg": (_int, [_vp, _int, _int, _long, _int, _vp, _vp, _dbl, _int, _vp, _vp, _vp,
                              _vp, C.c_uint]),
    "cgm_detect": (_int, [_vp, _int, _int, _int, _long, _int, _vp, _vp, _dbl, _dbl, _dbl, _int,
                          _int, _int, _vp, _vp, _vp, _vp, _vp, C.c_uint]),
    "cgm_precode": (_int, [_vp, _int, _int, _int, _long, _int, _vp, _vp, _dbl, _int, _vp, _vp,
                           _vp, _vp, C.c_uint]),
    "cgm_detect_precode_cg": (_int, [_vp, _int, _int, _long, _int, _vp, _vp, _dbl, _dbl, _dbl,
                                     _int, _int, _int, _vp, _vp, _vp, _vp, _vp, _int, _vp, _dbl,
                                     _int, _vp, _vp, _vp, _vp, C.c_uint]),
    "cgm_generate_uplink": (_int, [_vp, _int, _int, _long, _long, _int, _u64, _int, _dbl, _vp,
                                   _vp, _vp]),
    "cgm_generate_downlink": (_int, [_vp, _int, _int, _long, _long, _int, _u64, _int, _vp, _vp,
                                     _vp]),
    "cgm_generate_symbols": (_int, [_vp, _int, _long, _long, _int, _u64, _int, _vp, _vp]),
    "cgm_generate_uplink_correlated": (_int, [_vp, _int, _int, _long, _long, _int, _u64, _int,
                                              _dbl, _vp, _vp, _vp, _vp]),
    "cgm_uplink_trials": (_int, [_vp, _int, _int, _int, _int, _int, _int, _dbl, _long, _vp, _vp,
                                 _vp]),
    "cgm_sweep_trials": (_int, [_vp, _int, _int, _int, _int, _int, _int, _int, _int, _dbl, _long,
                                _vp, _vp, _vp]),
    "cgm_downlink_trials": (_int, [_vp, _int, _int, _int, _int, _int, _dbl, _long, _vp, _vp,
                                   _vp]),
    "cgm_sweep_trial_key": (_u64, [_u64, _int, _long, _long]),
    "cgm_viterbi_decode": (_int, [_vp, _vp, _long, _long, _vp]),
    "cgm_comm_unique_id": (_int, [C.c_char_p]),
    "cgm_comm_create": (_int, [_vp, _int, _int, C.c_char_p, C.POINTER(_vp)]),
    "cgm_comm_destroy": (_int, [_vp]),
    "cgm_gather": (_int, [_vp, _vp, _vp, C.POINTER(C.c_size_t), _vp, _int]),
    "cgm_gatherv": (_int, [_vp, _vp, _vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), _vp,
                           _int]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def symbols() -> list[str]:
    return sorted(SIGNATURES)
