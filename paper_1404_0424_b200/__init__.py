"""paper_1404_0424_b200 -- B200-native (sm_100a) batched CG soft-output MIMO
detection and CG precoding, a drop-in for the reference's
``cgmimo::detect::detect_cg`` / ``cgmimo::precode::precode_cg`` path.

The compute path is ``libcgmimo_b200.so`` (hand-written CUDA + C ABI, see
include/cgmimo_b200.h); this package is the host-side mirror over it.
"""
from ._lib import LIB_PATH, load as load_library, symbols
from .api import (Context, CudaError, SolverBreakdown, default_context, detect_cg,
                  detect_cg_single, precode_cg, precode_cg_single)
from .configs import CONFIGS, Config, get_config
from . import sim  # noqa: E402  (coded BLER sweeps)

__all__ = [
    "LIB_PATH", "load_library", "symbols", "Context", "CudaError", "SolverBreakdown",
    "default_context", "detect_cg", "detect_cg_single", "precode_cg", "precode_cg_single",
    "CONFIGS", "Config", "get_config",
]
