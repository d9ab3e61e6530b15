"""B200-native ADMM light-field super-resolution (arXiv 2206.05047) — the hot path.

``lfsr.Solver`` wraps the C ABI of ``liblfsr.so`` (include/lfsr.h), whose
sm_100a kernels run every step of Algorithm 1/2.  Build with ``build.build()``.
"""
from .lfsr import (Params, Solver, LFSRError, load_library, params_for, psnr, LIB_PATH, EXPORTS,  # noqa: F401
                   STAT_KEYS, GD_STAT_KEYS, strip_plan, LFSR_ERR_INVALID_ARG, LFSR_ERR_STATE,
                   LFSR_ERR_UNSUPPORTED, LFSR_ERR_DIVERGED, rgb_to_ycbcr, ycbcr_to_rgb,
                   color_super_resolve)

__all__ = ["Params", "Solver", "LFSRError", "load_library", "params_for", "psnr", "LIB_PATH", "EXPORTS"]
