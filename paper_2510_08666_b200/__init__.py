"""B200-native denoise-and-commit step of dInfer (arXiv 2510.08666).

The product is libdinfer.so (hand-written sm_100a CUDA kernels behind the C ABI
in include/dinfer.h); `dinfer` is its thin ctypes binding.  `synth` holds the
seeded synthetic input generators (no method arithmetic).
"""
from .dinfer import (DEC_HIERARCHICAL, DEC_THRESHOLD, Context, DInferError, GenConfig, Params,  # noqa: F401
                     VicinityKV, alpha_schedule, get_unique_id, lib, make_gen_config, make_params, tau_schedule)
