"""B200-native polynomial Reed-Solomon (arXiv 1312.5155): C-ABI library + thin binding.

    from paper_1312_5155_b200 import Plan
    plan = Plan(10, 4)            # RS(10,4) over GF(2^8), prim poly 0x11D, alpha = 2
    plan.encode_batch(stripes)    # stripes: torch.uint8 CUDA tensor [S][14][B]
    plan.decode_batch(stripes, erasures)   # erasures: int32 [S][4], -1 padded
"""
from .rs_poly import (DEFAULT_POLY, LIB_PATH, SYNTH_PATH, Plan, RSError, abi_version, launch_count,  # noqa: F401
                      RS_OK, RS_ERR_INVALID_ARG, RS_ERR_NOT_PRIMITIVE, RS_ERR_GEOMETRY, RS_ERR_TOO_MANY_ERASURES,
                      RS_ERR_BAD_ERASURE, RS_ERR_CUDA, RS_ERR_NOMEM, RS_JIT_OFF, RS_JIT_BACKGROUND, RS_JIT_SYNC,
                      RS_READ_ALL_SURVIVORS, RS_READ_K_SURVIVORS, strerror, synth_fill)

__all__ = ["Plan", "RSError", "synth_fill", "launch_count", "abi_version", "strerror", "DEFAULT_POLY"]
