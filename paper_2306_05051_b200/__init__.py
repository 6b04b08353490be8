"""B200-native glint evaluation (arXiv 2306.05051) -- distributed binomial
laws on anisotropic grids, as a fused sm_100a kernel behind a C ABI.

    from paper_2306_05051_b200 import Context, glint_eval, synth
    ctx = Context(0)
    frame = synth.c2(25.0, device="cuda")
    rgb = glint_eval(ctx, frame.gbuf, frame.scene)     # (H, W, 4) float32
"""
from ._lib import (Context, GlintError, DEBUG_REC_DTYPE, build_tables, glint_eval, glint_eval_batch,  # noqa: F401
                   glint_eval_host, glint_eval_host_batch, glint_count_active,
                   lib, strerror, version, FLAG_INVALID, FLAG_DEGENERATE, FLAG_RATIO_CLAMPED,
                   FLAG_P_CLAMPED, FLAG_UV_RANGE)
from . import synth  # noqa: F401
