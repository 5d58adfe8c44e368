"""B200-native (sm_100a) DCDS block-motion-estimation hot path (Jia & Zhang, arxiv 0806.0689).

The product is the C-ABI library ``libme.so`` (include/me.h) built from ``csrc/``;
``me`` is its thin Python binding (marshalling only) and ``synth`` the seeded synthetic
input generator.  There is no CPU fallback.
"""
from . import synth  # noqa: F401
from .me import (  # noqa: F401
    ALGS, MEError, alloc_outputs, load, me_bma_batch, me_dcds, me_dcds_batch, me_dcds_batch_host, me_dcds_s_batch,
    me_fullsearch, me_fullsearch_batch, me_init, me_launch_count, me_mc_psnr, me_mc_sse_batch,
    me_quality_batch, me_set_stream, me_shutdown, me_ideal_nsp_map, me_mv_hist,
    me_dcds_trace_batch, decode_trace, me_dcds_batch_packed, me_dcds_overflow_count,
)
