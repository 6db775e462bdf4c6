"""B200-native block-diffusion training attention for DiRL / DiPO (arXiv 2512.22234).

Python binding of the C-ABI library ``libbdattn.so`` (include/bd_attn.h).
"""

from .ops import (  # noqa: E402,F401
    Problem, attn_fwd, attn_bwd, block_diffusion_attention, BlockDiffusionAttention, logprob, tilemap_dump,
    tilemap_stats, packed_len, workspace_bytes, logprob_bwd, lmhead_logprob, lmhead_logprob_bwd, decode_attn,
    decode_select,
)
