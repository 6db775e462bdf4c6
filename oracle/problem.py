"""Problem statement of one block-diffusion attention call (oracle copy).

Parameters follow the paper's statement of the problem: prompt ("input")
length, response ("output") length and block size B ("each block
contains B tokens"; "input length 1024, output length 8192"), plus the
GQA head counts and head_dim of the SDAR/Qwen3 model family.

Packed-sequence reading (reading c1/c2, P:251, P:259-261, S:213,
S:250): per sequence the token axis is [x0 | xt] where x0 holds the clean
copy of clean positions 0..L-1 and xt the noisy copy of clean positions
xb..L-1, with xb = 0 when the prompt is repeated too (DiRL, Fig. 4b,
``repeat_prompt=1``) and xb = P when only the response is repeated
(TraceRL, Fig. 4a, ``repeat_prompt=0``).

Trace replay (reading c19): Eq. 6
conditions every decoded token o_k in tau_i(t) on the prefix tau_i(1:t-1),
the block's state *before* decoding step t.  With S decoding steps per block
(static decoding, B/S tokens per step) the packed axis becomes
[x0 | xt^(1) | ... | xt^(S)]: copy s holds every block's state before step s
("one NOISY copy of that block holding the block's state BEFORE
step t").  ``n_copies`` = S; S = 1 is the single-copy DiRL layout.

This module is part of the oracle and deliberately independent of the
package's own problem struct.
"""

from dataclasses import dataclass
import math


@dataclass(frozen=True)
class Problem:
    batch: int
    prompt_len: int
    response_len: int
    block_size: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    repeat_prompt: int = 1
    softmax_scale: float = 0.0  # <= 0 -> 1/sqrt(head_dim)  ("qk^T/sqrt(d)")
    n_copies: int = 1           # S noisy copies (trace replay, reading c19)

    @property
    def L(self) -> int:
        """Clean length L = P + R."""
        return self.prompt_len + self.response_len

    @property
    def xb(self) -> int:
        """First clean position that has a noisy copy."""
        return 0 if self.repeat_prompt else self.prompt_len

    @property
    def n_noisy(self) -> int:
        return self.L - self.xb

    @property
    def ntot(self) -> int:
        """Packed length: L + S (L - xb); 2L (DiRL) or 2L - P (response-only) at S = 1."""
        return self.L + self.n_copies * self.n_noisy

    @property
    def scale(self) -> float:
        return self.softmax_scale if self.softmax_scale > 0 else 1.0 / math.sqrt(self.head_dim)

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    def validate(self) -> None:
        if min(self.batch, self.block_size, self.n_q_heads, self.n_kv_heads, self.head_dim) <= 0:
            raise ValueError("non-positive dimension")
        if self.prompt_len < 0 or self.response_len < 0 or self.L <= 0:
            raise ValueError("bad lengths")
        if self.n_copies < 1:
            raise ValueError("n_copies < 1")
        if self.n_q_heads % self.n_kv_heads:
            raise ValueError("n_q_heads % n_kv_heads != 0")
        # S:214 "length not multiple of B -> layout error" (reading c4)
        if self.L % self.block_size:
            raise ValueError("L % block_size != 0")

    def kv_head_of(self, h: int) -> int:
        """Reading c7: contiguous grouping, kv = floor(h / (Hq/Hkv))."""
        return h // self.group
