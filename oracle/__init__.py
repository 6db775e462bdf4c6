"""fp64 CPU oracle for the DiRL/DiPO block-diffusion training hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the C-ABI library
under ``paper_2512_22234_b200/`` and its Python binding) may import, call,
link or execute anything in this package.  The only permitted users are
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg.

The oracle is the plain definition of what the path computes, written from
arXiv 2512.22234 (``/root/reference/PAPER.md``, cited as ``P:<line>``) and the
companion spec (``SPEC.md``, cited as ``S:<line>``):

* ``mask``      -- the block-diffusion visibility rule over the packed
                   sequence [x0 | xt].
* ``attention`` -- naive masked softmax attention, its analytic gradient
                   (S:51-59), fp64 throughout.
* ``logprob``   -- log-softmax gather and its gradient (P:78 CE).
* ``dipo``      -- group advantages and the DiPO / DAPO token-level
                   reduction at the stop-gradient behaviour policy
                   (S:462-479).
* ``lmhead``    -- LM head z = h W^T followed by the log-softmax gather, and
                   its gradients dh, dW.
* ``decode``    -- blockwise KV-cache decode attention and the dynamic
                   threshold token selection (P:62-83,
                   P:312).
* ``tilemap``   -- 128x128 tile classification computed *from the dense
                   mask* (FULL / PARTIAL / EMPTY), the definition the GPU
                   tile-map builder must match bit-exactly.

It shares no code with the CUDA path.  Every function is pinned by
``tests/test_oracle_*.py`` against values that do not come from the oracle
itself (brute force, closed forms, library special cases, finite
differences).  Parity status of each function is listed in DESIGN.md §3.
"""

from .problem import Problem  # noqa: F401
from . import mask, attention, logprob, dipo, tilemap, lmhead, decode  # noqa: F401
