"""LM head + per-token log-probabilities and their gradients, fp64
(the step upstream of ``bd_logprob``).

The policy probabilities in DiPO's importance ratio, pi_theta(o_k | .)
(Eqs. 6-8), are the softmax of the model's
output logits at the token's position; the logits are the LM head applied to
the final hidden states.  The paper does not write the LM head out; SDAR /
Qwen3 use a bias-free linear projection onto the vocabulary [ext], so

    z_{n,v}  = sum_c h_{n,c} W_{v,c}                  (z = h W^T)
    logp_n   = z_{n,t_n} - ln sum_v exp z_{n,v}        (oracle.logprob)
    dz_{n,v} = w_n (1[v = t_n] - softmax(z_n)_v)       (oracle.logprob_grad)
    dh       = dz W,      dW = dz^T h                  (chain rule through z = h W^T)

with w_n = dL/dlogp_n.  The fused GPU path never materialises z; this oracle
does (it is the plain definition).

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import numpy as np

from .attention import _f64
from .logprob import logprob as _logprob, logprob_grad as _logprob_grad


def logits(h, W):
    """z [N, V] fp64 = h [N, C] @ W[V, C]^T."""
    h, W = _f64(h), _f64(W)
    if h.ndim != 2 or W.ndim != 2 or h.shape[1] != W.shape[1]:
        raise ValueError("h must be [N, C] and W [V, C]")
    return h @ W.T


def lmhead_logprob(h, W, targets):
    """(logp [N], lse [N]) fp64 of the logits h W^T at the given targets."""
    return _logprob(logits(h, W), targets)


def lmhead_logprob_grad(h, W, targets, w):
    """(dh [N, C], dW [V, C]) fp64 for upstream gradient w = dL/dlogp [N]."""
    h, W = _f64(h), _f64(W)
    dz = _logprob_grad(logits(h, W), targets, w)
    return dz @ W, dz.T @ h
