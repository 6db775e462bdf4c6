"""Per-token log-probabilities and their gradient, fp64.

The numerators of DiPO's importance ratio (Eqs. 6-8, P:150-156, P:190-196,
P:216-218) are pi_theta(o_k | tau_i(1:t-1)); the NELBO CE (Eq. 3) is
-log softmax(z)[target].  The caller chooses which logit rows predict which
tokens (reading c9); this op takes explicit (row, target) pairs (S:69-77
``softmax_cross_entropy``: "numerically stabilized by max-subtraction",
"target out of range -> index error").

    LSE_n   = ln sum_v exp z_{n,v}
    logp_n  = z_{n, t_n} - LSE_n
    dz_{n,v}= w_n (1[v = t_n] - exp(z_{n,v} - LSE_n))     (w_n = dL/dlogp_n)

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import numpy as np

from .attention import _f64


def logprob(z, targets):
    """Return (logp [N] fp64, lse [N] fp64) for logits z [N, V]."""
    z = _f64(z)
    t = np.asarray(targets, dtype=np.int64)
    N, V = z.shape
    if t.shape != (N,):
        raise ValueError("targets must be [N]")
    if N and (t.min() < 0 or t.max() >= V):
        raise IndexError("target out of range")
    mx = z.max(axis=1, keepdims=True)
    lse = (mx + np.log(np.exp(z - mx).sum(axis=1, keepdims=True)))[:, 0]
    logp = z[np.arange(N), t] - lse
    return logp, lse


def logprob_grad(z, targets, w):
    """dz [N, V] fp64 for upstream gradient w = dL/dlogp [N]."""
    z = _f64(z)
    t = np.asarray(targets, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    _, lse = logprob(z, t)
    p = np.exp(z - lse[:, None])
    dz = -p * w[:, None]
    dz[np.arange(z.shape[0]), t] += w
    return dz
