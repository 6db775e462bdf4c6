"""DiPO objective at the stop-gradient behaviour policy, fp64.

* Group advantage: A_i = r_i - (1/G) sum_j r_j, assigned to every token
  of trajectory i ("its token-level assignment is simply A_{i,k} = A_i").
* Clip operator: C_eps(r, A) = min(r A, clip(r, 1-eps, 1+eps) A).
* Behaviour policy = sg(current policy) (Eq. 7), so the ratio
  rho_k = exp(logp_k - sg(logp_k)) has value 1 and gradient d logp_k.
* Token-level normalisation 1 / sum_i |tau_i| (Eq. 7 / Eq. 8),
  |tau_i| read as the token count (reading c10); the normaliser is taken per
  group as printed inside E_Q and the groups are averaged (reading c11);
  beta = 0 (Eq. 8 has no KL; reading c13).

    J_g    = (1/N_g) sum_{i in g} sum_{k in tau_i} C_eps(rho_k, A_i)
    loss   = -(1/n_groups) sum_g J_g
    dloss/dlogp_k = -(1/(n_groups N_g)) * rho_k * dC/drho

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import numpy as np


def advantages(rewards, group_of_traj):
    """A_i = r_i - mean of r over i's group."""
    r = np.asarray(rewards, dtype=np.float64)
    g = np.asarray(group_of_traj, dtype=np.int64)
    a = np.empty_like(r)
    for gid in np.unique(g):
        sel = g == gid
        a[sel] = r[sel] - r[sel].mean()
    return a


def clip_op(rho, adv, eps):
    """C_eps(r, A) and dC/dr."""
    rho = np.asarray(rho, dtype=np.float64)
    adv = np.asarray(adv, dtype=np.float64)
    unclipped = rho * adv
    clipped = np.clip(rho, 1 - eps, 1 + eps) * adv
    val = np.minimum(unclipped, clipped)
    inside = (rho > 1 - eps) & (rho < 1 + eps)
    # derivative of the selected branch; at a tie both branches agree when
    # rho is inside the clip range
    d = np.where(unclipped <= clipped, adv, np.where(inside, adv, 0.0))
    return val, d


def dipo_loss(logp, logp_old, traj_of_token, rewards, group_of_traj, eps=0.2):
    """Return (loss, dlogp [n_tokens], stats dict)."""
    logp = np.asarray(logp, dtype=np.float64)
    logp_old = np.asarray(logp_old, dtype=np.float64)
    tt = np.asarray(traj_of_token, dtype=np.int64)
    gt = np.asarray(group_of_traj, dtype=np.int64)
    adv = advantages(rewards, gt)
    rho = np.exp(logp - logp_old)
    if not np.all(np.isfinite(rho)):
        raise FloatingPointError("non-finite ratio")  # S:475 abort
    val, dc = clip_op(rho, adv[tt], eps)
    groups = np.unique(gt)
    n_groups = len(groups)
    group_of_token = gt[tt]
    n_g = {gid: int((group_of_token == gid).sum()) for gid in groups}
    loss = 0.0
    dlogp = np.zeros_like(logp)
    for gid in groups:
        sel = group_of_token == gid
        if n_g[gid] == 0:
            continue
        loss -= val[sel].sum() / n_g[gid] / n_groups
        dlogp[sel] = -(rho[sel] * dc[sel]) / (n_g[gid] * n_groups)
    clip_frac = float(np.mean(((rho <= 1 - eps) | (rho >= 1 + eps)) & (rho != 1.0))) if len(rho) else 0.0
    return loss, dlogp, {"n_groups": n_groups, "n_tokens": int(len(logp)),
                         "clip_frac": clip_frac}
