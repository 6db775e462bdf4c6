"""Parity metrics (SURVEY §8(c) "Parity procedure"): computed on the host in
fp64 against the fp64 oracle evaluated on the upcast bf16 inputs."""

import numpy as np

# BASELINE.json north star tolerances
FWD_MAX_ABS = 2e-2
FWD_REL_L2 = 1e-2
GRAD_REL_L2 = 3e-2
LOGP_MAX_ABS = 1e-3   # proposed (north star silent), SURVEY §8(c)
DZ_REL_L2 = 1e-2      # proposed


def metrics(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    diff = got - ref
    fin = np.isfinite(got).all()
    nref = np.linalg.norm(ref)
    return {
        "max_abs": float(np.abs(diff).max()) if diff.size else 0.0,
        "rel_l2": float(np.linalg.norm(diff) / nref) if nref > 0 else float(np.linalg.norm(diff)),
        "finite": bool(fin),
    }


def assert_fwd(name, got, ref):
    m = metrics(got, ref)
    assert m["finite"], (name, m)
    assert m["max_abs"] <= FWD_MAX_ABS and m["rel_l2"] <= FWD_REL_L2, (name, m)
    return m


def assert_grad(name, got, ref):
    m = metrics(got, ref)
    assert m["finite"], (name, m)
    assert m["rel_l2"] <= GRAD_REL_L2, (name, m)
    return m


def t2np(t):
    import torch
    return t.detach().to("cpu", torch.float64).numpy()
