"""Brute-force visibility *sets* for tiny inputs.

Written independently of ``oracle/mask.py``: instead of comparing block ids
element-wise, it enumerates blocks and unions whole sets of tokens, following
the prose of the paper:

* x0 block k sees x0 blocks 0..k (clean tokens attend block-causally);
* xt block k sees x0 blocks 0..k-1 and its own xt block, bidirectionally
  (Eq. 2: p(b^k_0 | b^k_t, b^{<k}));
* x0 never sees xt.

Pure Python loops -- only for small cases.
"""


def visibility_sets(L, P, B, repeat_prompt, n_copies=1):
    """Return (tokens, vis) where tokens[n] = (segment, clean_pos) in packed
    order [x0 | xt^(1) | ... | xt^(S)] and vis[n] is the set of visible packed
    indices.  Trace replay (S copies): copy s of block k is its own
    conditioning state -- it sees the clean blocks < k and itself only."""
    xb = 0 if repeat_prompt else P
    tokens = [("x0", p) for p in range(L)]
    for c in range(1, n_copies + 1):
        tokens += [("xt%d" % c, p) for p in range(xb, L)]
    # group packed indices by (segment, block)
    blocks = {}
    for n, (seg, p) in enumerate(tokens):
        blocks.setdefault((seg, p // B), set()).add(n)
    n_blocks = L // B
    vis = []
    for n, (seg, p) in enumerate(tokens):
        k = p // B
        s = set()
        if seg == "x0":
            for kk in range(0, k + 1):
                s |= blocks.get(("x0", kk), set())
        else:
            for kk in range(0, k):
                s |= blocks.get(("x0", kk), set())
            s |= blocks.get((seg, k), set())
        assert k < n_blocks
        vis.append(s)
    return tokens, vis


def read_grid(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.rstrip("\n")
            if not line or line.startswith("#") and set(line) - set("#."):
                continue
            rows.append([c == "#" for c in line])
    return rows
