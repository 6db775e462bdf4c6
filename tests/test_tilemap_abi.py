"""CPU tests of the C-ABI library: symbols, validation, host tile-map path
(bit-exact vs the oracle's dense-mask classification)."""

import ctypes
import os
import re

import pytest

import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib
from oracle import Problem as OProblem, tilemap
from workloads import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "bd_attn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    for n in names:
        assert n in _lib.SIGNATURES, f"binding lacks {n}"


def test_validation_errors():
    L = _lib.lib()
    p = bd.Problem(1, 3, 4, 2, 2, 2, 64).c()  # L = 7, B = 2
    assert L.bd_packed_len(ctypes.byref(p)) == -1
    assert L.bd_attn_workspace_bytes(ctypes.byref(p), 0) == 0
    assert b"multiple" in L.bd_last_error()
    p = bd.Problem(1, 4, 4, 2, 3, 2, 64).c()  # Hq % Hkv != 0
    assert L.bd_packed_len(ctypes.byref(p)) == -1
    rc = L.bd_attn_fwd(ctypes.byref(bd.Problem(1, 4, 4, 2, 2, 2, 64).c()), None, None, None, None, None, None, 0,
                       None)
    assert rc == 1  # BD_ERR_INVALID_ARG
    rc = L.bd_attn_fwd(ctypes.byref(bd.Problem(1, 4, 4, 2, 2, 2, 96).c()), 16, 16, 16, 16, 16, 16, 1 << 20, None)
    assert rc == 3  # BD_ERR_UNSUPPORTED head_dim
    rc = L.bd_attn_fwd(ctypes.byref(bd.Problem(1, 4, 4, 2, 2, 2, 64).c()), 8, 16, 16, 16, 16, 16, 1 << 20, None)
    assert rc == 4  # BD_ERR_ALIGNMENT
    rc = L.bd_attn_fwd(ctypes.byref(bd.Problem(1, 4, 4, 2, 2, 2, 64).c()), 16, 16, 16, 16, 16, 16, 8, None)
    assert rc == 5  # BD_ERR_WORKSPACE
    assert L.bd_error_string(5) == b"BD_ERR_WORKSPACE"


def test_packed_len_and_workspace():
    for cfg in CONFIGS.values():
        p = bd.Problem.from_cfg(cfg)
        assert bd.packed_len(p) == cfg.ntot
        assert bd.workspace_bytes(p, True) > bd.workspace_bytes(p, False) > 0
    p = bd.Problem(1, 10, 20, 5, 1, 1, 64, repeat_prompt=0)
    assert bd.packed_len(p) == 50


def _cases():
    for P, R, B, rp in [(32, 64, 4, 1), (0, 256, 4, 1), (0, 384, 128, 1), (64, 320, 8, 1), (40, 160, 8, 1),
                        (40, 160, 8, 0), (100, 300, 4, 0), (0, 512, 256, 1), (0, 512, 1, 1), (24, 0, 1, 0),
                        (130, 126, 2, 1), (7, 121, 128, 1), (300, 600, 300, 1), (5, 5, 10, 0),
                        # block sizes that do not divide 128 (blocks straddle tile edges) and
                        # response-only mode with P % B != 0 (first noisy row mid-block)
                        (36, 264, 12, 1), (42, 258, 12, 0), (42, 214, 8, 0), (48, 336, 48, 1),
                        (50, 334, 48, 0), (96, 288, 96, 1), (100, 284, 96, 0), (0, 600, 200, 1),
                        (130, 470, 200, 0), (33, 267, 3, 0)]:
        yield P, R, B, rp


@pytest.mark.parametrize("P,R,B,rp", list(_cases()))
def test_tilemap_bit_exact_vs_oracle(P, R, B, rp):
    """bd_tilemap_dump == tile kinds read off the oracle's dense mask."""
    got = bd.tilemap_dump(bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp))
    ref = tilemap.classify(OProblem(1, P, R, B, 1, 1, 64, repeat_prompt=rp))
    assert got == ref


@pytest.mark.parametrize("S", [2, 3])
@pytest.mark.parametrize("P,R,B,rp", [c for i, c in enumerate(_cases()) if i % 2 == 0 or c[3] == 0])
def test_tilemap_copies_bit_exact_vs_oracle(P, R, B, rp, S):
    """Trace replay (S noisy copies, reading c19): same bit-exact bar."""
    p = bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S)
    assert bd.packed_len(p) == OProblem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S).ntot == p.ntot
    got = bd.tilemap_dump(p)
    ref = tilemap.classify(OProblem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S))
    assert got == ref
    c = ctypes.c_int64(-1)
    if p.ntot <= 4096:
        assert _lib.lib().bd_tilemap_selfcheck(ctypes.byref(p.c()), ctypes.byref(c)) == 0 and c.value == 0


@pytest.mark.parametrize("name", ["sdar_1_7b", "sdar_8b", "sweep_b4", "sweep_b32"])
def test_tilemap_configs_closed_form(name):
    """Aligned configs: T^2 + 2T non-empty of 4T^2, 3T PARTIAL."""
    cfg = CONFIGS[name]
    st = bd.tilemap_stats(bd.Problem.from_cfg(cfg))
    T = cfg.L // 128
    assert st["tiles"] == 2 * T
    assert st["nonempty"] == T * T + 2 * T
    assert st["partial"] == 3 * T


def test_tilemap_sdar_1_7b_vs_oracle_dense():
    """Bit-exact at a BJ config (L = 2560, dense mask 5120^2)."""
    cfg = CONFIGS["sdar_1_7b"]
    got = bd.tilemap_dump(bd.Problem.from_cfg(cfg))
    ref = tilemap.classify(OProblem(1, cfg.prompt_len, cfg.response_len, cfg.block_size, 1, 1, 128))
    assert got == ref


def test_host_image_layout():
    img = bd.ops.tilemap_host_image(bd.Problem(1, 32, 64, 4, 2, 2, 64))
    assert img[0] == 0x42444D31 and img[4] == 2 and img[6] == 3


@pytest.mark.parametrize("P,R,B,rp", [(2, 6, 2, 1), (2, 6, 2, 0), (40, 160, 8, 0), (7, 121, 128, 1), (0, 512, 256, 1),
                                      (100, 300, 4, 0), (5, 5, 10, 0), (24, 0, 1, 0), (130, 126, 2, 1)])
def test_row_and_key_intervals_agree(P, R, B, rp):
    """The transpose interval view of the dK/dV kernel equals the row view."""
    p = bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp).c()
    n = ctypes.c_int64(-1)
    assert _lib.lib().bd_tilemap_selfcheck(ctypes.byref(p), ctypes.byref(n)) == 0
    assert n.value == 0


def test_varlen_validation_and_workspace(monkeypatch):
    """Per-sequence lengths are checked on the host (S:214 layout errors)."""
    monkeypatch.setenv("BD_BWD_DS", "0")  # compare map / vector space only (no stored-dS buffer)
    L = _lib.lib()
    ok = bd.Problem(3, 64, 320, 4, 4, 2, 128, seq_prompt_lens=(64, 32, 0), seq_response_lens=(320, 96, 200))
    assert bd.packed_len(ok) == 2 * 384
    ws_u = bd.workspace_bytes(bd.Problem(3, 64, 320, 4, 4, 2, 128), True)
    assert bd.workspace_bytes(ok, True) > ws_u > 0  # one map per sequence
    for P_, R_ in [((64, 33, 0), (320, 96, 200)),   # L % B != 0
                   ((65, 32, 0), (320, 96, 200)),   # P_i > prompt_len
                   ((64, 32, 0), (320, 96, 0))]:    # empty sequence
        p = bd.Problem(3, 64, 320, 4, 4, 2, 128, seq_prompt_lens=P_, seq_response_lens=R_)
        assert L.bd_attn_workspace_bytes(ctypes.byref(p.c()), 1) == 0
        assert L.bd_packed_len(ctypes.byref(p.c())) == -1
    half = bd.Problem(3, 64, 320, 4, 4, 2, 128, seq_prompt_lens=(64, 32, 0))
    assert L.bd_packed_len(ctypes.byref(half.c())) == -1


def test_row_length_within_capacity_stride_random():
    """Every q-tile's entry count fits the per-q-tile stride (capacity / NT)
    that the device builder stages entries with -- including block sizes that
    do not divide 128 and xb % B != 0 (a regression: B = 48, P = 50,
    response-only overflowed the stride and corrupted the device map)."""
    import random
    rng = random.Random(7)
    cases = [(50, 334, 48, 0, 1), (100, 284, 96, 0, 1), (130, 470, 200, 0, 1), (36, 264, 12, 1, 3)]
    for _ in range(300):
        B = rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 16, 24, 32, 48, 64, 96, 100, 128, 200, 256, 300])
        K = rng.randint(1, max(1, 1500 // B))
        L = K * B
        P = rng.randint(0, L)
        cases.append((P, L - P, B, rng.randint(0, 1), rng.choice([1, 1, 2, 3])))
    for P, R, B, rp, S in cases:
        if P + R - (0 if rp else P) <= 0:
            continue
        img = bd.ops.tilemap_host_image(bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S))
        NT, maxrow = img[4], img[7]
        cap = (len(img) - 16 - 2 * (NT + 1) - 2 * NT) // 3
        assert maxrow <= cap // NT, (P, R, B, rp, S, maxrow, cap // NT)


@pytest.mark.parametrize("name", ["sdar_8b", "sweep_b4", "sweep_b8", "sweep_b16", "sweep_b32"])
def test_tilemap_bj_configs_vs_oracle_dense(name):
    """bd_tilemap_dump equals the classification read off the
    oracle's dense mask at every BASELINE attention config (SDAR-8B: the full
    18,432^2 mask; SDAR-1.7B above)."""
    cfg = CONFIGS[name]
    got = bd.tilemap_dump(bd.Problem.from_cfg(cfg))
    ref = tilemap.classify(OProblem(1, cfg.prompt_len, cfg.response_len, cfg.block_size, 1, 1, cfg.head_dim))
    assert got == ref


def test_tilemap_varlen_sequences_vs_oracle_dense():
    """sdar_8b_varlen: the per-sequence maps are those of each sequence's own
    (P, R_i) -- shortest, median and longest rollout checked dense."""
    cfg = CONFIGS["sdar_8b_varlen"]
    lens = sorted(cfg.resp_lens)
    for R in (lens[0], lens[len(lens) // 2], lens[-1]):
        got = bd.tilemap_dump(bd.Problem(1, cfg.prompt_len, R, cfg.block_size, 1, 1, 128))
        ref = tilemap.classify(OProblem(1, cfg.prompt_len, R, cfg.block_size, 1, 1, 128))
        assert got == ref, R


def test_col_rpos_and_entries_bound():
    """The map's column-to-row-entry index (where the dK/dV kernel stores a
    tile's dS^T and the dQ kernel reads it, row by row): for every column entry
    of k-tile kt naming q-tile t, row_ent[col_rpos] is kt and lies in row t's
    range; every row entry is named exactly once.  And the O(NT) entry count
    from the candidate ranges equals the builder's count (every candidate tile
    is non-empty) on the BJ shapes and a randomised sweep of block sizes,
    prompt lengths, modes and copies."""
    import random
    rng = random.Random(5)
    cases = [(1024, 8192, 4, 1, 1), (512, 2048, 4, 1, 1), (1024, 8192, 4, 1, 4), (100, 300, 4, 0, 1),
             (50, 334, 48, 0, 1), (36, 264, 12, 1, 3), (7, 121, 128, 1, 1), (42, 214, 8, 0, 2)]
    for _ in range(150):
        B = rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 16, 32, 48, 64, 96, 128, 200, 300])
        K = rng.randint(1, max(1, 1200 // B))
        L = K * B
        cases.append((rng.randint(0, L), 0, B, rng.randint(0, 1), rng.choice([1, 1, 2, 3])))
        P = cases[-1][0]
        cases[-1] = (P, L - P, B, cases[-1][3], cases[-1][4])
    for P, R, B, rp, S in cases:
        if R <= 0 or (P + R - (0 if rp else P)) <= 0:
            continue
        prob = bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S)
        img = bd.ops.tilemap_host_image(prob)
        NT, n = img[4], img[6]
        cap = (len(img) - 16 - 2 * (NT + 1) - 2 * NT) // 3
        rp_, re = 16, 16 + NT + 1
        cp = re + cap
        ce = cp + NT + 1
        cr = ce + cap + 2 * NT
        seen = [0] * n
        for kt in range(NT):
            for c in range(img[cp + kt], img[cp + kt + 1]):
                t = img[ce + c] & 0x0FFFFFFF
                e = img[cr + c]
                assert img[rp_ + t] <= e < img[rp_ + t + 1], (P, R, B, rp, S, kt, t, e)
                assert img[re + e] & 0x0FFFFFFF == kt
                seen[e] += 1
        assert seen == [1] * n
        assert bd.ops.tilemap_entries_bound(prob) == n, (P, R, B, rp, S)
