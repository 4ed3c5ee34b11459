"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every symbol the public
header declares, and its host-side logic (SPEC ops that need no device) matches the oracle and the
reference's golden vectors.  Compute entry points are only called to check that they fail without a GPU."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

from oracle import sptrain_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def S():
    import paper_2506_13996_b200 as S

    if not os.path.exists(S.LIB_PATH):
        from paper_2506_13996_b200 import build as B

        B.build()
    S.lib()
    return S


def test_exports_every_header_symbol(S):
    hdr = open(os.path.join(ROOT, "include", "sptrain_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = sorted(set(re.findall(r"\b(spt_[a-z0-9_]+)\s*\(", hdr)))
    assert len(names) >= 40
    raw = C.CDLL(S.LIB_PATH)
    missing = [n for n in names if not hasattr(raw, n)]
    assert not missing, missing
    # and every header symbol has a binding in the Python mirror
    assert not [n for n in names if n not in S.SIGNATURES], [n for n in names if n not in S.SIGNATURES]


def test_version(S):
    assert b"sm_100a" in S.lib().spt_version()


@pytest.mark.parametrize("case", G["head_plans"], ids=lambda c: f"{c['Hq']}-{c['Hkv']}-{c['P']}")
def test_plan_matches_golden_and_oracle(S, case):
    p = S.plan_head_shards(case["Hq"], case["Hkv"], case["P"])
    assert (p.q_heads_per_rank, p.kv_heads_per_rank, p.kv_replication) == (case["q_per_rank"], case["kv_per_rank"],
                                                                           case["r"])
    po = O.plan_head_shards(case["Hq"], case["Hkv"], case["P"])
    for r in range(case["P"]):
        assert S.heads_of(p, r, 0) == po.q_heads_of(r)
        assert S.heads_of(p, r, 1) == po.kv_heads_of(r)


@pytest.mark.parametrize("case", G["head_plans_rejected"], ids=lambda c: f"{c['Hq']}-{c['Hkv']}-{c['P']}")
def test_plan_rejections(S, case):
    with pytest.raises(S.ValidationError):
        S.plan_head_shards(case["Hq"], case["Hkv"], case["P"])


def test_plan_message(S):
    with pytest.raises(S.ValidationError, match=r"q_heads not divisible by SP degree.*\[1, 3, 9\]"):
        S.plan_head_shards(9, 1, 8)


def test_plan_sweep_matches_oracle(S):
    for Hq in range(1, 65):
        for Hkv in [k for k in range(1, Hq + 1) if Hq % k == 0]:
            for P in [p for p in range(1, Hq + 1) if Hq % p == 0]:
                try:
                    po = O.plan_head_shards(Hq, Hkv, P)
                except O.ValidationError:
                    with pytest.raises(S.ValidationError):
                        S.plan_head_shards(Hq, Hkv, P)
                    continue
                pc = S.plan_head_shards(Hq, Hkv, P)
                assert (pc.q_heads_per_rank, pc.kv_heads_per_rank, pc.kv_replication) == (
                    po.q_heads_per_rank, po.kv_heads_per_rank, po.kv_replication)


def test_preshift_pad_blockcausal(S):
    for c in G["preshift"]:
        assert S.preshift_labels(c["labels"]).tolist() == c["shift"]
    rng = np.random.default_rng(0)
    v = rng.integers(0, 100, 37)
    assert np.array_equal(S.preshift_labels(v), O.preshift_labels(v))
    c = G["pad"]
    ids, pos, lab = S.pad_to_multiple(np.arange(c["s"]), np.arange(c["s"]), np.arange(c["s"]), c["P"])
    oi, op, ol = O.pad_to_multiple(np.arange(c["s"]), np.arange(c["s"]), np.arange(c["s"]), c["P"])
    assert ids.size == c["padded_s"] and np.array_equal(lab, ol) and np.array_equal(pos, op) and np.array_equal(ids, oi)
    bc = G["block_causal"]
    assert S.block_causal_starts(bc["position_ids"]).tolist() == O.block_causal_starts(bc["position_ids"]).tolist()
    with pytest.raises(S.ValidationError):
        S.block_causal_starts([0, 2])


@pytest.mark.parametrize("Hq,Hkv,P", [(32, 8, 8), (8, 2, 4), (64, 8, 8), (32, 4, 8)])
def test_a2a_counts_match_payloads(S, Hq, Hkv, P):
    """CommStats accounting: actual GQA payload per peer."""
    p = S.plan_head_shards(Hq, Hkv, P)
    s_loc, d = 1024, 128
    for direction, per in ((0, p.q_heads_per_rank + 2 * p.kv_heads_per_rank), (1, p.q_heads_per_rank),
                           (2, p.q_heads_per_rank), (3, p.q_heads_per_rank + 2 * p.kv_heads_per_rank)):
        send, recv = S.a2a_counts(p, s_loc, d, direction)
        assert (send == s_loc * per * d).all() and (recv == send).all()


def test_no_cpu_fallback(S):
    """Without a B200 every compute entry point fails loudly (SPT_ERR_CUDA-class status and a message): there
    is no CPU fallback on the product path.  Skipped where a GPU is visible."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    L = S.lib()
    h = C.c_void_p()
    assert L.spt_comm_init_loopback(1, 0, C.byref(h)) != 0
    assert L.spt_last_error()
    st = L.spt_attn_fwd(None, 256, 2, 1, 128, None, 0.1, None, None, None)
    assert st != 0 and L.spt_last_error()
    st = L.spt_embed_fwd(None, 8, 16, 8, None, None, None, None)
    assert st != 0
