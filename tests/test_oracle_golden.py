"""Pin the CPU oracle against every known-answer vector the reference holds (SPEC.md/PAPER.md)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import sptrain_oracle as O

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("case", G["head_plans"], ids=lambda c: f"{c['Hq']}-{c['Hkv']}-{c['P']}")
def test_head_plans(case):
    p = O.plan_head_shards(case["Hq"], case["Hkv"], case["P"])
    assert (p.q_heads_per_rank, p.kv_heads_per_rank, p.kv_replication) == (
        case["q_per_rank"], case["kv_per_rank"], case["r"])
    qs = sorted(h for r in range(case["P"]) for h in p.q_heads_of(r))
    assert qs == list(range(case["Hq"]))  # SPEC.md:291 disjoint union


@pytest.mark.parametrize("case", G["head_plans_rejected"], ids=lambda c: f"{c['Hq']}-{c['Hkv']}-{c['P']}")
def test_head_plans_rejected(case):
    with pytest.raises(O.ValidationError):
        O.plan_head_shards(case["Hq"], case["Hkv"], case["P"])


def test_head_plan_message_q9():
    with pytest.raises(O.ValidationError, match=r"q_heads not divisible by SP degree.*\[1, 3, 9\]"):
        O.plan_head_shards(9, 1, 8)


def test_head_plan_sweep():
    """SPEC.md:701 exhaustive sweep: Hq <= 64, Hkv | Hq, P | Hq."""
    for Hq in range(1, 65):
        for Hkv in [k for k in range(1, Hq + 1) if Hq % k == 0]:
            for P in [p for p in range(1, Hq + 1) if Hq % p == 0]:
                ok = (Hkv >= P and Hkv % P == 0) or (Hkv < P and P % Hkv == 0)
                if not ok:
                    with pytest.raises(O.ValidationError):
                        O.plan_head_shards(Hq, Hkv, P)
                    continue
                p = O.plan_head_shards(Hq, Hkv, P)
                if p.kv_replication > 1:
                    assert p.kv_heads_per_rank == 1 and p.kv_replication * Hkv == P
                kv = [h for r in range(P) for h in p.kv_heads_of(r)]
                assert sorted(set(kv)) == list(range(Hkv))


def test_all_to_all_definitional():
    c = G["all_to_all_2rank"]
    send = [[np.array([hash(x) % 1000]) for x in row] for row in c["send"]]
    names = {hash(x) % 1000: x for row in c["send"] for x in row}
    recv = O.all_to_all(send)
    assert [[names[int(a[0])] for a in row] for row in recv] == c["recv"]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_all_to_all_involution(P):
    rng = np.random.default_rng(P)
    send = [[rng.standard_normal(3) for _ in range(P)] for _ in range(P)]
    back = O.all_to_all(O.all_to_all(send))
    for i in range(P):
        for j in range(P):
            assert np.array_equal(back[i][j], send[i][j])


def test_seq_to_head_example():
    c = G["seq_to_head_P2"]
    x = np.arange(8).reshape(c["x_full_arange"])
    plan = O.plan_head_shards(2, 2, 2)
    ys = O.seq_to_head(O.shard_sequence(x, 2), plan.q_heads_of)
    assert ys[0].ravel().tolist() == c["rank0"]
    assert ys[1].ravel().tolist() == c["rank1"]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_seq_head_roundtrip_and_index_formula(P):
    rng = np.random.default_rng(10 + P)
    H, s, d = 16, 32, 3
    x = rng.standard_normal((s, H, d))
    plan = O.plan_head_shards(H, H, P)
    xs = O.shard_sequence(x, P)
    ys = O.seq_to_head(xs, plan.q_heads_of)
    s_loc, H_loc = s // P, H // P
    for j in range(P):  # y_j[t,h',e] = x_{t//s_loc}[t mod s_loc, j*H_loc+h', e]
        for t in range(s):
            assert np.array_equal(ys[j][t], xs[t // s_loc][t % s_loc, j * H_loc:(j + 1) * H_loc])
    back = O.head_to_seq(ys, plan.q_heads_of, H)
    for a, b in zip(back, xs):
        assert np.array_equal(a, b)


def test_replicate_kv_backward_is_sum():
    """grad of replicated kv = sum of per-rank upstream grads."""
    plan = O.plan_head_shards(4, 1, 4)
    rng = np.random.default_rng(3)
    s = 8
    ys = [rng.standard_normal((s, 1, 2)) for _ in range(4)]
    back = O.head_to_seq(ys, plan.kv_heads_of, 1, reduce_replicas=True)
    full = np.concatenate(back, axis=0)
    assert np.allclose(full, ys[0] + ys[1] + ys[2] + ys[3])


def test_preshift_and_shard():
    for c in G["preshift"]:
        assert O.preshift_labels(c["labels"]).tolist() == c["shift"]
    c = G["shard_after_preshift"]
    ids = O.shard_sequence(np.array(c["input_ids"]), c["P"])
    sh = O.shard_sequence(O.preshift_labels(c["input_ids"]), c["P"])
    assert [a.tolist() for a in ids] == c["ids"]
    assert [a.tolist() for a in sh] == c["shift"]
    # double shift != single shift
    v = np.arange(1, 20)
    assert not np.array_equal(O.preshift_labels(O.preshift_labels(v)), O.preshift_labels(v))


def test_naive_shift_drops_token():
    c = G["naive_shift_after_shard"]
    naive = O.naive_shift_after_shard(c["labels"], c["P"])
    assert [a.tolist() for a in naive] == c["shift"]
    good = np.concatenate(O.shard_sequence(O.preshift_labels(c["labels"]), c["P"]))
    bad = np.concatenate(naive)
    assert c["dropped_token"] in good.tolist() and c["dropped_token"] not in bad.tolist()
    # exactly one supervised token lost per non-final shard
    assert int((good != -100).sum() - (bad != -100).sum()) == c["P"] - 1


def test_pad():
    c = G["pad"]
    ids, pos, lab = O.pad_to_multiple(np.arange(c["s"]), np.arange(c["s"]), np.arange(c["s"]), c["P"])
    assert ids.size == c["padded_s"] and lab[c["s"]:].tolist() == c["pad_labels"]
    assert O.pad_to_multiple(np.arange(8), np.arange(8), np.arange(8), 4)[0].size == 8


def test_block_causal():
    c = G["block_causal"]
    pred = O.block_causal_predicate(c["position_ids"])
    for i, js in c["attends"].items():
        assert [j for j in range(4) if pred(int(i), j)] == js
    with pytest.raises(O.ValidationError):
        O.block_causal_starts([0, 2, 3])
    with pytest.raises(O.ValidationError):
        O.block_causal_starts([1, 2])


def test_block_causal_bruteforce():
    rng = np.random.default_rng(5)
    runs = [int(x) for x in rng.integers(1, 6, size=10)]
    pos = np.concatenate([np.arange(r) for r in runs])
    lab = np.concatenate([np.full(r, i) for i, r in enumerate(runs)])
    pred = O.block_causal_predicate(pos)
    for i in range(pos.size):
        for j in range(pos.size):
            assert pred(i, j) == (j <= i and lab[i] == lab[j])


def test_cross_entropy_known_answers():
    V = G["cross_entropy_uniform"]["V"]
    s, c, _ = O.cross_entropy(np.zeros((1, V)), np.array([3]))
    assert c == 1 and abs(s - math.log(V)) < 1e-12
    s, c, d = O.cross_entropy(np.random.default_rng(0).standard_normal((4, 7)), np.full(4, -100))
    assert (s, c) == (0.0, 0) and not d.any()
    with pytest.raises(O.ValidationError):
        O.cross_entropy(np.zeros((1, 5)), np.array([5]))
    # independent log-softmax-gather formula
    rng = np.random.default_rng(1)
    lg = rng.standard_normal((4, 7))
    lab = np.array([0, 6, -100, 2])
    s, c, _ = O.cross_entropy(lg, lab)
    ref = sum(-(lg[i, lab[i]] - np.log(np.exp(lg[i]).sum())) for i in range(4) if lab[i] != -100)
    assert c == 3 and abs(s - ref) < 1e-12


def test_tiles_and_logits_bytes():
    for c in G["tiled_mlp_tiles"]:
        assert O.default_mlp_tiles(c["s"], c["h"]) == c["tiles"]
    c = G["logits_gib"]
    assert abs(c["seqlen"] * c["vocab"] * c["bytes"] / 2**30 - c["gib"]) < 0.01
