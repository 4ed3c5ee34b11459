"""SPEC.md:333-341 ulysses_attention as one collective C-ABI op (spt_ulysses_attention_fwd / _bwd) over a loopback
group of P virtual ranks, against the single-rank attention on the whole sequence (pytest -m gpu).

SP invariance: each rank runs the same tcgen05 kernels on its heads over the full sequence,
so the forward output and the backward dQ are BITWISE equal to the P = 1 attention; dK / dV are bitwise equal when
no kv head is replicated (every q head of a GQA group on one rank) and equal to bf16 rounding of the replica sum
(fp32, rank order) when it is.  Packed sequences pass the block-causal run starts of the full
sequence to every rank."""
import math

import numpy as np
import pytest

from oracle import sptrain_oracle as O
from tests.gpu_util import rel_err

pytestmark = pytest.mark.gpu

import paper_2506_13996_b200 as S  # noqa: E402


def torch():
    import torch as T

    return T


def _single(T, L, qkv, s, hq, hkv, d, seg, dout):
    o = T.empty(s, hq, d, dtype=T.bfloat16, device="cuda")
    lse = T.empty(hq, s, device="cuda")
    S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, S.ptr(seg), 1 / math.sqrt(d), o.data_ptr(), lse.data_ptr(),
                           None))
    ws = T.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=T.uint8, device="cuda")
    dqkv = T.empty_like(qkv)
    S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), s, hq, hkv, d, S.ptr(seg),
                           1 / math.sqrt(d), dqkv.data_ptr(), ws.data_ptr(), None))
    T.cuda.synchronize()
    return o, dqkv


@pytest.mark.parametrize("P,hq,hkv,s,packed,d", [(2, 4, 2, 1024, False, 128), (4, 8, 2, 2048, False, 128),
                                                 (2, 4, 2, 1024, True, 128), (8, 8, 2, 2048, False, 128),
                                                 (8, 8, 2, 2048, True, 128), (4, 8, 4, 2048, True, 64),
                                                 (2, 4, 1, 1024, False, 32), (8, 32, 8, 8192, True, 128)])
def test_ulysses_attention_op_matches_single_rank(P, hq, hkv, s, packed, d):
    T = torch()
    L = S.lib()
    rng = np.random.default_rng(5 + P)
    qkv = T.from_numpy(O.f32_to_bf16_bits(rng.standard_normal((s, hq + 2 * hkv, d), dtype=np.float32)).view(np.int16)
                       ).cuda().view(T.bfloat16)
    dout = T.from_numpy(O.f32_to_bf16_bits(rng.standard_normal((s, hq, d), dtype=np.float32)).view(np.int16)
                        ).cuda().view(T.bfloat16)
    seg = None
    if packed:
        runs, tot = [], 0
        while tot < s:
            runs.append(int(rng.integers(64, s // 2)))
            tot += runs[-1]
        pos = np.concatenate([np.arange(r) for r in runs])[:s]
        seg = T.from_numpy(O.block_causal_starts(pos).astype(np.int32)).cuda()
    o_ref, dqkv_ref = _single(T, L, qkv, s, hq, hkv, d, seg, dout)

    plan = S.plan_head_shards(hq, hkv, P)
    ql, kl = plan.q_heads_per_rank, plan.kv_heads_per_rank
    s_loc = s // P
    grp = S.ProcessGroup.loopback_group(P)
    try:
        xs = [qkv[r * s_loc:(r + 1) * s_loc].contiguous() for r in range(P)]
        dos = [dout[r * s_loc:(r + 1) * s_loc].contiguous() for r in range(P)]
        qkv_head = [T.empty(s, ql + 2 * kl, d, dtype=T.bfloat16, device="cuda") for _ in range(P)]
        o_head = [T.empty(s, ql, d, dtype=T.bfloat16, device="cuda") for _ in range(P)]
        lse = [T.empty(ql, s, device="cuda") for _ in range(P)]
        out = [T.empty(s_loc, hq, d, dtype=T.bfloat16, device="cuda") for _ in range(P)]
        sc = 1 / math.sqrt(d)
        grp.ulysses_attention_fwd(plan, xs, s_loc, d, seg, sc, qkv_head, o_head, lse, out)
        do_head = [T.empty(s, ql, d, dtype=T.bfloat16, device="cuda") for _ in range(P)]
        dqkv_head = [T.empty(s, ql + 2 * kl, d, dtype=T.bfloat16, device="cuda") for _ in range(P)]
        ws = [T.empty(L.spt_attn_bwd_workspace(s, ql, kl, d), dtype=T.uint8, device="cuda") for _ in range(P)]
        dqkv = [T.empty(s_loc, hq + 2 * hkv, d, dtype=T.bfloat16, device="cuda") for _ in range(P)]
        grp.ulysses_attention_bwd(plan, qkv_head, o_head, lse, dos, s_loc, d, seg, sc, do_head, dqkv_head, ws, dqkv)
        T.cuda.synchronize()
    finally:
        grp.close()
    o_sp = T.cat(out).view(T.int16).cpu().numpy()
    assert np.array_equal(o_sp, o_ref.view(T.int16).cpu().numpy())
    g = T.cat(dqkv)
    assert T.equal(g[:, :hq], dqkv_ref[:, :hq])  # dQ: the same per-head kernel on the same inputs
    if plan.kv_replication == 1:
        assert T.equal(g, dqkv_ref)
    else:  # replicated kv heads: fp32 rank-order sum of bf16 per-replica partials
        gn, rn = g[:, hq:].float().cpu().numpy(), dqkv_ref[:, hq:].float().cpu().numpy()
        assert rel_err(gn, rn) < 1e-2
