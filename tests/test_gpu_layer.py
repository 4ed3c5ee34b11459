"""End-to-end parity of the Ulysses layer step (C-ABI engine) against the CPU oracle (pytest -m gpu).

Tolerance contract (BASELINE.json north_star): loss rel-err <= 1e-3, grad rel-err <= 2e-2 (norm-wise),
bf16 storage with fp32 accumulation on the GPU vs float64 oracle on identical bf16 inputs.
"""
import numpy as np
import pytest

from oracle import sptrain_oracle as O
from tests.gpu_util import rel_err, torch

pytestmark = pytest.mark.gpu

import paper_2506_13996_b200 as S  # noqa: E402

LOSS_TOL = 1e-3
GRAD_TOL = 2e-2
CFG = O.LayerConfig(hidden=256, q_heads=8, kv_heads=2, head_dim=32, intermediate=1024, vocab=32000)  # config T
SHAPE = S.ModelShape(256, 8, 2, 32, 1024, 32000)


def _run(P, N, packed=False, mlp_tiles=0, loss_tile=0, seed=0, cfg=CFG, shape=SHAPE):
    params = O.synth_params(cfg, seed)
    x, lab, pos = O.synth_batch(cfg, N, seed, packed=packed)
    grp = S.ProcessGroup.loopback_group(P)
    eng = S.UlyssesLayerStep(shape, N, grp, mlp_tiles=mlp_tiles, loss_tile=loss_tile, packed=packed)
    for k in O.LayerParams.NAMES:
        eng.set_param(k, O.f32_to_bf16_bits(params[k]))
    xb = O.f32_to_bf16_bits(x)
    loss, cnt = eng.step(xb, lab, pos if packed else None)
    grads = {k: eng.grad(k) for k in O.LayerParams.NAMES}
    dx = O.bf16_bits_to_f32(eng.dx_bits(N))
    mem = eng.memory()
    stats = grp.stats()
    eng.close()
    grp.close()
    return dict(loss=loss, count=cnt, grads=grads, dx=dx, params=params, x=x, lab=lab, pos=pos, mem=mem, stats=stats)


def _oracle(r, P=1, packed=False, cfg=CFG):
    p = O.LayerParams(**r["params"])
    return O.layer_step(p, cfg, r["x"], r["lab"], r["pos"] if packed else None, P=P)


@pytest.mark.parametrize("packed", [False, True])
def test_layer_step_matches_oracle(packed):
    N = 1024
    r = _run(1, N, packed=packed)
    ref = _oracle(r, packed=packed)
    assert r["count"] == ref.count
    assert abs(r["loss"] - ref.loss) / abs(ref.loss) <= LOSS_TOL
    for k in O.LayerParams.NAMES:
        e = rel_err(r["grads"][k], ref.grads[k])
        assert e <= GRAD_TOL, (k, e)
    assert rel_err(r["dx"], ref.dx) <= GRAD_TOL


@pytest.mark.parametrize("P", [2, 4, 8])
def test_ulysses_sp_equals_sp1(P):
    """SPEC.md:345 on the GPU: SP=P (loopback virtual ranks, real K1/K2 + all_to_all) vs the oracle;
    P=4/8 exercise kv replication r=2/4 (Hkv=2)."""
    N = 1024
    r = _run(P, N)
    ref = _oracle(r, P=1)
    assert r["count"] == ref.count
    assert abs(r["loss"] - ref.loss) / abs(ref.loss) <= LOSS_TOL
    for k in O.LayerParams.NAMES:
        e = rel_err(r["grads"][k], ref.grads[k])
        assert e <= GRAD_TOL, (k, e)
    assert rel_err(r["dx"], ref.dx) <= GRAD_TOL
    # CommStats: actual GQA payload bytes per rank
    plan = O.plan_head_shards(8, 2, P)
    n_loc = N // P
    qkv_loc = plan.q_heads_per_rank + 2 * plan.kv_heads_per_rank
    col = r["stats"]["collectives"]
    assert col["all_to_all_qkv"]["bytes_sent_per_rank"] == n_loc * qkv_loc * 32 * 2 * (P - 1)
    assert col["all_to_all_o"]["bytes_sent_per_rank"] == n_loc * plan.q_heads_per_rank * 32 * 2 * (P - 1)


def test_tiling_invariance_gpu():
    """SPEC.md:416 on the GPU: loss and grads independent of the tile counts (within fp tolerance)."""
    a = _run(1, 1024, mlp_tiles=1, loss_tile=1024)
    b = _run(1, 1024, mlp_tiles=7, loss_tile=128)
    assert a["count"] == b["count"]
    assert abs(a["loss"] - b["loss"]) / abs(a["loss"]) < 1e-5
    for k in O.LayerParams.NAMES:
        assert rel_err(b["grads"][k], a["grads"][k]) < 5e-3, k
    # ledger: largest logits allocation == tile * V * 4 (+ dlogits and row buffers)
    big = a["mem"]["ledger"]["largest_single"]["logits"]
    small = b["mem"]["ledger"]["largest_single"]["logits"]
    assert small < big / 4


def test_step_is_deterministic():
    a = _run(1, 512, seed=3)
    b = _run(1, 512, seed=3)
    assert a["loss"] == b["loss"]
    for k in O.LayerParams.NAMES:
        assert np.array_equal(a["grads"][k], b["grads"][k]), k


def test_invalid_label_raises():
    grp = S.ProcessGroup.loopback_group(1)
    eng = S.UlyssesLayerStep(SHAPE, 256, grp)
    x = np.zeros((256, 256), np.uint16)
    lab = np.full(256, 5, np.int64)
    lab[3] = 32000
    with pytest.raises(S.ValidationError):
        eng.step(x, lab)
    eng.close()
    grp.close()


def test_bad_sp_degree_rejected():
    grp = S.ProcessGroup.loopback_group(3)
    with pytest.raises(S.ValidationError, match="q_heads not divisible by SP degree"):
        S.UlyssesLayerStep(SHAPE, 384, grp)
    grp.close()


# ---- head_dim 128 shapes: the layer step runs the tcgen05 attention kernels (fwd_tc / dkdv_tc / dq_tc)
D128 = O.LayerConfig(hidden=256, q_heads=4, kv_heads=2, head_dim=128, intermediate=512, vocab=2048)
D128_SHAPE = S.ModelShape(256, 4, 2, 128, 512, 2048)
QWENISH = O.LayerConfig(hidden=320, q_heads=4, kv_heads=1, head_dim=128, intermediate=640, vocab=1024)  # h != Hq*d
QWENISH_SHAPE = S.ModelShape(320, 4, 1, 128, 640, 1024)


@pytest.mark.parametrize("P,packed", [(1, False), (2, False), (4, True), (4, False)])
def test_layer_tc_attention_matches_oracle(P, packed):
    """Llama-like head_dim 128 (tcgen05 attention) at SP=1/2/4 (loopback); P=4 with Hkv=2 replicates kv (r=2)."""
    N = 1024
    r = _run(P, N, packed=packed, cfg=D128, shape=D128_SHAPE)
    ref = _oracle(r, packed=packed, cfg=D128)
    assert r["count"] == ref.count
    assert abs(r["loss"] - ref.loss) / abs(ref.loss) <= LOSS_TOL
    for k in O.LayerParams.NAMES:
        e = rel_err(r["grads"][k], ref.grads[k])
        assert e <= GRAD_TOL, (k, e)
    assert rel_err(r["dx"], ref.dx) <= GRAD_TOL


@pytest.mark.parametrize("P", [1, 4])
def test_layer_hidden_ne_heads_times_dim(P):
    """Qwen3-style shape (attention width Hq*d != hidden) with MQA-like Hkv=1 (r=P)."""
    N = 1024
    r = _run(P, N, cfg=QWENISH, shape=QWENISH_SHAPE)
    ref = _oracle(r, cfg=QWENISH)
    assert abs(r["loss"] - ref.loss) / abs(ref.loss) <= LOSS_TOL
    for k in O.LayerParams.NAMES:
        e = rel_err(r["grads"][k], ref.grads[k])
        assert e <= GRAD_TOL, (k, e)


def test_set_param_rejects_wrong_sizes():
    """The C-ABI copies spt_layer_param_numel elements from the caller's pointer; the Python mirror checks the
    buffer's size first, so a weight of another shape (e.g. W_o as [h, h] where Hq*d != h) fails loudly instead
    of being read out of bounds."""
    shape = S.ModelShape(256, 4, 2, 128, 512, 2048)  # Hq*d = 512 != h = 256
    grp = S.ProcessGroup.loopback_group(1)
    eng = S.UlyssesLayerStep(shape, 256, grp)
    try:
        assert eng.param_numel("wo") == 256 * 512 and eng.param_numel("wqkv") == (4 + 4) * 128 * 256
        with pytest.raises(S.ShapeError):
            eng.set_param("wo", np.zeros(256 * 256, np.uint16))
        with pytest.raises(S.ValidationError):
            eng.param_numel("nope")
        eng.set_param("wo", np.zeros(256 * 512, np.uint16))
    finally:
        eng.close()
        grp.close()
