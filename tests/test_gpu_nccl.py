"""The NCCL transport of the engine (one process per GPU, `spt_comm_init_rank`) on the one GPU this
environment has: a single-rank NCCL group.  spt_comm_init_rank creates a real 1-rank communicator
(ncclCommInitRank) and the step's all-reduces (count, loss sum, grads) and the position-id all-gather
(packed) are issued as real ncclAllReduce / ncclAllGather calls; the step must be bitwise equal to the
loopback group's (SP=1: every collective is an identity).  A 1-rank group issues no all-to-all (P = 1 has no
reshard), and NCCL refuses two ranks on one GPU ("Duplicate GPU detected"), so the multi-rank grouped
send/recv stays unexecuted here; multi-rank exchange is tested with the peer transport (test_gpu_peer.py).
(pytest -m gpu)"""
import numpy as np
import pytest

from oracle import sptrain_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_13996_b200 as S  # noqa: E402

CFG = O.LayerConfig(hidden=256, q_heads=4, kv_heads=2, head_dim=128, intermediate=512, vocab=2048)
SHAPE = S.ModelShape(256, 4, 2, 128, 512, 2048)


def _step(grp, packed, N=1024, seed=5):
    p = O.synth_params(CFG, seed)
    x, lab, pos = O.synth_batch(CFG, N, seed, packed=packed)
    eng = S.UlyssesLayerStep(SHAPE, N, grp, packed=packed, n_layers=2)
    try:
        for i in range(2):
            for k in O.LAYER_NAMES:
                eng.set_param(f"layers.{i}.{k}", O.f32_to_bf16_bits(p[k]))
        eng.set_param("g3", O.f32_to_bf16_bits(p["g3"]))
        eng.set_param("wlm", O.f32_to_bf16_bits(p["wlm"]))
        loss, cnt = eng.step(O.f32_to_bf16_bits(x), lab, pos if packed else None)
        grads = {k: eng.grad(k) for k in ("layers.0.wqkv", "layers.1.wd", "g3", "wlm")}
        stats = grp_stats(grp)
    finally:
        eng.close()
    return loss, cnt, grads, stats


def grp_stats(grp):
    import ctypes as C
    import json

    b = C.create_string_buffer(1 << 16)
    S.check(S.lib().spt_comm_stats_json(grp.handle, b, len(b)))
    return json.loads(b.value.decode())


@pytest.mark.parametrize("packed", [False, True])
def test_single_rank_nccl_group_matches_loopback(packed):
    lb = S.ProcessGroup.loopback_group(1)
    try:
        ref = _step(lb, packed)
    finally:
        lb.close()
    nc = S.ProcessGroup.nccl_group(S.ProcessGroup.unique_id(), 1, 0, 0)
    try:
        got = _step(nc, packed)
    finally:
        nc.close()
    assert got[0] == ref[0] and got[1] == ref[1]
    for k in ref[2]:
        assert np.array_equal(got[2][k], ref[2][k]), k
    # the NCCL group really issued the step's collectives
    calls = got[3]
    assert any("all_reduce" in k for k in json_keys(calls)), calls
    if packed:
        assert any("all_gather" in k for k in json_keys(calls)), calls


def json_keys(d):
    out = []
    if isinstance(d, dict):
        for k, v in d.items():
            out.append(k)
            out.extend(json_keys(v))
    elif isinstance(d, list):
        for v in d:
            out.extend(json_keys(v))
    return out
