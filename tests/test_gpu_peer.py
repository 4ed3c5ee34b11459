"""The peer-memory transport with real multi-process ranks (pytest -m gpu).

Every rank is a separate process (its own CUDA context, like one process per GPU under torchrun); on the one
GPU this box has, all ranks share cuda:0 and map each other's buffers with CUDA IPC, which is the same
mapping the transport makes across GPUs over NVLink.  Checked against the loopback group (P virtual ranks in
one process, the SPEC's in-process SPMD) and against numpy:
  * a full layer step (fused K1 pack-and-store / K2 load-and-unpack all-to-alls, the fixed-order grad /
    count / loss all-reduces, the position-id all-gather when packed): dx, count and loss BITWISE equal to
    the loopback group, which the layer tests pin to the oracle; weight grads equal up to the association of
    per-tile fp32 partial sums (rel <= 1e-6);
  * all_reduce f32 / f64 / i64 bitwise equal to the rank-ascending numpy sum;
  * all_to_all bit-exact, seq_to_head / head_to_seq round trip with kv replication;
  * a rank that never enters a collective -> ProtocolError on the others after the timeout.
NCCL itself cannot run two ranks on one GPU ("Duplicate GPU detected", profiles/r2_probe_same_gpu.txt), so
its multi-rank path stays unexecuted here; the single-rank NCCL group is tested in test_gpu_nccl.py."""
import ast
import os
import socket

import numpy as np
import pytest

from oracle import sptrain_oracle as O
from tests import peer_worker as W
from tests.gpu_util import rel_err

pytestmark = pytest.mark.gpu

import paper_2506_13996_b200 as S  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, tmp_path, *args):
    import torch.multiprocessing as mp

    mp.start_processes(fn, args=(world, _port(), str(tmp_path), *args), nprocs=world, join=True,
                       start_method="spawn")
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)] if fn is not W.timeout_case else None


def _loopback(cfg, N, world, seed, packed, rope):
    shape = S.ModelShape(cfg.hidden, cfg.q_heads, cfg.kv_heads, cfg.head_dim, cfg.intermediate, cfg.vocab)
    params = O.synth_params(cfg, seed)
    x, lab, pos = O.synth_batch(cfg, N, seed, packed=packed)
    grp = S.ProcessGroup.loopback_group(world)
    eng = S.UlyssesLayerStep(shape, N, grp, packed=packed, rope_theta=rope)
    for k in O.LayerParams.NAMES:
        eng.set_param(k, O.f32_to_bf16_bits(params[k]))
    loss, cnt = eng.step(O.f32_to_bf16_bits(x), lab, pos if packed else None)
    out = dict(loss=loss, count=cnt, dx=eng.dx_bits(N), grads={k: eng.grad(k) for k in O.LayerParams.NAMES})
    eng.close()
    grp.close()
    return out


CASES = {
    # (cfg, N, world, packed, rope, graph)
    "llama_d128_p2": (dict(hidden=256, q_heads=4, kv_heads=2, head_dim=128, intermediate=512, vocab=2048), 1024, 2,
                      False, 0.0, True),
    "tiny_d32_p4_kvrep": (dict(hidden=256, q_heads=8, kv_heads=2, head_dim=32, intermediate=1024, vocab=32000), 1024,
                          4, False, 0.0, False),
    "packed_rope_p2": (dict(hidden=256, q_heads=4, kv_heads=2, head_dim=128, intermediate=512, vocab=2048), 1024, 2,
                       True, 10000.0, False),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_peer_layer_step_bitwise_equals_loopback(case, tmp_path):
    cfg_kw, N, world, packed, rope, graph = CASES[case]
    cfg = O.LayerConfig(**cfg_kw)
    ranks = _spawn(W.engine_case, world, tmp_path, cfg_kw, N, 7, packed, rope, graph)
    ref = _loopback(cfg, N, world, 7, packed, rope)
    n_loc = N // world
    for r, out in enumerate(ranks):
        assert int(out["count"]) == ref["count"]
        assert float(out["loss"]) == ref["loss"], (r, float(out["loss"]), ref["loss"])
        assert np.array_equal(out["dx"], ref["dx"][r * n_loc:(r + 1) * n_loc]), r
        for k in O.LayerParams.NAMES:
            # weight grads: fp32, same terms, but a rank with several TiledMLP / loss tiles sums them before the
            # all-reduce ((r0t0 + r0t1) + (r1t0 + r1t1)), the loopback ranks into one buffer in sequence
            # ((r0t0 + r0t1) + r1t0) + r1t1: equal up to fp32 rounding of the association
            g, gr = out["g_" + k], ref["grads"][k]
            assert np.array_equal(g, gr) or rel_err(g, gr) <= 1e-6, (r, k, rel_err(g, gr))
        st = ast.literal_eval(bytes(out["stats"]).decode())
        assert st["transport"] == "peer" and st["world_size"] == world
        col = st["collectives"]
        for tag in ("all_to_all_qkv", "all_to_all_o", "all_to_all_do", "all_to_all_dqkv", "all_reduce_grads",
                    "all_reduce_count", "all_reduce_loss_sum"):
            assert col[tag]["calls"] >= 1, tag
        if packed:
            assert col["all_gather_position_ids"]["calls"] >= 1
        if graph:
            assert float(out["graph_loss"]) == ref["loss"]
            assert np.array_equal(out["graph_dx"], out["dx"])
            assert np.array_equal(out["graph_g_wqkv"], out["g_wqkv"])


@pytest.mark.parametrize("world", [2, 4])
def test_peer_collectives(world, tmp_path):
    ranks = _spawn(W.collectives_case, world, tmp_path)
    for k in ("f32", "f64", "i64"):
        ins = [r["in_" + k] for r in ranks]
        want = ins[0].copy()
        for v in ins[1:]:
            want = want + v  # ascending rank order
        for r in ranks:
            assert np.array_equal(r["ar_" + k], want), k
    nb = ranks[0]["payload"].size // world
    for i, r in enumerate(ranks):  # recv[j] on rank i = send[i] from rank j
        for j in range(world):
            assert np.array_equal(r["a2a"][j * nb:(j + 1) * nb], ranks[j]["payload"][i * nb:(i + 1) * nb])
    # seq_to_head vs the oracle's definition, then the head_to_seq round trip
    hq, hkv, d, s_loc = 8, 2, 32, 96
    plan = O.plan_head_shards(hq, hkv, world)
    shards = [O.bf16_bits_to_f32(r["qkv_bits"]).reshape(s_loc, hq + 2 * hkv, d) for r in ranks]
    qh = O.seq_to_head([x[:, :hq] for x in shards], plan.q_heads_of)
    kh = O.seq_to_head([x[:, hq:hq + hkv] for x in shards], plan.kv_heads_of)
    vh = O.seq_to_head([x[:, hq + hkv:] for x in shards], plan.kv_heads_of)
    for i, r in enumerate(ranks):
        want = np.concatenate([qh[i], kh[i], vh[i]], axis=1)
        got = O.bf16_bits_to_f32(r["head"]).reshape(world * s_loc, -1, d)
        assert np.array_equal(got, want), i
        back = O.bf16_bits_to_f32(r["back"]).reshape(s_loc, hq + 2 * hkv, d)
        rep = plan.kv_replication
        assert np.array_equal(back[:, :hq], shards[i][:, :hq])
        assert np.array_equal(back[:, hq:], shards[i][:, hq:] * rep)


def test_peer_stalled_rank_raises_protocol_error(tmp_path):
    import torch.multiprocessing as mp

    mp.start_processes(W.timeout_case, args=(2, _port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    msg = open(tmp_path / "rank0.txt").read()
    assert msg.startswith("ProtocolError"), msg
