"""World-size-2 (gloo, CPU) coverage of the multi-rank Ulysses path's host logic: the head plan and
the all-to-all schedule come from the C-ABI library, the exchange runs as torch.distributed
all_to_all_single over gloo, and the result must equal the oracle's in-process SPMD seq_to_head /
head_to_seq (bit-exact) and the (loss_sum, count) all-reduce."""
import os
import socket

import numpy as np
import pytest

from oracle import sptrain_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, Hq, Hkv, q):
    import torch
    import torch.distributed as dist

    import paper_2506_13996_b200 as S

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, s_loc = 8, 6
        rng = np.random.default_rng(42)
        xs = [O.round_bf16(rng.standard_normal((s_loc, Hq + 2 * Hkv, d), dtype=np.float32)) for _ in range(world)]
        plan = S.plan_head_shards(Hq, Hkv, world)
        def heads(j):
            return (S.heads_of(plan, j, 0) + [Hq + h for h in S.heads_of(plan, j, 1)] +
                    [Hq + Hkv + h for h in S.heads_of(plan, j, 1)])
        send_counts, recv_counts = S.a2a_counts(plan, s_loc, d, 0)
        # K1 pack (host restatement of the device kernel's index map): send[j] = x[:, heads(j)]
        send = np.concatenate([xs[rank][:, heads(j), :].reshape(-1) for j in range(world)])
        assert send.size == send_counts.sum()
        recv = torch.empty(int(recv_counts.sum()))
        dist.all_to_all_single(recv, torch.from_numpy(send), [int(c) for c in recv_counts],
                               [int(c) for c in send_counts])
        got = recv.numpy().reshape(world * s_loc, len(heads(rank)), d)
        exp = O.seq_to_head(xs, lambda j: heads(j))[rank]
        ok_fwd = bool(np.array_equal(got, exp))
        # reverse (replicate_kv backward sums replicas in rank order)
        g_all = [O.round_bf16(np.random.default_rng(7 + j).standard_normal((world * s_loc, len(heads(j)), d),
                                                                          dtype=np.float32)) for j in range(world)]
        send2 = np.concatenate([g_all[rank][i * s_loc:(i + 1) * s_loc].reshape(-1) for i in range(world)])
        recv2 = torch.empty(send2.size)
        dist.all_to_all_single(recv2, torch.from_numpy(send2))
        parts = recv2.numpy().reshape(world, s_loc, len(heads(rank)), d)
        out = np.zeros((s_loc, Hq + 2 * Hkv, d), np.float32)
        for j in range(world):
            for a, hg in enumerate(heads(j)):
                out[:, hg] += parts[j][:, a]
        exp2 = O.head_to_seq(g_all, lambda j: heads(j), Hq + 2 * Hkv, reduce_replicas=True)[rank]
        ok_bwd = bool(np.allclose(out, exp2, atol=1e-6))
        # (loss_sum, count) reduction
        t = torch.tensor([1.5 * (rank + 1), float(10 + rank)], dtype=torch.float64)
        dist.all_reduce(t)
        ok_red = bool(t.tolist() == [1.5 * sum(r + 1 for r in range(world)), float(sum(10 + r for r in range(world)))])
        q.put((rank, ok_fwd, ok_bwd, ok_red))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Hq,Hkv", [(8, 2), (4, 1)])
def test_ulysses_exchange_world2(Hq, Hkv):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, Hq, Hkv, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, a, b, c in res:
        assert a and b and c, (rank, a, b, c)


# ---- SP-over-DP iteration over gloo, world size 2
def _iter_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2506_13996_b200 as S

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 0's stream: A, B (, E); rank 1's: C, D -> collaborative order A, C, B, D, then stop (min length)
        names = [["A", "B", "E"], ["C", "D"]][rank]

        def batch(nm):
            base = {"A": 1, "B": 100, "C": 200, "D": 300, "E": 400}[nm]
            n = 7 if nm in ("A", "D") else 8  # odd length exercises pad_to_multiple
            return {"input_ids": np.arange(base, base + n, dtype=np.int64),
                    "position_ids": np.arange(n, dtype=np.int64),
                    "labels": np.arange(base, base + n, dtype=np.int64), "name": nm}

        out = []
        for src, ids, pos, lab in S.sp_over_dp_iterator((batch(n) for n in names), None, rank, world):
            out.append((src, ids.tolist(), pos.tolist(), lab.tolist()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sp_over_dp_iterator_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_iter_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    order = [src for src, *_ in res[0]]
    assert order == [0, 1, 0, 1] == [src for src, *_ in res[1]]  # A, C, B, D; E dropped (shortest stream)
    firsts = [res[0][i][1][0] for i in range(4)]
    assert firsts == [1, 200, 100, 300]
    for i in range(4):
        ids = res[0][i][1] + res[1][i][1]
        lab = res[0][i][3] + res[1][i][3]
        pos = res[0][i][2] + res[1][i][2]
        # reconstruction of the padded, pre-shifted source batch
        base = ids[0]
        n = 7 if base in (1, 300) else 8
        src_lab = list(range(base, base + n))
        exp_ids, exp_pos, exp_lab = O.pad_to_multiple(np.arange(base, base + n), np.arange(n),
                                                      O.preshift_labels(np.asarray(src_lab)), 2)
        assert ids == list(exp_ids) and pos == list(exp_pos) and lab == list(exp_lab)
        assert lab[-1] == -100 and len(ids) % 2 == 0
