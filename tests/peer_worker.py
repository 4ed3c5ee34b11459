"""Rank bodies of the multi-process peer-transport tests (tests/test_gpu_peer.py).

Each rank is its own process with its own CUDA context; on the one-GPU test box every rank runs on cuda:0,
and the peer transport maps the other processes' buffers with CUDA IPC exactly as it does across GPUs
(there, over NVLink).  torch.distributed (gloo) is only the bootstrap that all-gathers the IPC handles."""
from __future__ import annotations

import os
import time

import numpy as np


def _init(rank, world, port, device=0):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(device)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return torch, dist


def engine_case(rank, world, port, outdir, cfg_kw, N, seed, packed, rope, graph, transport="peer", multi_gpu=False):
    """One layer step on this rank's sequence shard through a peer (or NCCL) group; saves loss, grads, dx.
    multi_gpu: rank r runs on cuda:r (one process per GPU, as under torchrun) instead of every rank on cuda:0."""
    device = rank if multi_gpu else 0
    torch, dist = _init(rank, world, port, device)
    import paper_2506_13996_b200 as S
    from oracle import sptrain_oracle as O

    cfg = O.LayerConfig(**cfg_kw)
    shape = S.ModelShape(cfg.hidden, cfg.q_heads, cfg.kv_heads, cfg.head_dim, cfg.intermediate, cfg.vocab)
    params = O.synth_params(cfg, seed)
    x, lab, pos = O.synth_batch(cfg, N, seed, packed=packed)
    n_loc = N // world
    sl = slice(rank * n_loc, (rank + 1) * n_loc)
    if transport == "nccl":
        uid = [S.ProcessGroup.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        grp = S.ProcessGroup.nccl_group(uid[0], world, rank, device)
    else:
        grp = S.ProcessGroup.peer_group(world, rank, device, timeout_ms=60000)
    assert grp.transport == transport
    eng = S.UlyssesLayerStep(shape, N, grp, packed=packed, rope_theta=rope)
    for k in O.LayerParams.NAMES:
        eng.set_param(k, O.f32_to_bf16_bits(params[k]))
    xb = O.f32_to_bf16_bits(x)[sl].copy()
    lab_r = lab[sl].copy()
    pos_r = pos[sl].copy() if packed else None
    loss, cnt = eng.step(xb, lab_r, pos_r)
    out = dict(loss=np.float64(loss), count=np.int64(cnt), dx=eng.dx_bits(n_loc))
    for k in O.LayerParams.NAMES:
        out["g_" + k] = eng.grad(k)
    if graph:  # a captured step replays bit-identically (the barrier epochs live on the device)
        dev = torch.device("cuda", device)
        xd = torch.from_numpy(xb.view(np.int16)).to(dev)
        ld = torch.from_numpy(lab_r).to(dev)
        pd = torch.from_numpy(pos_r).to(dev) if packed else None
        s = torch.cuda.Stream(dev)
        eng.graph_capture(xd, ld, pd, stream=s.cuda_stream)
        for _ in range(2):
            eng.graph_launch(stream=s.cuda_stream)
        gl, gc = eng.read_loss(stream=s.cuda_stream)
        out["graph_loss"] = np.float64(gl)
        out["graph_dx"] = eng.dx_bits(n_loc)
        out["graph_g_wqkv"] = eng.grad("wqkv")
    out["stats"] = np.frombuffer(repr(grp.stats()).encode(), np.uint8)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    eng.close()
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


def collectives_case(rank, world, port, outdir):
    """all_reduce (f32 / f64 / i64), all_to_all, seq_to_head / head_to_seq through a peer group."""
    torch, dist = _init(rank, world, port)
    import paper_2506_13996_b200 as S

    grp = S.ProcessGroup.peer_group(world, rank, 0, timeout_ms=60000)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(100 + rank)
    out = {}
    # all-reduce: symmetric buffers from grp.alloc, filled with this rank's values
    n = 10_007
    vals = {"f32": rng.standard_normal(n).astype(np.float32), "f64": rng.standard_normal(n),
            "i64": rng.integers(-1 << 40, 1 << 40, n)}
    bufs = {k: grp.alloc(v.nbytes) for k, v in vals.items()}
    a2a_bytes = 4096 + 48
    send = grp.alloc(a2a_bytes * world)
    recv = grp.alloc(a2a_bytes * world)
    # reshard: Hq=8, Hkv=2, d=32 over `world` ranks (r = world / 2 when world > 2)
    hq, hkv, d, s_loc = 8, 2, 32, 96
    plan = S.plan_head_shards(hq, hkv, world)
    qkv_loc = plan.q_heads_per_rank + 2 * plan.kv_heads_per_rank
    head_side = grp.alloc(world * s_loc * qkv_loc * d * 2)
    grp.connect()
    for k, v in vals.items():
        t = torch.from_numpy(v.view(np.uint8)).to(dev)
        torch.cuda.synchronize()
        _dev_copy(torch, bufs[k], t)
    payload = rng.integers(0, 256, a2a_bytes * world, dtype=np.uint8)
    _dev_copy(torch, send, torch.from_numpy(payload).to(dev))
    torch.cuda.synchronize()
    for k in vals:
        grp.all_reduce(bufs[k], n, k)
    grp.all_to_all(send, recv, a2a_bytes)
    # seq_to_head of a q|k|v shard, then head_to_seq of the result as if it were d(q|k|v): the round trip
    # gives back q exactly and each kv head times its replica count
    qkv = rng.standard_normal((s_loc, hq + 2 * hkv, d)).astype(np.float32)
    qkv_bits = _bf16(qkv)
    src = torch.from_numpy(qkv_bits.view(np.int16)).to(dev)
    back = torch.empty_like(src)
    grp.seq_to_head(plan, 0, src.data_ptr(), s_loc, d, head_side)
    head_copy = torch.empty(world * s_loc * qkv_loc * d, dtype=torch.int16, device=dev)
    _dev_copy(torch, head_copy.data_ptr(), None, src_ptr=head_side, nbytes=head_copy.numel() * 2)
    grp.head_to_seq(plan, 1, head_side, s_loc, d, back.data_ptr())
    grp.wait()
    torch.cuda.synchronize()
    for k in vals:
        out["ar_" + k] = _read(torch, bufs[k], vals[k].nbytes).view(vals[k].dtype)
    out["a2a"] = _read(torch, recv, a2a_bytes * world)
    out["payload"] = payload
    out["qkv_bits"] = qkv_bits
    out["head"] = head_copy.cpu().numpy().view(np.uint16)
    out["back"] = back.cpu().numpy().view(np.uint16)
    for k, v in vals.items():
        out["in_" + k] = v
    out["stats"] = np.frombuffer(repr(grp.stats()).encode(), np.uint8)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


def timeout_case(rank, world, port, outdir):
    """Rank 1 never enters the collective: rank 0's barrier must give ProtocolError after the timeout."""
    torch, dist = _init(rank, world, port)
    import paper_2506_13996_b200 as S

    grp = S.ProcessGroup.peer_group(world, rank, 0)
    grp.set_timeout_ms(1500)
    buf = grp.alloc(4096)
    grp.connect()
    result = "none"
    if rank == 0:
        t0 = time.time()
        try:
            grp.all_reduce(buf, 1024, "f32")
            grp.wait()
            result = "no error"
        except S.ProtocolError as e:
            result = f"ProtocolError after {time.time() - t0:.1f}s: {e}"
    with open(os.path.join(outdir, f"rank{rank}.txt"), "w") as f:
        f.write(result)
    dist.barrier()  # rank 1 leaves only after rank 0 has seen the timeout
    grp.close()
    dist.destroy_process_group()


def _bf16(a):
    from oracle import sptrain_oracle as O

    return O.f32_to_bf16_bits(a)


def _dev_copy(torch, dst_ptr, src_tensor, src_ptr=None, nbytes=None):
    import ctypes as C

    cudart = _cudart()
    if src_tensor is not None:
        src_ptr, nbytes = src_tensor.data_ptr(), src_tensor.numel() * src_tensor.element_size()
    rc = cudart.cudaMemcpy(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), C.c_size_t(nbytes), 3)
    assert rc == 0, rc


def _read(torch, p, nbytes):
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    _dev_copy(torch, out.data_ptr(), None, src_ptr=p, nbytes=nbytes)
    return out.cpu().numpy()


_CUDART = None


def _cudart():
    """The CUDA runtime torch already loaded (raw-pointer copies to / from the group's buffers)."""
    global _CUDART
    if _CUDART is None:
        import ctypes as C

        import torch

        torch.cuda.init()
        _CUDART = C.CDLL("libcudart.so.12")
    return _CUDART
