"""B200-native ALST (arXiv 2506.13996) sequence-parallel layer step — Python host mirror.

The product is `libsptrain_b200.so` (C++ host engine + sm_100a CUDA kernels behind the C-ABI in
`include/sptrain_b200.h`).  This module is a thin ctypes binding that mirrors the reference's
operation names (SPEC.md: plan_head_shards, preshift_labels, pad_to_multiple, ProcessGroup,
ulysses layer step).  There is no CPU fallback: if the library is missing or the device is not
sm_100a the calls raise.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsptrain_b200.so")

SPT_OK = 0
STATUS_NAMES = {0: "OK", 1: "SHAPE", 2: "VALIDATION", 3: "COLLECTIVE", 4: "PROTOCOL", 5: "OOM", 6: "CUDA",
                7: "CONFIG", 8: "DETERMINISM", 9: "INTERNAL"}


class SptError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{STATUS_NAMES.get(status, status)}] {msg}")
        self.status = status


class ValidationError(SptError, ValueError):
    """errors.hpp:13"""


class ShapeError(ValidationError):
    """errors.hpp:19"""


class ConfigError(SptError):
    """errors.hpp:68"""


class CollectiveError(SptError):
    """errors.hpp:24-28: a collective saw incompatible payloads across ranks"""


class ProtocolError(CollectiveError):
    """errors.hpp:30-34: ranks diverged from lock-step collective order, or a rank died / timed out"""


class OomError(SptError, MemoryError):
    """errors.hpp:55-65 SimulatedOomError (ledger budget) or a device allocation failure"""


class DeterminismError(SptError):
    """errors.hpp:36-40: a replayed region produced values different from its recorded forward"""


_EXC = {1: ShapeError, 2: ValidationError, 3: CollectiveError, 4: ProtocolError, 5: OomError, 7: ConfigError,
        8: DeterminismError}

_lib = None


class HeadShardPlan(C.Structure):
    """SPEC.md:286-292"""

    _fields_ = [("sp_degree", C.c_int32), ("q_heads", C.c_int32), ("kv_heads", C.c_int32),
                ("q_heads_per_rank", C.c_int32), ("kv_heads_per_rank", C.c_int32), ("kv_replication", C.c_int32)]


class LayerConfig(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("q_heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("intermediate", C.c_int32), ("vocab", C.c_int64), ("seq_len", C.c_int64), ("mlp_tiles", C.c_int32),
                ("loss_tile", C.c_int64), ("rms_eps", C.c_float), ("packed", C.c_int32), ("lr", C.c_float),
                ("n_layers", C.c_int32), ("ckpt_offload", C.c_int32), ("rope_theta", C.c_float),
                ("embed", C.c_int32), ("verify_replay", C.c_int32)]


P = C.c_void_p
I32, I64, F32, SZ = C.c_int32, C.c_int64, C.c_float, C.c_size_t
PI32, PI64, PF32 = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_float)

SIGNATURES = {
    "spt_last_error": (C.c_char_p, []),
    "spt_version": (C.c_char_p, []),
    "spt_tuning_set": (I32, [C.c_char_p, I32]),
    "spt_plan_head_shards": (I32, [I32, I32, I32, C.POINTER(HeadShardPlan)]),
    "spt_plan_heads_of": (I32, [C.POINTER(HeadShardPlan), I32, I32, PI32, I32, PI32]),
    "spt_preshift_labels": (I32, [P, I64, P]),
    "spt_pad_to_multiple": (I32, [P, P, P, I64, I32, I64, PI64]),
    "spt_block_causal_starts": (I32, [P, I64, P]),
    "spt_a2a_counts": (I32, [C.POINTER(HeadShardPlan), I64, I32, I32, P, P]),
    "spt_gemm_bf16": (I32, [P, I64, I32, P, I64, I32, P, I64, I32, I32, P, I64, I64, I64, I64, F32, P]),
    "spt_rmsnorm_fwd": (I32, [P, P, P, P, I64, I64, F32, P]),
    "spt_rmsnorm_bwd_workspace": (SZ, [I64, I64]),
    "spt_rmsnorm_bwd": (I32, [P, P, P, P, P, P, P, P, I64, I64, P]),
    "spt_reshard_pack": (I32, [P, I64, I32, I32, I32, I32, P, P, P]),
    "spt_layer_graph_capture": (I32, [P, P, P, P, P]),
    "spt_layer_graph_launch": (I32, [P, P]),
    "spt_reshard_pack_rope": (I32, [P, I64, I32, I32, I32, I32, P, P, I32, P, I64, F32, P, P]),
    "spt_rope_table": (I32, [P, I64, I32, F32, P]),
    "spt_reshard_unpack": (I32, [P, I64, I32, I32, I32, I32, P, I32, P, P]),
    "spt_attn_fwd": (I32, [P, I64, I32, I32, I32, P, F32, P, P, P]),
    "spt_attn_bwd_workspace": (SZ, [I64, I32, I32, I32]),
    "spt_attn_bwd": (I32, [P, P, P, P, I64, I32, I32, I32, P, F32, P, P, P]),
    "spt_label_stats": (I32, [P, I64, I64, P, P, P]),
    "spt_segment_starts": (I32, [P, I64, P, P, P]),
    "spt_flce_workspace": (SZ, [I64, I64]),
    "spt_rope": (I32, [P, I64, I32, I32, I32, P, I64, F32, I32, P]),
    "spt_embed_fwd": (I32, [P, I64, I64, I64, P, P, P, P]),
    "spt_embed_bwd_workspace": (SZ, [I64, I64]),
    "spt_embed_bwd": (I32, [P, I64, I64, I64, P, P, I32, P, P, P]),
    "spt_memest_fixed_bytes": (I32, [C.c_double, I32, I32, I32, P]),
    "spt_memest_logits_bytes": (C.c_double, [C.c_double, C.c_double, C.c_double]),
    "spt_memest_activation_ckpt_bytes": (I32, [C.c_double, C.c_double, C.c_double, C.c_double, I32, I32, P, P]),
    "spt_memest_4d_mask_bytes": (C.c_double, [C.c_double, C.c_double]),
    "spt_memest_position_ids_bytes": (C.c_double, [C.c_double, C.c_double]),
    "spt_memest_engine_device_bytes": (I32, [P, C.c_double, P]),
    "spt_max_seqlen_solver": (I32, [P, C.c_double, I64, P]),
    "spt_flce": (I32, [P, P, P, I64, I64, I64, I64, P, P, P, P, I32, P, P, P]),
    "spt_mlp_workspace": (SZ, [I64, I64]),
    "spt_mlp_fwd": (I32, [P, P, P, P, P, I64, I64, I64, I64, P, P]),
    "spt_mlp_bwd": (I32, [P, P, P, P, P, P, P, I32, I64, I64, I64, I64, P, P]),
    "spt_comm_unique_id": (I32, [P]),
    "spt_comm_init_rank": (I32, [P, I32, I32, I32, C.POINTER(P)]),
    "spt_comm_init_loopback": (I32, [I32, I32, C.POINTER(P)]),
    "spt_comm_destroy": (I32, [P]),
    "spt_comm_init_peer": (I32, [I32, I32, I32, P, P, C.POINTER(P)]),
    "spt_comm_set_timeout_ms": (I32, [P, I64]),
    "spt_comm_world": (I32, [P, PI32, PI32, PI32]),
    "spt_comm_check": (I32, [P]),
    "spt_comm_wait": (I32, [P, P]),
    "spt_comm_alloc": (I32, [P, SZ, C.POINTER(P)]),
    "spt_comm_free": (I32, [P, P]),
    "spt_comm_connect": (I32, [P]),
    "spt_comm_barrier": (I32, [P, P]),
    "spt_all_reduce_f32": (I32, [P, C.POINTER(P), I64, P]),
    "spt_all_reduce_f64": (I32, [P, C.POINTER(P), I64, P]),
    "spt_all_reduce_i64": (I32, [P, C.POINTER(P), I64, P]),
    "spt_all_to_all": (I32, [P, C.POINTER(P), C.POINTER(P), SZ, P]),
    "spt_reshard_scratch_bytes": (SZ, [C.POINTER(HeadShardPlan), I32, I64, I32]),
    "spt_seq_to_head": (I32, [P, C.POINTER(HeadShardPlan), I32, C.POINTER(P), I64, I32, C.POINTER(P), P, P]),
    "spt_head_to_seq": (I32, [P, C.POINTER(HeadShardPlan), I32, C.POINTER(P), I64, I32, C.POINTER(P), P, P]),
    "spt_ulysses_attention_fwd": (I32, [P, C.POINTER(HeadShardPlan), C.POINTER(P), I64, I32, P, F32, C.POINTER(P),
                                        C.POINTER(P), C.POINTER(P), C.POINTER(P), P, P]),
    "spt_ulysses_attention_bwd": (I32, [P, C.POINTER(HeadShardPlan), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                        C.POINTER(P), I64, I32, P, F32, C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                        C.POINTER(P), P, P]),
    "spt_comm_stats_json": (I32, [P, C.c_char_p, SZ]),
    "spt_layer_create": (I32, [C.POINTER(LayerConfig), P, C.POINTER(P)]),
    "spt_layer_destroy": (I32, [P]),
    "spt_layer_param_numel": (I32, [P, C.c_char_p, C.POINTER(I64)]),
    "spt_layer_set_param": (I32, [P, C.c_char_p, P, I32]),
    "spt_layer_step": (I32, [P, P, P, P, I32, PF32, PI64, P]),
    "spt_layer_step_async": (I32, [P, P, P, P, I32, P]),
    "spt_layer_read_loss": (I32, [P, PF32, PI64, P]),
    "spt_layer_loss_async": (I32, [P, I32, P]),
    "spt_layer_loss_slot": (I32, [P, I32, PF32, PI64]),
    "spt_layer_step_accumulate": (I32, [P, P, P, P, I32, I32, P]),
    "spt_layer_finish_accumulation": (I32, [P, PF32, PI64, P]),
    "spt_layer_get_grad": (I32, [P, C.c_char_p, P]),
    "spt_layer_get_dx": (I32, [P, P]),
    "spt_layer_memory_json": (I32, [P, C.c_char_p, SZ]),
    "spt_layer_memory_timeline_csv": (I32, [P, C.c_char_p, SZ]),
    "spt_layer_set_profiling": (I32, [P, I32]),
    "spt_layer_timing_json": (I32, [P, C.c_char_p, SZ]),
    "spt_kernel_launch_count": (I64, []),
}


def lib():
    """Load the in-tree library (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing — run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    if status != SPT_OK:
        msg = lib().spt_last_error().decode()
        raise _EXC.get(status, SptError)(status, msg)


def ptr(t) -> int | None:
    """Raw pointer of a torch tensor / numpy array / int / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


# ----------------------------------------------------------------- host-only mirror (SPEC ops)
def plan_head_shards(q_heads: int, kv_heads: int, sp: int) -> HeadShardPlan:
    """SPEC.md:296-305"""
    p = HeadShardPlan()
    check(lib().spt_plan_head_shards(q_heads, kv_heads, sp, C.byref(p)))
    return p


def heads_of(plan: HeadShardPlan, rank: int, kind: int) -> list[int]:
    buf = (C.c_int32 * 1024)()
    n = C.c_int32()
    check(lib().spt_plan_heads_of(C.byref(plan), rank, kind, buf, 1024, C.byref(n)))
    return list(buf[: n.value])


def preshift_labels(labels):
    """SPEC.md:512-519"""
    import numpy as np

    a = np.ascontiguousarray(labels, dtype=np.int64)
    out = np.empty_like(a)
    check(lib().spt_preshift_labels(ptr(a), a.size, ptr(out)))
    return out


def pad_to_multiple(input_ids, position_ids, shift_labels, sp: int):
    """SPEC.md:531-535"""
    import numpy as np

    s = len(input_ids)
    n = C.c_int64()
    check(lib().spt_pad_to_multiple(None, None, None, s, sp, 0, C.byref(n)))
    bufs = []
    for a in (input_ids, position_ids, shift_labels):
        b = np.zeros(n.value, dtype=np.int64)
        b[:s] = a
        bufs.append(b)
    check(lib().spt_pad_to_multiple(ptr(bufs[0]), ptr(bufs[1]), ptr(bufs[2]), s, sp, n.value, C.byref(n)))
    return tuple(bufs)


def block_causal_starts(position_ids):
    import numpy as np

    a = np.ascontiguousarray(position_ids, dtype=np.int64)
    out = np.empty_like(a)
    check(lib().spt_block_causal_starts(ptr(a), a.size, ptr(out)))
    return out


# ---------------------------------------------------------------- memest
class MemestFixed(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("weights_bytes", "optimizer_bytes", "master_weights_bytes", "grads_bytes",
                                           "total_bytes", "device_bytes_per_gpu", "host_bytes_per_gpu")]


class MemestEngine(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("q_heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("intermediate", C.c_int32), ("vocab", C.c_int64), ("n_layers", C.c_int32), ("sp", C.c_int32),
                ("ckpt_offload", C.c_int32), ("act_bytes_per_token", C.c_double),
                ("act_bytes_per_seq_token", C.c_double), ("embed", C.c_int32)]


def memest_fixed(param_count: float, world_size: int = 1, zero3: bool = False, offload_optimizer: bool = False):
    out = MemestFixed()
    check(lib().spt_memest_fixed_bytes(float(param_count), world_size, int(zero3), int(offload_optimizer),
                                       C.byref(out)))
    return {n: getattr(out, n) for n, _ in MemestFixed._fields_}


def memest_logits(seqlen, vocab, nbytes=4):
    return lib().spt_memest_logits_bytes(float(seqlen), float(vocab), float(nbytes))


def memest_activation_ckpt(seqlen, hidden, layers, nbytes=2, sp=1, gpus_per_node=8):
    dev, host = C.c_double(), C.c_double()
    check(lib().spt_memest_activation_ckpt_bytes(float(seqlen), float(hidden), float(layers), float(nbytes), sp,
                                                 gpus_per_node, C.byref(dev), C.byref(host)))
    return dev.value, host.value


def memest_4d_mask(seqlen, nbytes=2):
    return lib().spt_memest_4d_mask_bytes(float(seqlen), float(nbytes))


def memest_position_ids(seqlen, nbytes=2):
    return lib().spt_memest_position_ids_bytes(float(seqlen), float(nbytes))


def memest_engine(shape: "ModelShape", n_layers=1, sp=1, ckpt_offload=False, act_bytes_per_token=0.0,
                  act_bytes_per_seq_token=0.0) -> MemestEngine:
    return MemestEngine(shape.hidden, shape.q_heads, shape.kv_heads, shape.head_dim, shape.intermediate, shape.vocab,
                        n_layers, sp, int(ckpt_offload), act_bytes_per_token, act_bytes_per_seq_token)


def memest_engine_bytes(cfg: MemestEngine, seqlen) -> float:
    out = C.c_double()
    check(lib().spt_memest_engine_device_bytes(C.byref(cfg), float(seqlen), C.byref(out)))
    return out.value


def max_seqlen(cfg: MemestEngine, device_budget_bytes, granularity=128) -> int:
    out = C.c_int64()
    check(lib().spt_max_seqlen_solver(C.byref(cfg), float(device_budget_bytes), granularity, C.byref(out)))
    return out.value


def sp_over_dp_iterator(loader, group=None, rank: int = 0, world_size: int = 1):
    """SPEC.md:537-545 / PAPER §4.2 "SP over DP": every rank owns a data stream; the SP group processes ONE
    rank's batch at a time, collaboratively, iterating over ranks: global order rank0's batch 0, rank1's batch
    0, ..., rank(P-1)'s batch 0, rank0's batch 1, ...  Each yielded item is (source_rank, input_ids,
    position_ids, shift_labels) for THIS rank's contiguous sequence shard (already pre-shifted and padded to a
    multiple of P before sharding).

    `loader` yields dicts with int64 numpy arrays "input_ids", "position_ids" and "labels" (unshifted) for
    this rank's stream.  With world_size > 1 the batches are exchanged with torch.distributed broadcasts
    (`group`: a process group, gloo or nccl; only the source rank's batch is sent).  The iterator stops at
    the shortest stream (every rank learns whether the source still has data)."""
    import numpy as np

    it = iter(loader)
    if world_size == 1:
        for b in it:
            ids, pos, lab = pad_to_multiple(b["input_ids"], b["position_ids"], preshift_labels(b["labels"]), 1)
            yield 0, ids, pos, lab
        return
    import torch
    import torch.distributed as dist

    while True:
        mine = next(it, None)
        # a round runs only if EVERY stream still has a batch (stop at the shortest stream)
        have = torch.tensor([0 if mine is None else 1], dtype=torch.int64)
        dist.all_reduce(have, op=dist.ReduceOp.MIN, group=group)
        if int(have.item()) == 0:
            return
        for src in range(world_size):
            n = torch.tensor([len(mine["input_ids"]) if src == rank else 0], dtype=torch.int64)
            dist.broadcast(n, src, group=group)
            buf = torch.empty(3, int(n.item()), dtype=torch.int64)
            if src == rank:
                buf[0] = torch.from_numpy(np.asarray(mine["input_ids"], np.int64))
                buf[1] = torch.from_numpy(np.asarray(mine["position_ids"], np.int64))
                buf[2] = torch.from_numpy(np.asarray(mine["labels"], np.int64))
            dist.broadcast(buf, src, group=group)
            ids, pos, lab = (buf[i].numpy() for i in range(3))
            ids, pos, lab = pad_to_multiple(ids, pos, preshift_labels(lab), world_size)
            s_loc = len(ids) // world_size
            sl = slice(rank * s_loc, (rank + 1) * s_loc)
            yield src, ids[sl], pos[sl], lab[sl]


def a2a_counts(plan: HeadShardPlan, s_loc: int, head_dim: int, direction: int):
    import numpy as np

    s = np.zeros(plan.sp_degree, np.int64)
    r = np.zeros(plan.sp_degree, np.int64)
    check(lib().spt_a2a_counts(C.byref(plan), s_loc, head_dim, direction, ptr(s), ptr(r)))
    return s, r


# ----------------------------------------------------------------- process group + layer engine
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
TRANSPORTS = {0: "loopback", 1: "nccl", 2: "peer"}


def _torch_allgather(group=None):
    """spt_allgather_fn over torch.distributed (any backend): every rank's `bytes` into out, rank order."""

    def fn(inp, out, nbytes, _user):
        try:
            import torch.distributed as dist

            mine = C.string_at(inp, nbytes)
            objs = [None] * dist.get_world_size(group)
            dist.all_gather_object(objs, mine, group=group)
            for r, b in enumerate(objs):
                if len(b) != nbytes:
                    return 2
                C.memmove(out + r * nbytes, b, nbytes)
            return 0
        except Exception:  # noqa: BLE001 - the C side turns a non-zero return into CollectiveError
            return 1

    return ALLGATHER_FN(fn)


class ProcessGroup:
    """loopback virtual ranks on one GPU, NCCL (one process per GPU), or the peer-memory
    transport (one process or thread per GPU; buffers mapped over NVLink, fused reshard collectives)."""

    def __init__(self, handle, world_size: int, rank: int, loopback: bool, keep=None):
        self.handle, self.world_size, self.rank, self.loopback = handle, world_size, rank, loopback
        self._keep = keep  # the exchange callback must outlive the group

    @property
    def transport(self) -> str:
        t = C.c_int32()
        check(lib().spt_comm_world(self.handle, None, None, C.byref(t)))
        return TRANSPORTS[t.value]

    @classmethod
    def peer_group(cls, world_size: int, rank: int, device: int, exchange=None, group=None,
                   timeout_ms: int | None = None) -> "ProcessGroup":
        """Peer-memory group; `exchange(bytes) -> list[bytes]` all-gathers the handle blobs (default:
        torch.distributed.all_gather_object over `group`, which must be initialised)."""
        if exchange is None:
            cb = _torch_allgather(group)
        else:
            def fn(inp, out, nbytes, _user):
                try:
                    blobs = exchange(C.string_at(inp, nbytes))
                    for r, b in enumerate(blobs):
                        C.memmove(out + r * nbytes, b, nbytes)
                    return 0
                except Exception:  # noqa: BLE001
                    return 1
            cb = ALLGATHER_FN(fn)
        h = C.c_void_p()
        check(lib().spt_comm_init_peer(world_size, rank, device, C.cast(cb, C.c_void_p), None, C.byref(h)))
        g = cls(h, world_size, rank, False, keep=cb)
        if timeout_ms is not None:
            g.set_timeout_ms(timeout_ms)
        return g

    def set_timeout_ms(self, ms: int):
        check(lib().spt_comm_set_timeout_ms(self.handle, int(ms)))

    def check(self):
        check(lib().spt_comm_check(self.handle))

    def wait(self, stream=None):
        check(lib().spt_comm_wait(self.handle, ptr(stream)))

    def barrier(self, stream=None):
        check(lib().spt_comm_barrier(self.handle, ptr(stream)))

    def alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        check(lib().spt_comm_alloc(self.handle, nbytes, C.byref(p)))
        return p.value

    def free(self, p: int):
        check(lib().spt_comm_free(self.handle, p))

    def connect(self):
        check(lib().spt_comm_connect(self.handle))

    def _ptrs(self, bufs):
        bufs = bufs if isinstance(bufs, (list, tuple)) else [bufs]
        return (C.c_void_p * len(bufs))(*[ptr(b) for b in bufs])

    def all_reduce(self, bufs, n: int, dtype: str = "f32", stream=None):
        """SPEC.md:155-163 in place; bufs: one per local rank (peer: from alloc())."""
        f = {"f32": lib().spt_all_reduce_f32, "f64": lib().spt_all_reduce_f64, "i64": lib().spt_all_reduce_i64}[dtype]
        check(f(self.handle, self._ptrs(bufs), n, ptr(stream)))

    def all_to_all(self, send, recv, bytes_per_peer: int, stream=None):
        """SPEC.md:145-153"""
        check(lib().spt_all_to_all(self.handle, self._ptrs(send), self._ptrs(recv), bytes_per_peer, ptr(stream)))

    def seq_to_head(self, plan, kind: int, x, s_loc: int, head_dim: int, out, scratch=None, stream=None):
        """SPEC.md:307-315 (K1 with the all-to-all fused)"""
        check(lib().spt_seq_to_head(self.handle, C.byref(plan), kind, self._ptrs(x), s_loc, head_dim, self._ptrs(out),
                                    ptr(scratch), ptr(stream)))

    def head_to_seq(self, plan, kind: int, x, s_loc: int, head_dim: int, out, scratch=None, stream=None):
        """SPEC.md:317-326 (K2 with the all-to-all fused; kind 1 sums kv replicas in rank order)"""
        check(lib().spt_head_to_seq(self.handle, C.byref(plan), kind, self._ptrs(x), s_loc, head_dim, self._ptrs(out),
                                    ptr(scratch), ptr(stream)))

    def ulysses_attention_fwd(self, plan, qkv, s_loc: int, head_dim: int, seg, scale: float, qkv_head, o_head, lse,
                              out, scratch=None, stream=None):
        """SPEC.md:333-341 ulysses_attention: seq_to_head -> tcgen05 attention -> head_to_seq (one pointer per
        local rank in every list; qkv_head / o_head / lse are kept by the caller for the backward)."""
        check(lib().spt_ulysses_attention_fwd(self.handle, C.byref(plan), self._ptrs(qkv), s_loc, head_dim, ptr(seg),
                                              scale, self._ptrs(qkv_head), self._ptrs(o_head), self._ptrs(lse),
                                              self._ptrs(out), ptr(scratch), ptr(stream)))

    def ulysses_attention_bwd(self, plan, qkv_head, o_head, lse, dout, s_loc: int, head_dim: int, seg, scale: float,
                              do_head, dqkv_head, ws, dqkv, scratch=None, stream=None):
        """The mirrored backward: dout [s_loc][Hq][d] -> dqkv [s_loc][Hq + 2 Hkv][d] (kv replicas summed in rank order)."""
        check(lib().spt_ulysses_attention_bwd(self.handle, C.byref(plan), self._ptrs(qkv_head), self._ptrs(o_head),
                                              self._ptrs(lse), self._ptrs(dout), s_loc, head_dim, ptr(seg), scale,
                                              self._ptrs(do_head), self._ptrs(dqkv_head), self._ptrs(ws),
                                              self._ptrs(dqkv), ptr(scratch), ptr(stream)))

    @classmethod
    def loopback_group(cls, world_size: int, device: int = 0) -> "ProcessGroup":
        h = C.c_void_p()
        check(lib().spt_comm_init_loopback(world_size, device, C.byref(h)))
        return cls(h, world_size, 0, True)

    @classmethod
    def nccl_group(cls, unique_id: bytes, world_size: int, rank: int, device: int) -> "ProcessGroup":
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib().spt_comm_init_rank(buf, world_size, rank, device, C.byref(h)))
        return cls(h, world_size, rank, False)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().spt_comm_unique_id(buf))
        return bytes(buf)

    def stats(self) -> dict:
        b = C.create_string_buffer(1 << 16)
        check(lib().spt_comm_stats_json(self.handle, b, len(b)))
        return json.loads(b.value.decode())

    def close(self):
        if self.handle:
            check(lib().spt_comm_destroy(self.handle))
            self.handle = None


@dataclass
class ModelShape:
    hidden: int
    q_heads: int
    kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int


TINY = ModelShape(256, 8, 2, 32, 1024, 32000)
LLAMA8B = ModelShape(4096, 32, 8, 128, 14336, 128256)
QWEN32B = ModelShape(5120, 64, 8, 128, 25600, 151936)

PARAM_NAMES = ("g1", "wqkv", "wo", "g2", "wg", "wu", "wd", "g3", "wlm")


class UlyssesLayerStep:
    """One decoder layer + lm_head fwd+bwd with Ulysses SP, TiledMLP and tiled logits+loss."""

    def __init__(self, shape: ModelShape, seq_len: int, group: ProcessGroup, mlp_tiles: int = 0,
                 loss_tile: int = 0, packed: bool = False, lr: float = 0.0, rms_eps: float = 1e-5,
                 n_layers: int = 1, ckpt_offload: bool = False, rope_theta: float = 0.0, embed: bool = False,
                 verify_replay: bool = False):
        self.shape, self.seq_len, self.group, self.n_layers = shape, seq_len, group, n_layers
        self.cfg = LayerConfig(shape.hidden, shape.q_heads, shape.kv_heads, shape.head_dim, shape.intermediate,
                               shape.vocab, seq_len, mlp_tiles, loss_tile, rms_eps, int(packed), lr, n_layers,
                               int(ckpt_offload), rope_theta, int(embed), int(verify_replay))
        h = C.c_void_p()
        check(lib().spt_layer_create(C.byref(self.cfg), group.handle, C.byref(h)))
        self.handle = h

    def param_numel(self, name: str) -> int:
        n = C.c_int64()
        check(lib().spt_layer_param_numel(self.handle, name.encode(), C.byref(n)))
        return n.value

    def set_param(self, name: str, data, on_host: bool | None = None):
        if on_host is None:
            on_host = not hasattr(data, "is_cuda") or not data.is_cuda
        size = data.numel() if hasattr(data, "numel") and callable(data.numel) else getattr(data, "size", None)
        want = self.param_numel(name)
        if size is not None and int(size) != want:  # the C-ABI copies `want` elements from the pointer
            raise ShapeError(1, f"set_param({name!r}): {int(size)} elements given, the engine expects {want}")
        check(lib().spt_layer_set_param(self.handle, name.encode(), ptr(data), int(on_host)))

    def step(self, x, shift_labels, position_ids=None, on_host: bool | None = None, stream=None):
        if on_host is None:
            on_host = not hasattr(x, "is_cuda") or not x.is_cuda
        loss, cnt = C.c_float(), C.c_int64()
        check(lib().spt_layer_step(self.handle, ptr(x), ptr(shift_labels), ptr(position_ids), int(on_host),
                                   C.byref(loss), C.byref(cnt), ptr(stream)))
        return loss.value, cnt.value

    def step_async(self, x, shift_labels, position_ids=None, on_host=False, stream=None):
        check(lib().spt_layer_step_async(self.handle, ptr(x), ptr(shift_labels), ptr(position_ids), int(on_host),
                                         ptr(stream)))

    def graph_capture(self, x, shift_labels, position_ids=None, stream=None):
        """Capture one device-resident step (fixed input addresses) into a CUDA graph on `stream` (non-default)."""
        check(lib().spt_layer_graph_capture(self.handle, ptr(x), ptr(shift_labels), ptr(position_ids), ptr(stream)))

    def graph_launch(self, stream=None):
        """Replay the captured step (same effect as step_async with the captured inputs)."""
        check(lib().spt_layer_graph_launch(self.handle, ptr(stream)))

    def step_accumulate(self, x, shift_labels, position_ids=None, first: bool = False, on_host: bool | None = None,
                        stream=None):
        """One micro-step of a gradient-accumulation window (grads of the loss sum)."""
        if on_host is None:
            on_host = not hasattr(x, "is_cuda") or not x.is_cuda
        check(lib().spt_layer_step_accumulate(self.handle, ptr(x), ptr(shift_labels), ptr(position_ids), int(on_host),
                                              int(first), ptr(stream)))

    def finish_accumulation(self, stream=None):
        """All-reduce the window's grads, divide by its global valid count; returns (mean loss, count)."""
        loss, cnt = C.c_float(), C.c_int64()
        check(lib().spt_layer_finish_accumulation(self.handle, C.byref(loss), C.byref(cnt), ptr(stream)))
        return loss.value, cnt.value

    def loss_async(self, slot: int, stream=None):
        """Enqueue the D2H of this step's (loss, count) into pinned slot `slot` (no synchronisation)."""
        check(lib().spt_layer_loss_async(self.handle, slot, ptr(stream)))

    def loss_slot(self, slot: int):
        loss, cnt = C.c_float(), C.c_int64()
        check(lib().spt_layer_loss_slot(self.handle, slot, C.byref(loss), C.byref(cnt)))
        return loss.value, cnt.value

    def read_loss(self, stream=None):
        loss, cnt = C.c_float(), C.c_int64()
        check(lib().spt_layer_read_loss(self.handle, C.byref(loss), C.byref(cnt), ptr(stream)))
        return loss.value, cnt.value

    def grad(self, name: str):
        import numpy as np

        s = self.shape
        bare = name.split(".", 2)[2] if name.startswith("layers.") else name
        shapes = {"g1": (s.hidden,), "g2": (s.hidden,), "g3": (s.hidden,),
                  "wqkv": ((s.q_heads + 2 * s.kv_heads) * s.head_dim, s.hidden),
                  "wo": (s.hidden, s.q_heads * s.head_dim), "wg": (s.intermediate, s.hidden),
                  "wu": (s.intermediate, s.hidden), "wd": (s.hidden, s.intermediate), "wlm": (s.vocab, s.hidden),
                  "emb": (s.vocab, s.hidden)}
        out = np.empty(shapes[bare], dtype=np.float32)
        check(lib().spt_layer_get_grad(self.handle, name.encode(), ptr(out)))
        return out

    def dx_bits(self, n_tokens: int):
        import numpy as np

        out = np.empty((n_tokens, self.shape.hidden), dtype=np.uint16)
        check(lib().spt_layer_get_dx(self.handle, ptr(out)))
        return out

    def memory(self) -> dict:
        b = C.create_string_buffer(1 << 16)
        check(lib().spt_layer_memory_json(self.handle, b, len(b)))
        return json.loads(b.value.decode())

    def memory_timeline_csv(self) -> str:
        """The device ledger's event timeline (reference MemoryLedger::timeline_csv columns)."""
        b = C.create_string_buffer(1 << 20)
        check(lib().spt_layer_memory_timeline_csv(self.handle, b, len(b)))
        return b.value.decode()

    def set_profiling(self, on: bool):
        check(lib().spt_layer_set_profiling(self.handle, int(on)))

    def timing(self) -> dict:
        b = C.create_string_buffer(1 << 16)
        check(lib().spt_layer_timing_json(self.handle, b, len(b)))
        return json.loads(b.value.decode())

    def close(self):
        if self.handle:
            check(lib().spt_layer_destroy(self.handle))
            self.handle = None


def kernel_launch_count() -> int:
    return lib().spt_kernel_launch_count()
