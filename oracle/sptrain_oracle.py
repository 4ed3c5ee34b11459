"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the ALST (arXiv 2506.13996) reference algorithm for the
hot path this repo accelerates: one Llama-shaped decoder layer + lm_head,
fwd+bwd, under Ulysses sequence parallelism with TiledMLP and tiled
logits+loss.  The reference (`/root/reference`) ships the algorithm only as a
behavioural spec (`SPEC.md`) plus a C++ substrate (`proj/`) that contains none
of the path, so every function here restates a SPEC.md
operation and cites the line it follows.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import this module, and only as the checker / the timed CPU port — the CUDA
path in `paper_2506_13996_b200` never calls into it.

Parity pinning: the integer/index functions (plan_head_shards, seq_to_head,
head_to_seq, all_to_all, preshift/shard/pad, block-causal predicate) are
pinned against every worked example in SPEC.md / PAPER.md
(`tests/golden/spec_examples.json`, checked by `tests/test_oracle_golden.py`).
The floating-point functions are pinned by the SPEC's own self-oracles
(finite differences, tiled == untiled, SP=P == SP=1, closed-form CE cases);
no reference test pins their absolute values because none exists
("parity is unpinned by reference tests" for FP outputs).

Precision: float64 by default ("Default precision 64-bit for test
rigor; 32-bit mode available for throughput runs"); pass dtype=np.float32 for
the timed CPU baseline.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

IGNORE_INDEX = -100  # SPEC.md:69, "-100 is the special label value to be ignored"
RMS_EPS = 1e-5


# --------------------------------------------------------------------------------------
# errors (mirror proj/include/sptrain/errors.hpp:12-72)
# --------------------------------------------------------------------------------------
class ValidationError(ValueError):
    """errors.hpp:13 — bad user input (labels, position ids, config values)."""


class ShapeError(ValidationError):
    """errors.hpp:19 — tensor shape disagreement."""


class CollectiveError(RuntimeError):
    """errors.hpp:25 — a collective saw incompatible payloads across ranks."""


class ConfigError(RuntimeError):
    """errors.hpp:68 — run configuration rejected."""


# --------------------------------------------------------------------------------------
# bf16 helpers (the GPU consumes bf16; the oracle consumes the same bits upcast)
# --------------------------------------------------------------------------------------
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit pattern (uint16)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    r = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(a)
    if nan.any():
        r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Values exactly representable in bf16 (as float32)."""
    return bf16_bits_to_f32(f32_to_bf16_bits(a))


# --------------------------------------------------------------------------------------
# ulysses: head-shard plan (§7.1 limits PAPER.md:946-957)
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class HeadShardPlan:
    """SPEC.md:286-292 `HeadShardPlan`."""

    sp_degree: int
    q_heads: int
    kv_heads: int
    q_heads_per_rank: int
    kv_heads_per_rank: int
    kv_replication: int

    def q_heads_of(self, rank: int) -> list[int]:
        """Contiguous block assignment, SPEC.md:299 / :350."""
        n = self.q_heads_per_rank
        return list(range(rank * n, (rank + 1) * n))

    def kv_heads_of(self, rank: int) -> list[int]:
        """r == 1: contiguous Hkv/P block; r > 1: head floor(rank / r)."""
        if self.kv_replication > 1:
            return [rank // self.kv_replication]
        n = self.kv_heads_per_rank
        return list(range(rank * n, (rank + 1) * n))


def plan_head_shards(q_heads: int, kv_heads: int, sp: int) -> HeadShardPlan:
    """SPEC.md:296-305. Rejects exactly the §7.1 cases."""
    if q_heads < 1 or kv_heads < 1 or sp < 1:
        raise ValidationError("head counts and SP degree must be >= 1")
    if q_heads % kv_heads != 0:  # SPEC.md:298 pre: Hq % Hkv == 0
        raise ValidationError(f"q_heads ({q_heads}) not divisible by kv_heads ({kv_heads})")
    if q_heads % sp != 0:
        ok = [p for p in range(1, q_heads + 1) if q_heads % p == 0]
        raise ValidationError(
            f"q_heads not divisible by SP degree: q_heads={q_heads}, sp={sp}; "
            f"you'd need SP to be one of {ok}")
    if kv_heads >= sp:
        if kv_heads % sp != 0:  # SPEC.md:300 second clause
            raise ValidationError(f"kv_heads ({kv_heads}) >= SP ({sp}) but not divisible by it")
        return HeadShardPlan(sp, q_heads, kv_heads, q_heads // sp, kv_heads // sp, 1)
    if sp % kv_heads != 0:  # implied by SPEC.md:290 (r*Hkv == P)
        raise ValidationError(f"SP ({sp}) not a multiple of kv_heads ({kv_heads}); cannot replicate")
    return HeadShardPlan(sp, q_heads, kv_heads, q_heads // sp, 1, sp // kv_heads)


# --------------------------------------------------------------------------------------
# collectives: in-process SPMD
# --------------------------------------------------------------------------------------
def all_to_all(send_parts_per_rank: list[list[np.ndarray]]) -> list[list[np.ndarray]]:
    """recv_parts[j] on rank i == send_parts[i] from rank j."""
    world = len(send_parts_per_rank)
    for r, parts in enumerate(send_parts_per_rank):
        if len(parts) != world:
            raise CollectiveError(f"rank {r} sent {len(parts)} parts for world_size {world}")
    recv = [[None] * world for _ in range(world)]
    for i in range(world):
        for j in range(world):
            if send_parts_per_rank[j][i].shape != send_parts_per_rank[0][i].shape:
                raise CollectiveError(f"part {i} shape differs between ranks 0 and {j}")
            recv[i][j] = send_parts_per_rank[j][i]
    return recv


def all_reduce_sum(xs: list[np.ndarray]) -> list[np.ndarray]:
    """element-wise sum, fixed rank-ascending order."""
    acc = np.array(xs[0], copy=True)
    for x in xs[1:]:
        if x.shape != acc.shape:
            raise CollectiveError("all_reduce_sum shape divergence")
        acc = acc + x
    return [acc.copy() for _ in xs]


# --------------------------------------------------------------------------------------
# ulysses reshard (layout SPEC.md:350-352)
# --------------------------------------------------------------------------------------
def seq_to_head(xs: list[np.ndarray], heads_of) -> list[np.ndarray]:
    """SPEC.md:307-315. xs[i]: [s_loc, H, d] on rank i; heads_of(j) = global heads rank j owns.

    Split the head dim per the plan, all_to_all, concatenate received sequence segments in
    rank order (payload sequence-major, heads inner: SPEC.md:351).  With kv replication a head
    appears in several ranks' lists, i.e. it is delivered to all r consumers.
    """
    P = len(xs)
    send = [[x[:, heads_of(j), :] for j in range(P)] for x in xs]
    recv = all_to_all(send)
    return [np.concatenate(recv[j], axis=0) for j in range(P)]


def head_to_seq(ys: list[np.ndarray], heads_of, num_heads: int, reduce_replicas: bool = False) -> list[np.ndarray]:
    """SPEC.md:317-321 exact inverse of seq_to_head.

    With replication (several ranks own the same head) the forward direction is undefined
    unless reduce_replicas=True, which is the backward of replicate_kv: sum over the r
    consumers in rank-ascending order.
    """
    P = len(ys)
    s = ys[0].shape[0]
    if s % P:
        raise ShapeError(f"s={s} not divisible by P={P}")
    s_loc = s // P
    send = [[y[i * s_loc:(i + 1) * s_loc] for i in range(P)] for y in ys]
    recv = all_to_all(send)
    out = []
    for i in range(P):
        d = ys[0].shape[2]
        x = np.zeros((s_loc, num_heads, d), dtype=ys[0].dtype)
        seen = np.zeros(num_heads, dtype=np.int64)
        for j in range(P):  # rank-ascending
            hs = heads_of(j)
            for a, hglob in enumerate(hs):
                if seen[hglob] and not reduce_replicas:
                    raise CollectiveError(f"head {hglob} owned by several ranks; use reduce_replicas")
                x[:, hglob, :] = x[:, hglob, :] + recv[i][j][:, a, :]
                seen[hglob] += 1
        out.append(x)
    return out


# --------------------------------------------------------------------------------------
# dataloader
# --------------------------------------------------------------------------------------
def preshift_labels(labels) -> np.ndarray:
    """out[i] = labels[i+1], out[s-1] = -100."""
    labels = np.asarray(labels, dtype=np.int64)
    out = np.full_like(labels, IGNORE_INDEX)
    if labels.size > 1:
        out[:-1] = labels[1:]
    return out


def naive_shift_after_shard(labels, P: int) -> list[np.ndarray]:
    """The defective variant PAPER.md:549-567 describes (kept as a regression oracle)."""
    labels = np.asarray(labels, dtype=np.int64)
    return [preshift_labels(c) for c in np.split(labels, P)]


def pad_to_multiple(input_ids, position_ids, shift_labels, P: int):
    """pad token 0, label -100, isolated position run."""
    input_ids = np.asarray(input_ids, dtype=np.int64)
    position_ids = np.asarray(position_ids, dtype=np.int64)
    shift_labels = np.asarray(shift_labels, dtype=np.int64)
    s = input_ids.size
    pad = (-s) % P
    if pad == 0:
        return input_ids.copy(), position_ids.copy(), shift_labels.copy()
    return (np.concatenate([input_ids, np.zeros(pad, np.int64)]),
            np.concatenate([position_ids, np.arange(pad, dtype=np.int64)]),
            np.concatenate([shift_labels, np.full(pad, IGNORE_INDEX, np.int64)]))


def shard_sequence(arr, P: int) -> list[np.ndarray]:
    """contiguous equal slices in rank order."""
    arr = np.asarray(arr)
    if arr.shape[0] % P:
        raise ShapeError(f"sequence length {arr.shape[0]} not divisible by P={P}; pad first")
    return list(np.split(arr, P, axis=0))


def block_causal_starts(position_ids) -> np.ndarray:
    """SPEC.md:243-251 `derive_block_causal_mask_predicate`, represented lazily.

    Returns start[t] = first index of t's run; predicate(i, j) = start[i] <= j <= i.
    position_ids must be a concatenation of zero-based ascending runs, else ValidationError.
    """
    p = np.asarray(position_ids, dtype=np.int64)
    if p.size == 0:
        return p.copy()
    ok = np.empty(p.size, dtype=bool)
    ok[0] = p[0] == 0
    ok[1:] = (p[1:] == 0) | (p[1:] == p[:-1] + 1)
    if not ok.all():
        bad = int(np.argmin(ok))
        raise ValidationError(f"position_ids not zero-based ascending runs at index {bad}")
    idx = np.arange(p.size, dtype=np.int64)
    return idx - p


def block_causal_predicate(position_ids):
    starts = block_causal_starts(position_ids)

    def pred(i: int, j: int) -> bool:
        return bool(starts[i] <= j <= i)

    return pred


# --------------------------------------------------------------------------------------
# core ops and layer pieces
# --------------------------------------------------------------------------------------
def rmsnorm_fwd(x, g, eps=RMS_EPS):
    """SPEC.md:259 RMS-style normalization with learnable scale."""
    rstd = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * rstd * g, rstd


def rmsnorm_bwd(x, g, rstd, dy):
    xhat = x * rstd
    dg = np.sum(dy * xhat, axis=0)
    dxhat = dy * g
    dx = rstd * (dxhat - xhat * np.mean(dxhat * xhat, axis=-1, keepdims=True))
    return dx, dg


def silu(x):
    return x / (1.0 + np.exp(-x))


def cross_entropy(logits, labels, ignore_index=IGNORE_INDEX):
    """returns (sum of NLL over non-ignored tokens, valid count) + dlogits of the sum."""
    labels = np.asarray(labels, dtype=np.int64)
    V = logits.shape[-1]
    bad = (labels != ignore_index) & ((labels < 0) | (labels >= V))
    if bad.any():
        raise ValidationError(f"label out of range [0,{V}) at index {int(np.argmax(bad))}")
    valid = labels != ignore_index
    m = logits.max(axis=-1, keepdims=True)
    e = np.exp(logits - m)
    se = e.sum(axis=-1, keepdims=True)
    lse = (m + np.log(se))[:, 0]
    safe = np.where(valid, labels, 0)
    picked = logits[np.arange(logits.shape[0]), safe]
    nll = np.where(valid, lse - picked, 0.0)
    dlogits = e / se
    dlogits[np.arange(logits.shape[0]), safe] -= 1.0
    dlogits *= valid[:, None]
    return float(nll.sum()), int(valid.sum()), dlogits


def attention_fwd(q, k, v, starts=None, scale=None, q_block=256):
    """Inner AttentionCallback: softmax(q k^T * scale + mask) v, GQA.

    q [s, Hq, d], k/v [s, Hkv, d]; starts[t] gives block-causal runs;
    None = plain causal.  The mask is evaluated per query block, never as an [s,s] tensor.
    Returns o [s, Hq, d] and lse [Hq, s].
    """
    s, Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    if starts is None:
        starts = np.zeros(s, dtype=np.int64)
    o = np.zeros_like(q)
    lse = np.zeros((Hq, s), dtype=q.dtype)
    kj = np.arange(s)
    for h in range(Hq):
        kh, vh = k[:, h // g, :], v[:, h // g, :]
        for q0 in range(0, s, q_block):
            q1 = min(s, q0 + q_block)
            qi = np.arange(q0, q1)
            sc = (q[q0:q1, h, :] @ kh[:q1].T) * scale
            allowed = (kj[None, :q1] <= qi[:, None]) & (kj[None, :q1] >= starts[q0:q1, None])
            sc = np.where(allowed, sc, -np.inf)
            m = sc.max(axis=1, keepdims=True)
            p = np.exp(sc - m)
            l = p.sum(axis=1, keepdims=True)
            o[q0:q1, h, :] = (p / l) @ vh[:q1]
            lse[h, q0:q1] = (m + np.log(l))[:, 0]
    return o, lse


def attention_bwd(q, k, v, o, lse, do, starts=None, scale=None, q_block=256):
    s, Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    if starts is None:
        starts = np.zeros(s, dtype=np.int64)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    kj = np.arange(s)
    for h in range(Hq):
        kh, vh = k[:, h // g, :], v[:, h // g, :]
        for q0 in range(0, s, q_block):
            q1 = min(s, q0 + q_block)
            qi = np.arange(q0, q1)
            sc = (q[q0:q1, h, :] @ kh[:q1].T) * scale
            allowed = (kj[None, :q1] <= qi[:, None]) & (kj[None, :q1] >= starts[q0:q1, None])
            p = np.where(allowed, np.exp(sc - lse[h, q0:q1, None]), 0.0)
            dO = do[q0:q1, h, :]
            dv[:q1, h // g, :] += p.T @ dO
            dp = dO @ vh[:q1].T
            D = np.sum(dO * o[q0:q1, h, :], axis=1, keepdims=True)
            ds = p * (dp - D) * scale
            dq[q0:q1, h, :] = ds @ kh[:q1]
            dk[:q1, h // g, :] += ds.T @ q[q0:q1, h, :]
    return dq, dk, dv


# ---- attention restricted to sampled rows / columns (SURVEY.md §8(c) parity protocol item 3: the L8 / Q8 rank
# shapes, s = 2^19 .. 2^20, are checked on sampled query rows and key columns; the full [s, s] problem is
# out of reach on the CPU).  Same formulas as attention_fwd / attention_bwd above (SPEC.md:216-219, :243-251,
# :59-67), float64, keys or queries walked in chunks with a running (max, sum) so no [rows, s] matrix lives.


def _chunk64(a, lo, hi, dtype=np.float64):
    return np.asarray(a[lo:hi], dtype=dtype)


def attention_rows(q, k, v, rows, starts=None, scale=None, key_chunk=65536, dtype=np.float64):
    """O and LSE of query rows `rows` (int array) of attention_fwd: q [s, Hq, d], k / v [s, Hkv, d] (any float
    dtype, upcast per chunk).  Returns o [R, Hq, d] and lse [Hq, R] in `dtype` (float64 for parity checks; bench.py's
    CPU arm times it in float32 like the rest of its f32 layer step)."""
    rows = np.asarray(rows, np.int64)
    s, Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    st = np.zeros(len(rows), np.int64) if starts is None else np.asarray(starts)[rows]
    qr = np.asarray(q[rows], dtype)  # [R, Hq, d]
    m = np.full((Hq, len(rows)), -np.inf, dtype)
    l = np.zeros((Hq, len(rows)), dtype)
    acc = np.zeros((Hq, len(rows), d), dtype)
    for k0 in range(0, int(rows.max()) + 1, key_chunk):
        k1 = min(s, k0 + key_chunk)
        kc, vc = _chunk64(k, k0, k1, dtype), _chunk64(v, k0, k1, dtype)
        kj = np.arange(k0, k1)
        allowed = (kj[None, :] <= rows[:, None]) & (kj[None, :] >= st[:, None])
        for h in range(Hq):
            sc = (qr[:, h, :] @ kc[:, h // g, :].T) * scale
            sc = np.where(allowed, sc, -np.inf)
            mn = np.maximum(m[h], sc.max(axis=1))
            safe = np.where(np.isfinite(mn), mn, 0.0)
            p = np.exp(sc - safe[:, None])
            alpha = np.exp(np.where(np.isfinite(m[h]), m[h] - safe, -np.inf))
            l[h] = l[h] * alpha + p.sum(axis=1)
            acc[h] = acc[h] * alpha[:, None] + p @ vc[:, h // g, :]
            m[h] = mn
    o = (acc / l[:, :, None]).transpose(1, 0, 2)
    return o, m + np.log(l)


def attention_bwd_rows(q, k, v, do, rows, o_rows, lse_rows, starts=None, scale=None, key_chunk=65536,
                       dtype=np.float64):
    """dQ of query rows `rows` (attention_bwd): dq_i = scale * sum_j P_ij (dO_i . v_j - D_i) k_j, D_i = dO_i . o_i,
    with o_rows [R, Hq, d] / lse_rows [Hq, R] from attention_rows.  Returns dq [R, Hq, d] in `dtype`."""
    rows = np.asarray(rows, np.int64)
    s, Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    st = np.zeros(len(rows), np.int64) if starts is None else np.asarray(starts)[rows]
    qr = np.asarray(q[rows], dtype)
    dor = np.asarray(do[rows], dtype)
    D = np.sum(dor * o_rows, axis=2)  # [R, Hq]
    dq = np.zeros((len(rows), Hq, d), dtype)
    for k0 in range(0, int(rows.max()) + 1, key_chunk):
        k1 = min(s, k0 + key_chunk)
        kc, vc = _chunk64(k, k0, k1, dtype), _chunk64(v, k0, k1, dtype)
        kj = np.arange(k0, k1)
        allowed = (kj[None, :] <= rows[:, None]) & (kj[None, :] >= st[:, None])
        for h in range(Hq):
            sc = (qr[:, h, :] @ kc[:, h // g, :].T) * scale
            p = np.where(allowed, np.exp(sc - lse_rows[h][:, None]), 0.0)
            dp = dor[:, h, :] @ vc[:, h // g, :].T
            dq[:, h, :] += (p * (dp - D[:, h][:, None]) * scale) @ kc[:, h // g, :]
    return dq


def attention_bwd_cols(q, k, v, do, lse, D, cols, starts=None, scale=None, row_chunk=65536):
    """dK and dV of key rows `cols` (attention_bwd): every query i >= j of every q head of the kv head's group
    contributes.  Needs the LSE [Hq, s] and D = rowsum(dO * O) [s, Hq] of ALL queries (callers pass the
    device's, checked separately on sampled rows).  Returns dk, dv [C, Hkv, d] float64."""
    cols = np.asarray(cols, np.int64)
    s, Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    kc = np.asarray(k[cols], np.float64)
    vc = np.asarray(v[cols], np.float64)
    st_all = None if starts is None else np.asarray(starts)
    dk = np.zeros((len(cols), Hkv, d))
    dv = np.zeros((len(cols), Hkv, d))
    for i0 in range(int(cols.min()) // row_chunk * row_chunk, s, row_chunk):
        i1 = min(s, i0 + row_chunk)
        qi = np.arange(i0, i1)
        st = np.zeros(i1 - i0, np.int64) if st_all is None else st_all[i0:i1]
        allowed = (cols[None, :] <= qi[:, None]) & (cols[None, :] >= st[:, None])  # [c, C]
        qc, doc = _chunk64(q, i0, i1), _chunk64(do, i0, i1)
        for h in range(Hq):
            hk = h // g
            sc = (qc[:, h, :] @ kc[:, hk, :].T) * scale
            p = np.where(allowed, np.exp(sc - np.asarray(lse[h, i0:i1], np.float64)[:, None]), 0.0)
            dv[:, hk, :] += p.T @ doc[:, h, :]
            dp = doc[:, h, :] @ vc[:, hk, :].T
            ds = p * (dp - np.asarray(D[i0:i1, h], np.float64)[:, None]) * scale
            dk[:, hk, :] += ds.T @ qc[:, h, :]
    return dk, dv


def tile_bounds(s: int, num_tiles: int) -> list[tuple[int, int]]:
    """SPEC.md:378-381 TileSpec: uniform tiles of ceil(s/num_tiles), final tile may be smaller."""
    if num_tiles < 1:
        raise ValidationError("num_tiles must be >= 1")
    tl = -(-s // num_tiles)
    return [(a, min(s, a + tl)) for a in range(0, s, tl)]


def default_mlp_tiles(s: int, h: int) -> int:
    """num_tiles = ceil(s/h) (ceil(256000/4096) = 63)."""
    return max(1, -(-s // h))


def gated_mlp_fwd(x, wg, wu, wd):
    """SPEC.md:260 gated MLP: y = Wd (silu(Wg x) * Wu x)."""
    gt = x @ wg.T
    ut = x @ wu.T
    a = silu(gt) * ut
    return a @ wd.T


def tiled_mlp(x, wg, wu, wd, num_tiles=None):
    """SPEC.md:395-403 forward; returns y."""
    s, h = x.shape
    num_tiles = default_mlp_tiles(s, h) if num_tiles is None else num_tiles
    y = np.empty_like(x)
    for a, b in tile_bounds(s, num_tiles):
        y[a:b] = gated_mlp_fwd(x[a:b], wg, wu, wd)
    return y


def tiled_mlp_bwd(x, wg, wu, wd, dy, num_tiles=None):
    """SPEC.md:385-393 backward: per-tile recompute, param grads summed in ascending tile order (:421-422)."""
    s, h = x.shape
    num_tiles = default_mlp_tiles(s, h) if num_tiles is None else num_tiles
    dx = np.empty_like(x)
    dwg = np.zeros_like(wg)
    dwu = np.zeros_like(wu)
    dwd = np.zeros_like(wd)
    for a, b in tile_bounds(s, num_tiles):
        xt, dyt = x[a:b], dy[a:b]
        gt = xt @ wg.T
        ut = xt @ wu.T
        sg = 1.0 / (1.0 + np.exp(-gt))
        si = gt * sg
        act = si * ut
        dwd += dyt.T @ act
        da = dyt @ wd
        du = da * si
        dg = da * ut * sg * (1.0 + gt * (1.0 - sg))
        dwg += dg.T @ xt
        dwu += du.T @ xt
        dx[a:b] = dg @ wg + du @ wu
    return dx, dwg, dwu, dwd


def lm_head_and_loss(hidden, w_lm, shift_labels):
    """SPEC.md:233-241 untiled reference: cross_entropy(hidden W^T, shift_labels)."""
    ls, cnt, _ = cross_entropy(hidden @ w_lm.T, shift_labels)
    return ls, cnt


def tiled_logits_loss(hidden, w_lm, shift_labels, tile_len, grad_scale=None):
    """per-tile logits + CE, (sum, count); grads with scale `grad_scale`.

    When grad_scale is given, returns d hidden and d W_lm of grad_scale * loss_sum,
    dW accumulated in ascending tile order.
    """
    s = hidden.shape[0]
    total, count = 0.0, 0
    dh = np.zeros_like(hidden) if grad_scale is not None else None
    dw = np.zeros_like(w_lm) if grad_scale is not None else None
    for a in range(0, s, tile_len):
        b = min(s, a + tile_len)
        logits = hidden[a:b] @ w_lm.T
        ls, cnt, dl = cross_entropy(logits, shift_labels[a:b])
        total += ls
        count += cnt
        if grad_scale is not None:
            dl = dl * grad_scale
            dh[a:b] = dl @ w_lm
            dw += dl.T @ hidden[a:b]
    return total, count, dh, dw


# --------------------------------------------------------------------------------------
# layer step: norm -> ulysses attention -> +res -> norm -> tiled MLP -> +res -> final norm
#             -> tiled logits+loss, fwd + bwd
# --------------------------------------------------------------------------------------
@dataclass
class LayerConfig:
    hidden: int
    q_heads: int
    kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int

    @property
    def qkv_out(self) -> int:
        return (self.q_heads + 2 * self.kv_heads) * self.head_dim


TINY = LayerConfig(hidden=256, q_heads=8, kv_heads=2, head_dim=32, intermediate=1024, vocab=32000)
LLAMA8B = LayerConfig(hidden=4096, q_heads=32, kv_heads=8, head_dim=128, intermediate=14336, vocab=128256)
QWEN32B = LayerConfig(hidden=5120, q_heads=64, kv_heads=8, head_dim=128, intermediate=25600, vocab=151936)


@dataclass
class LayerParams:
    """Weights in [out, in] row-major (PyTorch Linear convention)."""

    g1: np.ndarray
    wqkv: np.ndarray  # [(Hq + 2Hkv) d, h]: q heads, then k heads, then v heads
    wo: np.ndarray  # [h, Hq d]
    g2: np.ndarray
    wg: np.ndarray  # [I, h]
    wu: np.ndarray  # [I, h]
    wd: np.ndarray  # [h, I]
    g3: np.ndarray
    wlm: np.ndarray  # [V, h]

    def astype(self, dt):
        return LayerParams(**{k: np.asarray(getattr(self, k), dtype=dt) for k in self.__dataclass_fields__})

    NAMES = ("g1", "wqkv", "wo", "g2", "wg", "wu", "wd", "g3", "wlm")


@dataclass
class StepResult:
    loss_sum: float
    count: int
    loss: float
    dx: np.ndarray  # [N, h] d loss / d input hidden (sequence order)
    grads: dict = field(default_factory=dict)
    out_hidden: np.ndarray | None = None  # final-norm output (pre lm_head), sequence order


def synth_params(cfg: LayerConfig, seed: int, wstd: float = 0.02) -> dict:
    """SURVEY.md §8(d) value distributions, rounded to bf16 (the bits the GPU consumes)."""
    rng = np.random.default_rng(seed)
    h, I, V = cfg.hidden, cfg.intermediate, cfg.vocab
    qd = cfg.q_heads * cfg.head_dim

    def w(*shape):
        return round_bf16(rng.standard_normal(shape, dtype=np.float32) * wstd)

    def gam():
        return round_bf16(1.0 + 0.05 * rng.standard_normal(h, dtype=np.float32))

    return dict(g1=gam(), wqkv=w(cfg.qkv_out, h), wo=w(h, qd), g2=gam(), wg=w(I, h), wu=w(I, h),
                wd=w(h, I), g3=gam(), wlm=w(V, h))


def synth_batch(cfg: LayerConfig, n: int, seed: int, ignore_frac: float = 0.05, packed: bool = False):
    """Hidden x ~ N(0,1) in bf16; labels U[0,V) with ~5% -100, pre-shifted; position ids."""
    rng = np.random.default_rng(seed + 7919)
    x = round_bf16(rng.standard_normal((n, cfg.hidden), dtype=np.float32))
    labels = rng.integers(0, cfg.vocab, size=n, dtype=np.int64)
    labels[rng.random(n) < ignore_frac] = IGNORE_INDEX
    if packed:
        pos = []
        while len(pos) < n:
            run = int(rng.integers(1, max(2, n // 3)))
            pos.extend(range(run))
        position_ids = np.asarray(pos[:n], dtype=np.int64)
    else:
        position_ids = np.arange(n, dtype=np.int64)
    # pre-shift within each packed sample would be the data pipeline's job; the
    # shift is applied once over the whole (already packed) sequence
    shift = preshift_labels(labels)
    return x, shift, position_ids


def embed_fwd(input_ids, table):
    """Token embedding gather (SPEC.md:205 model "embedding", :223-227 forward(model, input_ids, ...)):
    x[t] = table[input_ids[t]]; an id outside [0, V) is a validation error."""
    ids = np.asarray(input_ids, dtype=np.int64)
    V = table.shape[0]
    if ids.size and (ids.min() < 0 or ids.max() >= V):
        raise ValueError("token id outside [0, V)")
    return table[ids]


def embed_bwd(input_ids, dx, vocab: int, dtable=None):
    """Embedding backward: dtable[v] (+)= sum of dx[t] over t with input_ids[t] == v, each per-id sum taken
    in ascending t in float32 and then added to the existing row (the CUDA path's deterministic order).
    Plain loops: test sizes only."""
    ids = np.asarray(input_ids, dtype=np.int64)
    dx = np.asarray(dx, dtype=np.float32)
    out = np.zeros((vocab, dx.shape[1]), np.float32) if dtable is None else np.array(dtable, np.float32)
    sums = {}
    for t, v in enumerate(ids.tolist()):
        if v in sums:
            sums[v] = sums[v] + dx[t]
        else:
            sums[v] = dx[t].copy()
    for v, acc in sums.items():
        out[v] = out[v] + acc
    return out


def rope_angles(positions, head_dim: int, theta: float):
    """Rotary position embedding angles (the reference SPEC omits RoPE).
    Llama / HF convention: inv_freq[j] = theta^(-2j/d), angle[t, j] = position[t] * inv_freq[j], both in
    float32 exactly as HF computes them (so long positions carry the same fp32 rounding), cos/sin in f64."""
    j = np.arange(0, head_dim, 2, dtype=np.int64).astype(np.float32) / np.float32(head_dim)
    inv_freq = (np.float32(1.0) / np.power(np.float32(theta), j)).astype(np.float32)
    ang = (np.asarray(positions, np.int64).astype(np.float32)[:, None] * inv_freq[None, :]).astype(np.float32)
    return np.cos(ang.astype(np.float64)), np.sin(ang.astype(np.float64))


def rope_apply(x, cos, sin, inverse: bool = False):
    """x [n, heads, d] -> x*cos + rotate_half(x)*sin (rotate_half(x) = [-x2, x1]); inverse=True applies the
    transpose rotation (the backward of the forward rotation)."""
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    if inverse:
        s = -s
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope_positions(position_ids, packed: bool):
    """RoPE positions: the position_ids themselves for packed samples (each sample restarts at 0), else the
    global token index (SPEC.md:333 position_ids_full = arange for a single sample)."""
    return np.asarray(position_ids, np.int64)


def decoder_layer_fwd(p, cfg: LayerConfig, xs: list, starts, P: int, mlp_tiles=None, rope=None):
    """One decoder layer forward over P in-process ranks: per rank
    x1 = x + Wo·ulysses_attention(Wqkv·rms1(x)), x2 = x1 + tiled_mlp(rms2(x1)).  rope: None or per-rank
    (cos, sin) applied to q and k after the projection (row f4).  Returns (x2 per rank, cache)."""
    Hq, Hkv, d = cfg.q_heads, cfg.kv_heads, cfg.head_dim
    plan = plan_head_shards(Hq, Hkv, P)
    n_loc = xs[0].shape[0]
    st = [dict(x=xs[r]) for r in range(P)]
    for r in range(P):  # phase A: norm + qkv projection per rank
        xn1, rstd1 = rmsnorm_fwd(xs[r], p.g1)
        qkv = xn1 @ p.wqkv.T
        q = qkv[:, :Hq * d].reshape(n_loc, Hq, d)
        k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(n_loc, Hkv, d)
        v = qkv[:, (Hq + Hkv) * d:].reshape(n_loc, Hkv, d)
        if rope is not None:
            q = rope_apply(q, *rope[r])
            k = rope_apply(k, *rope[r])
        st[r].update(xn1=xn1, rstd1=rstd1, q=q, k=k, v=v)
    # seq -> head all-to-all, inner attention over the full sequence, head -> seq
    qh = seq_to_head([s_["q"] for s_ in st], plan.q_heads_of)
    kh = seq_to_head([s_["k"] for s_ in st], plan.kv_heads_of)
    vh = seq_to_head([s_["v"] for s_ in st], plan.kv_heads_of)
    oh, lse = [], []
    for j in range(P):
        o_, l_ = attention_fwd(qh[j], kh[j], vh[j], starts)
        oh.append(o_)
        lse.append(l_)
    os_ = head_to_seq(oh, plan.q_heads_of, Hq)
    for r in range(P):
        o = os_[r].reshape(n_loc, Hq * d)
        x1 = xs[r] + o @ p.wo.T
        xn2, rstd2 = rmsnorm_fwd(x1, p.g2)
        x2 = x1 + tiled_mlp(xn2, p.wg, p.wu, p.wd, mlp_tiles)
        st[r].update(o=o, x1=x1, xn2=xn2, rstd2=rstd2, x2=x2)
    cache = dict(st=st, qh=qh, kh=kh, vh=vh, oh=oh, lse=lse, plan=plan, starts=starts, mlp_tiles=mlp_tiles, rope=rope)
    return [s_["x2"] for s_ in st], cache


def decoder_layer_bwd(p, cfg: LayerConfig, cache: dict, dys: list, P: int):
    """Backward of decoder_layer_fwd: d(layer output) per rank -> (d(layer input) per rank, per-rank grads)."""
    Hq, Hkv, d = cfg.q_heads, cfg.kv_heads, cfg.head_dim
    st, plan, starts, mlp_tiles = cache["st"], cache["plan"], cache["starts"], cache["mlp_tiles"]
    n_loc = st[0]["x"].shape[0]
    grads = [dict() for _ in range(P)]
    for r in range(P):
        s_ = st[r]
        dx2 = dys[r]
        dxn2, dwg, dwu, dwd = tiled_mlp_bwd(s_["xn2"], p.wg, p.wu, p.wd, dx2, mlp_tiles)
        dx1n, dg2 = rmsnorm_bwd(s_["x1"], p.g2, s_["rstd2"], dxn2)
        dx1 = dx2 + dx1n
        do = (dx1 @ p.wo).reshape(n_loc, Hq, d)
        dwo = dx1.T @ s_["o"]
        grads[r].update(wg=dwg, wu=dwu, wd=dwd, g2=dg2, wo=dwo)
        s_.update(dx1=dx1, do=do)
    doh = seq_to_head([s_["do"] for s_ in st], plan.q_heads_of)
    dqh, dkh, dvh = [], [], []
    for j in range(P):
        a, b, c = attention_bwd(cache["qh"][j], cache["kh"][j], cache["vh"][j], cache["oh"][j], cache["lse"][j], doh[j],
                                starts)
        dqh.append(a)
        dkh.append(b)
        dvh.append(c)
    dqs = head_to_seq(dqh, plan.q_heads_of, Hq)
    dks = head_to_seq(dkh, plan.kv_heads_of, Hkv, reduce_replicas=True)  # replicate_kv bwd
    dvs = head_to_seq(dvh, plan.kv_heads_of, Hkv, reduce_replicas=True)
    dxs = []
    for r in range(P):
        s_ = st[r]
        dq_r, dk_r = dqs[r], dks[r]
        if cache["rope"] is not None:  # back through the rotation (transpose)
            dq_r = rope_apply(dq_r, *cache["rope"][r], inverse=True)
            dk_r = rope_apply(dk_r, *cache["rope"][r], inverse=True)
        dqkv = np.concatenate([dq_r.reshape(n_loc, -1), dk_r.reshape(n_loc, -1), dvs[r].reshape(n_loc, -1)], axis=1)
        grads[r]["wqkv"] = dqkv.T @ s_["xn1"]
        dxn1 = dqkv @ p.wqkv
        dx0n, dg1 = rmsnorm_bwd(s_["x"], p.g1, s_["rstd1"], dxn1)
        grads[r]["g1"] = dg1
        dxs.append(s_["dx1"] + dx0n)
    return dxs, grads


LAYER_NAMES = ("g1", "wqkv", "wo", "g2", "wg", "wu", "wd")


def model_step(layers: list, g3, wlm, cfg: LayerConfig, x, shift_labels, position_ids=None, P: int = 1,
               mlp_tiles=None, loss_tile=None, dtype=np.float64, keep_out=False, rope_theta: float = 0.0,
               emb=None) -> StepResult:
    """One SP=P training step (fwd+bwd) of an L-layer decoder stack + final norm + lm_head as
    P in-process ranks.  `layers` holds one dict / LayerParams-like object per layer with LAYER_NAMES.
    Global mean loss via all_reduce of (sum, count); weight grads all-reduced over the SP group
    (SPEC.md:353).  Activation checkpointing and offload do not change these values,
    so this uncheckpointed restatement is the oracle for every checkpoint mode.
    Grads are returned as {"layers.<i>.<name>": ..., "g3": ..., "wlm": ...} (plus bare names for layer 0).
    emb: token embedding table [V, h]; x then holds input_ids [N] and grads["emb"] is
    embed_bwd of the stack's input gradient (summed over ranks like every weight grad)."""
    def get(o, k):
        return np.asarray(o[k] if isinstance(o, dict) else getattr(o, k), dtype=dtype)

    ps = [type("LP", (), {k: get(lp, k) for k in LAYER_NAMES}) for lp in layers]
    g3 = np.asarray(g3, dtype=dtype)
    wlm = np.asarray(wlm, dtype=dtype)
    ids = None
    if emb is not None:
        ids = np.asarray(x, dtype=np.int64)
        x = embed_fwd(ids, np.asarray(emb, dtype=dtype))
    x = np.asarray(x, dtype=dtype)
    N, h = x.shape
    if N % P:
        raise ShapeError(f"N={N} not divisible by P={P}")
    plan_head_shards(cfg.q_heads, cfg.kv_heads, P)  # validates the SP degree
    n_loc = N // P
    if position_ids is None:
        position_ids = np.arange(N, dtype=np.int64)
    starts = block_causal_starts(position_ids)
    loss_tile = n_loc if loss_tile is None else loss_tile
    xs = shard_sequence(x, P)
    labs = shard_sequence(np.asarray(shift_labels, np.int64), P)
    rope = None
    if rope_theta > 0:  # row f4: positions = position_ids (per packed sample) / global token index
        cos, sin = rope_angles(rope_positions(position_ids, True), cfg.head_dim, rope_theta)
        rope = [(cos[r * n_loc:(r + 1) * n_loc], sin[r * n_loc:(r + 1) * n_loc]) for r in range(P)]
    caches = []
    for p in ps:
        xs, cache = decoder_layer_fwd(p, cfg, xs, starts, P, mlp_tiles, rope)
        caches.append(cache)
    # final norm + tiled logits/loss; global (sum, count) via all-reduce
    counts = [int(np.sum(l_ != IGNORE_INDEX)) for l_ in labs]
    count = all_reduce_sum([np.array([c], np.int64) for c in counts])[0][0]
    scale = 1.0 / count if count > 0 else 0.0
    sums, dys, zs, head_grads = [], [], [], []
    for r in range(P):
        z, rstd3 = rmsnorm_fwd(xs[r], g3)
        ls, cnt, dz, dwlm = tiled_logits_loss(z, wlm, labs[r], loss_tile, grad_scale=scale)
        sums.append(np.array([ls], dtype))
        dx2, dg3 = rmsnorm_bwd(xs[r], g3, rstd3, dz)
        dys.append(dx2)
        zs.append(z)
        head_grads.append(dict(g3=dg3, wlm=dwlm))
    loss_sum = float(all_reduce_sum(sums)[0][0])
    out_grads = {k: all_reduce_sum([head_grads[r][k] for r in range(P)])[0] for k in ("g3", "wlm")}
    for i in range(len(ps) - 1, -1, -1):
        dys, grads = decoder_layer_bwd(ps[i], cfg, caches[i], dys, P)
        for k in LAYER_NAMES:  # SP-group weight-grad all-reduce, rank-ascending
            out_grads[f"layers.{i}.{k}"] = all_reduce_sum([grads[r][k] for r in range(P)])[0]
    for k in LAYER_NAMES:
        out_grads[k] = out_grads[f"layers.0.{k}"]
    if ids is not None:
        dx_all = np.concatenate(dys, axis=0)
        demb = np.zeros((wlm.shape[0], h), dtype)
        np.add.at(demb, ids, dx_all)
        out_grads["emb"] = demb
    res = StepResult(loss_sum=loss_sum, count=int(count), loss=loss_sum * scale, dx=np.concatenate(dys, axis=0),
                     grads=out_grads)
    if keep_out:
        res.out_hidden = np.concatenate(zs, axis=0)
    return res


def layer_step(params: LayerParams, cfg: LayerConfig, x, shift_labels, position_ids=None, P: int = 1,
               mlp_tiles=None, loss_tile=None, dtype=np.float64, keep_out=False) -> StepResult:
    """One SP=P training step (fwd+bwd) of ONE decoder layer + final norm + lm_head, as P in-process ranks:
    model_step with a single layer.  Forward per rank: x1 = x + Wo·ulysses_attention(Wqkv·rms(x));
    x2 = x1 + tiled_mlp(rms(x1)); z = rms_final(x2); (loss_sum, count) = tiled_logits_loss(z)."""
    p = params.astype(dtype)
    res = model_step([p], p.g3, p.wlm, cfg, x, shift_labels, position_ids, P, mlp_tiles, loss_tile, dtype, keep_out)
    res.grads = {k: res.grads[k] for k in LayerParams.NAMES}
    return res


def layer_flops(cfg: LayerConfig, n: int) -> float:
    """Model flops of one fwd+bwd step: N[6(P_layer + P_lm) + 6 N Hq d]."""
    h, I, V = cfg.hidden, cfg.intermediate, cfg.vocab
    qd = cfg.q_heads * cfg.head_dim
    p_layer = h * qd + 2 * h * cfg.kv_heads * cfg.head_dim + qd * h + 3 * h * I
    p_lm = V * h
    return n * (6.0 * (p_layer + p_lm) + 6.0 * n * qd)


def finite_diff_grad(f, x: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    """autograd.hpp:34-37 / SPEC.md:89-97 central-difference gradient."""
    g = np.zeros_like(x, dtype=np.float64)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        old = x[i]
        x[i] = old + eps
        fp = f(x)
        x[i] = old - eps
        fm = f(x)
        x[i] = old
        g[i] = (fp - fm) / (2 * eps)
    return g
