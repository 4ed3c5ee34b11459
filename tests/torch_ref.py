"""Plain-PyTorch fp32 reference of the layer step, usable at BASELINE sizes (test infrastructure only).

The numpy oracle (oracle/sptrain_oracle.py) is the parity anchor but cannot run config L1
(N=32768, V=128256) in test time.  This module restates the same step with torch autograd so the
full-size GPU parity test can run it on the B200 itself in fp32 (TF32 off):
  * same composition as oracle.layer_step — rms -> Wqkv -> attention ->
    Wo + res -> rms -> gated MLP + res -> final rms -> lm_head + CE (sum / global count);
  * attention and logits are evaluated in query / token chunks under torch.utils.checkpoint, so no
    [s, s] or [N, V] tensor is ever live (the memory rule of SPEC.md:408 applied to the checker);
  * checked against the oracle at small sizes in tests/test_torch_ref_cpu.py before it is trusted.
It is never imported by the product package.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F
from torch.utils.checkpoint import checkpoint

NAMES = ("g1", "wqkv", "wo", "g2", "wg", "wu", "wd", "g3", "wlm")


def rms(x, g, eps=1e-5):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g


def _attn_chunk(q, k, v, q0, seg_start, scale):
    # q [H, c, d] for queries q0..q0+c-1; k/v [H, q0+c, d] (GQA already expanded)
    c = q.shape[1]
    s = torch.matmul(q, k.transpose(1, 2)) * scale
    qi = torch.arange(q0, q0 + c, device=q.device)[:, None]
    kj = torch.arange(k.shape[1], device=q.device)[None, :]
    allowed = (kj <= qi) & (kj >= seg_start[q0:q0 + c, None])
    s = s.masked_fill(~allowed, float("-inf"))
    return torch.matmul(torch.softmax(s, dim=-1), v)


def attention(q, k, v, seg_start, chunk=1024):
    """Causal (block-causal by seg_start) GQA attention. q [s, Hq, d], k/v [s, Hkv, d] -> [s, Hq, d]."""
    s, Hq, d = q.shape
    g = Hq // k.shape[1]
    scale = 1.0 / math.sqrt(d)
    qh = q.permute(1, 0, 2)
    kh = k.permute(1, 0, 2).repeat_interleave(g, dim=0)
    vh = v.permute(1, 0, 2).repeat_interleave(g, dim=0)
    outs = []
    for q0 in range(0, s, chunk):
        q1 = min(s, q0 + chunk)
        outs.append(checkpoint(_attn_chunk, qh[:, q0:q1], kh[:, :q1], vh[:, :q1], q0, seg_start, scale,
                               use_reentrant=False))
    return torch.cat(outs, dim=1).permute(1, 0, 2)


def _ce_chunk(z, w, lab):
    return F.cross_entropy(z @ w.t(), lab, ignore_index=-100, reduction="sum")


def seg_starts_of(position_ids):
    """Per-token start index of its zero-based position run."""
    n = position_ids.shape[0]
    idx = torch.arange(n, device=position_ids.device)
    is_start = position_ids == 0
    is_start[0] = True
    st = torch.where(is_start, idx, torch.zeros_like(idx))
    return torch.cummax(st, dim=0).values


def layer_step(params: dict, x, labels, position_ids=None, q_heads=None, kv_heads=None, head_dim=None,
               attn_chunk=1024, loss_chunk=4096):
    """fp32 (or f64) autograd reference.  params: name -> tensor (float); x [N, h]; labels [N] int64.

    Returns (loss_mean, count, grads dict, dx).
    """
    p = {k: params[k].detach().clone().requires_grad_(True) for k in NAMES}
    x = x.detach().clone().requires_grad_(True)
    N, h = x.shape
    Hq, Hkv, d = q_heads, kv_heads, head_dim
    if position_ids is None:
        position_ids = torch.arange(N, device=x.device)
    seg = seg_starts_of(position_ids)
    xn1 = rms(x, p["g1"])
    qkv = xn1 @ p["wqkv"].t()
    q = qkv[:, :Hq * d].reshape(N, Hq, d)
    k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(N, Hkv, d)
    v = qkv[:, (Hq + Hkv) * d:].reshape(N, Hkv, d)
    o = attention(q, k, v, seg, attn_chunk).reshape(N, Hq * d)
    x1 = x + o @ p["wo"].t()
    xn2 = rms(x1, p["g2"])
    x2 = x1 + (F.silu(xn2 @ p["wg"].t()) * (xn2 @ p["wu"].t())) @ p["wd"].t()
    z = rms(x2, p["g3"])
    count = int((labels != -100).sum())
    total = x.new_zeros(())
    for a in range(0, N, loss_chunk):
        b = min(N, a + loss_chunk)
        total = total + checkpoint(_ce_chunk, z[a:b], p["wlm"], labels[a:b], use_reentrant=False)
    loss = total / max(count, 1)
    loss.backward()
    grads = {k: p[k].grad.detach() for k in NAMES}
    return float(loss.detach()), count, grads, x.grad.detach()
