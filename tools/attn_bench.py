"""Time attention fwd/bwd kernels at the L1 shape (s=32768, 32q/8kv, d=128) with CUDA events."""
import os
import sys
import math

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
hq, hkv, d = 32, 8, 128
L = S.lib()
qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda").bfloat16()
o = torch.empty(s, hq, d, device="cuda").bfloat16()
lse = torch.empty(hq, s, device="cuda")
do = torch.randn(s, hq, d, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
ws = torch.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=torch.uint8, device="cuda")
sc = 1 / math.sqrt(d)
fl = 4.0 * s * s * hq * d / 2


def fwd():
    S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))


def bwd():
    S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s, hq, hkv, d, None, sc,
                           dqkv.data_ptr(), ws.data_ptr(), None))


for name, f, flops in (("fwd", fwd, fl), ("bwd", bwd, 2.5 * fl)):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 5
    for _ in range(n):
        f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    print(f"attn {name} impl={os.environ.get('SPT_ATTN_IMPL', 'tc')} s={s}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
# reference check vs flash_attn/sdpa for fwd output
ref = torch.nn.functional.scaled_dot_product_attention(
    qkv[:, :hq].transpose(0, 1).unsqueeze(0), qkv[:, hq:hq + hkv].repeat_interleave(hq // hkv, 1).transpose(0, 1).unsqueeze(0),
    qkv[:, hq + hkv:].repeat_interleave(hq // hkv, 1).transpose(0, 1).unsqueeze(0), is_causal=True) if s <= 8192 else None
if ref is not None:
    fwd()
    err = (o.float() - ref[0].transpose(0, 1).float()).norm() / ref.float().norm()
    print("fwd rel err vs torch sdpa", float(err))
