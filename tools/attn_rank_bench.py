"""Attention fwd/bwd at a per-rank shape (default: L8 rank, s=524288, 4 q / 1 kv heads, d=128)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
hq = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hkv = int(sys.argv[3]) if len(sys.argv) > 3 else 1
d = 128
L = S.lib()
g = torch.Generator(device="cuda").manual_seed(3)
qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(hq, s, device="cuda")
do = torch.randn(s, hq, d, device="cuda", generator=g).bfloat16()
dqkv = torch.empty_like(qkv)
ws = torch.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=torch.uint8, device="cuda")
sc = 1 / math.sqrt(d)
fl = 4.0 * s * s * hq * d / 2
fwd = lambda: S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
bwd = lambda: S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s, hq, hkv, d, None,
                                     sc, dqkv.data_ptr(), ws.data_ptr(), None))
fwd()
bwd()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
fwd()
ev[1].record()
bwd()
ev[2].record()
torch.cuda.synchronize()
fw, bw = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
print(f"s={s} hq={hq} hkv={hkv}: fwd {fw:.1f} ms ({fl / fw / 1e9:.0f} TF/s)  bwd {bw:.1f} ms ({2.5 * fl / bw / 1e9:.0f} TF/s)")
