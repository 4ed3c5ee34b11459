"""One causal GQA attention forward of ours and one of FlashAttention-4 (library comparator, vllm_flash_attn.cute)
at the same shape, each after a warm-up, for a side-by-side `ncu --set full` capture:

  ncu --set full --clock-control none -k regex:'fwd_tc128|flash|Flash' -c 4 -o out python tools/attn_fwd_ncu_pair.py

Shape s:hq:hkv (default 32768:32:8, the L1 shape), d = 128."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

s, hq, hkv = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32768:32:8").split(":"))
d = 128
L = S.lib()
g = torch.Generator(device="cuda").manual_seed(1)
qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(hq, s, device="cuda")
for _ in range(2):
    S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, 1 / math.sqrt(d), o.data_ptr(), lse.data_ptr(), None))
torch.cuda.synchronize()
try:
    from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd

    q = qkv[:, :hq].unsqueeze(0).contiguous()
    k = qkv[:, hq:hq + hkv].unsqueeze(0).contiguous()
    v = qkv[:, hq + hkv:].unsqueeze(0).contiguous()
    for _ in range(2):
        o2 = _flash_attn_fwd(q, k, v, causal=True, return_lse=True)[0]
    torch.cuda.synchronize()
    err = ((o2[0].float() - o.float()).norm() / o.float().norm()).item()
    print(f"FA4 vs ours O rel err {err:.2e}")
except Exception as ex:  # comparator only
    print("FA4 unavailable:", type(ex).__name__, str(ex).splitlines()[0][:200])
