"""Wait-cycle breakdown of the dQ pass from an SPT_DQ_PROF build (SPT_EXTRA_DEFS=SPT_DQ_PROF)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

s, hq, hkv, d = (int(x) for x in (sys.argv[1:4] + ["128"])) if len(sys.argv) > 3 else (32768, 32, 8, 128)
L = S.lib()
f = L.spt_debug_dq_prof
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda").bfloat16()
o = torch.empty(s, hq, d, device="cuda").bfloat16()
lse = torch.empty(hq, s, device="cuda")
do = torch.randn(s, hq, d, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
ws = torch.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=torch.uint8, device="cuda")
sc = 1 / math.sqrt(d)
S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
buf = (C.c_ulonglong * 8)()
for rep in range(2):
    f(buf, 1)
    S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s, hq, hkv, d, None, sc,
                           dqkv.data_ptr(), ws.data_ptr(), None))
    torch.cuda.synchronize()
f(buf, 0)
v = list(buf)
tot = v[4] or 1
print(f"CTAs {v[5]} iterations {v[6]}  per-iteration MMA-warp cycles {tot / max(1, v[6]):.0f}")
print(f"MMA warp: waiting K/V {100 * v[0] / tot:.1f}%  waiting dS (elementwise) {100 * v[1] / tot:.1f}%")
print(f"elementwise warp 0: waiting S {100 * v[2] / tot:.1f}% of the MMA-warp span")
