import math, sys, torch
sys.path.insert(0, '.')
import paper_2506_13996_b200 as S
L = S.lib()
S.check(L.spt_tuning_set(b"attn_bwd", 2))
dbg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
S.check(L.spt_tuning_set(b"attn_bwd4_dbg", dbg))
s, hq, hkv, d = 32768, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(3)
qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(hq, s, device="cuda")
do = torch.randn(s, hq, d, device="cuda", generator=g).bfloat16()
ws = torch.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=torch.uint8, device="cuda")
sc = 1 / math.sqrt(d)
S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
dqkv = torch.zeros_like(qkv)
S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s, hq, hkv, d, None, sc, dqkv.data_ptr(), ws.data_ptr(), None))
torch.cuda.synchronize()
print("done")
