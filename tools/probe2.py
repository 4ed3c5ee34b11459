import sys, math, torch
sys.path.insert(0, "/root/repo")
import paper_2506_13996_b200 as S
s, hq, hkv = 256, 148, 148
qkv = torch.randn(s, hq + 2 * hkv, 128, device="cuda").bfloat16()
o = torch.empty(s, hq, 128, device="cuda").bfloat16(); lse = torch.empty(hq, s, device="cuda")
S.check(S.lib().spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, 128, None, 1 / math.sqrt(128), o.data_ptr(), lse.data_ptr(), None))
torch.cuda.synchronize(); print("ok")
