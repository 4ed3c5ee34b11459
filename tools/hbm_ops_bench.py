"""HBM-bound ops added late in round 1, timed with CUDA events (and, under ncu, their DRAM bytes):
token embedding gather / sorted-run backward at L1 size (32768 tokens, h=4096, V=128256) and the K1 pack with
RoPE fused at the L8 rank shape (SP=8 loopback ranks of a 512K-token Llama-3-8B layer, one rank's pack).

  python tools/hbm_ops_bench.py [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
L = S.lib()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json"))) if os.path.exists("MEASURED_PEAKS.json") else {}
hbm = peaks.get("hbm_gbs", 6553.6)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


out = {}
n, h, V = 32768, 4096, 128256
g = torch.Generator(device="cuda").manual_seed(0)
ids = torch.randint(0, V, (n,), device="cuda", generator=g)
table = torch.randn(V, h, device="cuda", generator=g).bfloat16()
x = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
err = torch.zeros(1, dtype=torch.int32, device="cuda")
ms = timed(lambda: S.check(L.spt_embed_fwd(ids.data_ptr(), n, V, h, table.data_ptr(), x.data_ptr(), err.data_ptr(),
                                            None)))
b = 2 * n * h * 2 + n * 8  # rows read + written, ids
out["embed_fwd"] = {"ms": round(ms, 4), "algorithmic_bytes": b, "GB/s": round(b / ms / 1e6, 1),
                    "frac_hbm": round(b / ms / 1e6 / hbm, 3)}
dE = torch.zeros(V, h, device="cuda")
ws = torch.empty(L.spt_embed_bwd_workspace(n, V), dtype=torch.uint8, device="cuda")
ms = timed(lambda: S.check(L.spt_embed_bwd(ids.data_ptr(), n, V, h, x.data_ptr(), dE.data_ptr(), 1, err.data_ptr(),
                                            ws.data_ptr(), None)))
touched = int(torch.unique(ids).numel())
b = n * h * 2 + 2 * touched * h * 4 + n * 32  # dx rows, touched fp32 rows read+written, sort keys/values
out["embed_bwd_accumulate"] = {"ms": round(ms, 4), "algorithmic_bytes": b, "GB/s": round(b / ms / 1e6, 1),
                               "frac_hbm": round(b / ms / 1e6 / hbm, 3), "touched_rows": touched}
del table, dE
torch.cuda.empty_cache()

# K1 pack with fused RoPE at the L8 rank shape: s_loc = 65536 tokens, 32 q + 8 kv heads in, P = 8, 4 q + 2 kv
# (one kv head, replicated r=1... plan from the library) per destination
plan = S.plan_head_shards(32, 8, 8)
s_loc, d, P = 65536, 128, 8
hin = 32 + 2 * 8
qkv = torch.randn(s_loc, hin, d, device="cuda", generator=g).bfloat16()
heads_out = plan.q_heads_per_rank + 2 * plan.kv_heads_per_rank
hm = []
for r in range(P):
    q = S.heads_of(plan, r, 0)
    kv = S.heads_of(plan, r, 1)
    hm += list(q) + [32 + k for k in kv] + [40 + k for k in kv]
head_map = torch.tensor(hm, dtype=torch.int32, device="cuda")
send = torch.empty(P, s_loc, heads_out, d, device="cuda", dtype=torch.bfloat16)
tab = torch.empty(s_loc, d // 2, 2, device="cuda")  # positions 0 .. s_loc - 1 (pos_offset 0)
S.check(L.spt_rope_table(tab.data_ptr(), s_loc, d, 500000.0, None))
b = 2 * P * s_loc * heads_out * d * 2  # every destination row read + written (replicated kv rows read again)
for name, fn in (("reshard_pack", lambda: S.check(L.spt_reshard_pack(qkv.data_ptr(), s_loc, hin, d, P, heads_out,
                                                                     head_map.data_ptr(), send.data_ptr(), None))),
                 ("reshard_pack_rope_in_kernel_angles", lambda: S.check(L.spt_reshard_pack_rope(
                     qkv.data_ptr(), s_loc, hin, d, P, heads_out, head_map.data_ptr(), send.data_ptr(), 40, None,
                     0, 500000.0, None, None))),
                 ("reshard_pack_rope_table", lambda: S.check(L.spt_reshard_pack_rope(
                     qkv.data_ptr(), s_loc, hin, d, P, heads_out, head_map.data_ptr(), send.data_ptr(), 40, None,
                     0, 500000.0, tab.data_ptr(), None)))):
    ms = timed(fn)
    out[name] = {"ms": round(ms, 4), "algorithmic_bytes": b, "GB/s": round(b / ms / 1e6, 1),
                 "frac_hbm": round(b / ms / 1e6 / hbm, 3)}
# the unfused alternative: in-place rope pass over the q/k heads, then the plain pack
rb = 2 * s_loc * 40 * d * 2
ms = timed(lambda: S.check(L.spt_rope(qkv.data_ptr(), s_loc, hin, 40, d, None, 0, 500000.0, 0, None)))
out["rope_inplace_pass"] = {"ms": round(ms, 4), "algorithmic_bytes": rb, "GB/s": round(rb / ms / 1e6, 1),
                            "frac_hbm": round(rb / ms / 1e6 / hbm, 3)}
print(json.dumps(out))
