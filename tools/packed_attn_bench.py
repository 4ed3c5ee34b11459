"""Block-diagonal (packed-sample) attention on the tcgen05 kernels vs plain causal over the same total length
(the paper's position_ids note).

Samples of random lengths are packed into one sequence of s tokens; the kernels skip every key block outside
a query's sample (block-causal), so time should track the useful work sum_i len_i^2 rather than s^2.
Reported per mean sample length: fwd / bwd ms, useful TF/s (sum over samples of the causal flops), and the
ratio of the packed time to the full-causal time.

  python tools/packed_attn_bench.py [--seq 131072] [--hq 32 --hkv 8] [--means 2048,8192,32768]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=131072)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--means", default="2048,8192,32768")
ap.add_argument("--out", default="")
a = ap.parse_args()
L = S.lib()
s, hq, hkv, d = a.seq, a.hq, a.hkv, 128
g = torch.Generator(device="cuda").manual_seed(1)
qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
do = torch.randn(s, hq, d, device="cuda", generator=g).bfloat16()
o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(hq, s, device="cuda")
dqkv = torch.empty_like(qkv)
ws = torch.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=torch.uint8, device="cuda")
sc = 1 / math.sqrt(d)


def timed(seg, reps=3):
    sp = None if seg is None else seg.data_ptr()
    fwd = lambda: S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, sp, sc, o.data_ptr(), lse.data_ptr(), None))
    bwd = lambda: S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s, hq, hkv, d,
                                         sp, sc, dqkv.data_ptr(), ws.data_ptr(), None))
    fwd()
    bwd()
    res = []
    for f in (fwd, bwd):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    return res


def causal_flops(n):  # fwd model flops of causal attention over n tokens (4 n^2 hq d / 2)
    return 4.0 * n * n * hq * d / 2.0


full_f, full_b = timed(None)
rows = [{"mean_len": s, "samples": 1, "fwd_ms": round(full_f, 3), "bwd_ms": round(full_b, 3),
         "fwd_tflops_useful": round(causal_flops(s) / full_f / 1e9, 1),
         "bwd_tflops_useful": round(2.5 * causal_flops(s) / full_b / 1e9, 1), "time_vs_causal": 1.0,
         "useful_work_vs_causal": 1.0}]
rng = np.random.default_rng(0)
for mean in (int(m) for m in a.means.split(",")):
    lens = []
    while sum(lens) < s:
        lens.append(int(max(1, rng.exponential(mean))))
    lens[-1] -= sum(lens) - s
    lens = [n for n in lens if n > 0]
    starts = np.concatenate([np.full(n, sum(lens[:i]), np.int32) for i, n in enumerate(lens)])
    seg = torch.from_numpy(starts).cuda()
    f, b = timed(seg)
    useful = sum(causal_flops(n) for n in lens)
    rows.append({"mean_len": mean, "samples": len(lens), "fwd_ms": round(f, 3), "bwd_ms": round(b, 3),
                 "fwd_tflops_useful": round(useful / f / 1e9, 1), "bwd_tflops_useful": round(2.5 * useful / b / 1e9, 1),
                 "time_vs_causal": round((f + b) / (full_f + full_b), 4),
                 "useful_work_vs_causal": round(useful / causal_flops(s), 4)})
res = {"config": f"attention fwd+bwd, s={s}, {hq}q/{hkv}kv, d=128, packed samples with exponential lengths",
       "rows": rows}
print(json.dumps(res))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
