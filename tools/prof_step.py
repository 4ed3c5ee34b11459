"""Run W warm-up + K layer steps of the bench workload (device-resident inputs) for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--sp", type=int, default=1)
a = ap.parse_args()
shp = S.LLAMA8B
grp = S.ProcessGroup.loopback_group(a.sp)
eng = S.UlyssesLayerStep(shp, a.seq, grp)
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
for k, s_ in {"g1": (shp.hidden,), "wqkv": (qkv, shp.hidden), "wo": (shp.hidden, shp.q_heads * shp.head_dim), "g2": (shp.hidden,),
              "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
              "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}.items():
    w = (1 + 0.05 * torch.randn(s_, device="cuda", generator=g)) if k[0] == "g" else 0.02 * torch.randn(s_, device="cuda", generator=g)
    eng.set_param(k, w.bfloat16(), on_host=False)
x = torch.randn(a.seq, shp.hidden, device="cuda", generator=g).bfloat16()
lab = torch.randint(0, shp.vocab, (a.seq,), device="cuda", generator=g)
for _ in range(a.warmup + a.steps):
    eng.step_async(x, lab, None, on_host=False)
print(eng.read_loss())
