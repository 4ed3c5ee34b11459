"""Step-level A/B of a run-time tuning switch (spt_tuning_set) inside one process: the L1 layer step is timed
(CUDA events, --group steps, default 3, after 1 warm-up) alternately under each value, several rounds, and the best time per
value is reported.  Interleaving cancels most of the pod-to-pod and thermal/power drift that makes separate
bench runs differ by several percent.

  python tools/step_ab.py gemm_pair_mn=0,1 [--rounds 4] [--seq 32768]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("switch")
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--group", type=int, default=3, help="timed steps per value per round (10+: sustained, power-capped)")
a = ap.parse_args()
key, vals = a.switch.split("=")
vals = [int(v) for v in vals.split(",")]
L = S.lib()
shp = S.LLAMA8B
grp = S.ProcessGroup.loopback_group(1)
eng = S.UlyssesLayerStep(shp, a.seq, grp)
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
for k, s_ in {"g1": (shp.hidden,), "wqkv": (qkv, shp.hidden), "wo": (shp.hidden, shp.q_heads * shp.head_dim), "g2": (shp.hidden,),
              "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
              "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}.items():
    w = (1 + 0.05 * torch.randn(s_, device="cuda", generator=g)) if k[0] == "g" else 0.02 * torch.randn(
        s_, device="cuda", generator=g)
    eng.set_param(k, w.bfloat16(), on_host=False)
x = torch.randn(a.seq, shp.hidden, device="cuda", generator=g).bfloat16()
lab = torch.randint(0, shp.vocab, (a.seq,), device="cuda", generator=g)
best = {v: 1e9 for v in vals}
losses = {}
for _ in range(a.rounds):
    for v in vals:
        S.check(L.spt_tuning_set(key.encode(), v))
        eng.step_async(x, lab, None, on_host=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.group):
            eng.step_async(x, lab, None, on_host=False)
        e1.record()
        torch.cuda.synchronize()
        best[v] = min(best[v], e0.elapsed_time(e1) / a.group)
        losses[v] = eng.read_loss()[0]
S.check(L.spt_tuning_set(key.encode(), vals[0]))
print(json.dumps({"switch": key, "ms_per_step_best": {str(v): round(t, 2) for v, t in best.items()},
                  "tokens_per_s": {str(v): round(a.seq / t * 1e3, 1) for v, t in best.items()},
                  "loss": {str(v): losses[v] for v in vals}}))
eng.close()
grp.close()
