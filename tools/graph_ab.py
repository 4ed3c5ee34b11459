"""Eager step_async vs CUDA-graph replay of the same L1 layer step, interleaved groups on one stream
(loss compared bitwise).

  python tools/graph_ab.py [--rounds 4] [--group 12] [--seq 32768]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--group", type=int, default=12)
ap.add_argument("--seq", type=int, default=32768)
a = ap.parse_args()
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
stream = torch.cuda.Stream()
sp = stream.cuda_stream
with torch.cuda.stream(stream):
    eng.graph_capture(x, lab, None, stream=sp)
    best = {"eager": 1e9, "graph": 1e9}
    loss = {}
    for _ in range(a.rounds):
        for mode in ("eager", "graph"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.group):
                if mode == "eager":
                    eng.step_async(x, lab, None, on_host=False, stream=sp)
                else:
                    eng.graph_launch(stream=sp)
            e1.record(stream)
            stream.synchronize()
            best[mode] = min(best[mode], e0.elapsed_time(e1) / a.group)
            loss[mode] = eng.read_loss(stream=sp)[0]
print(json.dumps({"ms_per_step_best": {k: round(v, 2) for k, v in best.items()},
                  "tokens_per_s": {k: round(a.seq / v * 1e3, 1) for k, v in best.items()}, "loss": loss,
                  "loss_bitwise_equal": loss["eager"] == loss["graph"]}))
eng.close()
grp.close()
