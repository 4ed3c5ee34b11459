"""Step-level A/B of an engine CONFIG field (not a run-time switch): one engine per value, each timed over
--group steps in turn for several interleaved rounds; best ms per value.  Same weights / inputs for all.

  python tools/config_ab.py mlp_tiles=0,4,2 [--rounds 3] [--group 10] [--seq 32768] [--loss-tile 0]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("field")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--group", type=int, default=10)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--shape", default="llama", choices=["llama", "qwen"])
a = ap.parse_args()
key, vals = a.field.split("=")
vals = [int(v) for v in vals.split(",")]
shp = S.LLAMA8B if a.shape == "llama" else S.QWEN32B
grp = S.ProcessGroup.loopback_group(1)
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
ws = {k: ((1 + 0.05 * torch.randn(s_, device="cuda", generator=g)) if k[0] == "g" else
          0.02 * torch.randn(s_, device="cuda", generator=g)).bfloat16()
      for k, s_ in {"g1": (shp.hidden,), "wqkv": (qkv, shp.hidden), "wo": (shp.hidden, shp.q_heads * shp.head_dim),
                    "g2": (shp.hidden,), "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
                    "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}.items()}
x = torch.randn(a.seq, shp.hidden, device="cuda", generator=g).bfloat16()
lab = torch.randint(0, shp.vocab, (a.seq,), device="cuda", generator=g)
engs = {}
for v in vals:
    engs[v] = S.UlyssesLayerStep(shp, a.seq, grp, **{key: v})
    for k, w in ws.items():
        engs[v].set_param(k, w, on_host=False)
best = {v: 1e9 for v in vals}
losses, mem = {}, {}
for _ in range(a.rounds):
    for v in vals:
        eng = engs[v]
        eng.step_async(x, lab, None, on_host=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.group):
            eng.step_async(x, lab, None, on_host=False)
        e1.record()
        torch.cuda.synchronize()
        best[v] = min(best[v], e0.elapsed_time(e1) / a.group)
        losses[v] = eng.read_loss()[0]
for v in vals:
    m = engs[v].memory()
    mem[v] = {"peak_gib": round(m["ledger"]["device"]["peak_bytes"] / 2**30, 2), "mlp_tile": m["mlp_tile"],
              "loss_tile": m["loss_tile"]}
    engs[v].close()
print(json.dumps({"field": key, "seq": a.seq, "ms_per_step_best": {str(v): round(t, 2) for v, t in best.items()},
                  "tokens_per_s": {str(v): round(a.seq / t * 1e3, 1) for v, t in best.items()},
                  "loss": {str(v): losses[v] for v in vals}, "memory": {str(v): mem[v] for v in vals}}))
grp.close()
