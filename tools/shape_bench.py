"""Device-resident step throughput for another model shape (default: BASELINE configs[4]'s Qwen 64q/8kv, h=5120,
I=25600, V=151936 at 32K tokens on one GPU, SP=1), with the per-class device-time breakdown.

  python tools/shape_bench.py [--shape qwen|llama] [--seq 32768] [--sp 1] [--steps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="qwen")
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--sp", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
shp = S.QWEN32B if a.shape == "qwen" else S.LLAMA8B
grp = S.ProcessGroup.loopback_group(a.sp)
eng = S.UlyssesLayerStep(shp, a.seq, grp)
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
qd = shp.q_heads * shp.head_dim
for k, s_ in {"g1": (shp.hidden,), "wqkv": (qkv, shp.hidden), "wo": (shp.hidden, qd), "g2": (shp.hidden,),
              "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
              "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}.items():
    w = (1 + 0.05 * torch.randn(s_, device="cuda", generator=g)) if k[0] == "g" else 0.02 * torch.randn(
        s_, device="cuda", generator=g)
    eng.set_param(k, w.bfloat16(), on_host=False)
    del w
x = torch.randn(a.seq, shp.hidden, device="cuda", generator=g).bfloat16()
lab = torch.randint(0, shp.vocab, (a.seq,), device="cuda", generator=g)
lab[-1] = -100
eng.step_async(x, lab, None, on_host=False)
eng.read_loss()
eng.set_profiling(True)
cls = {}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    eng.step_async(x, lab, None, on_host=False)
    for k, v in eng.timing()["classes"].items():
        if k != "sites" and v["ms"] > 0:
            c = cls.setdefault(k, {"ms": 0.0, "flops": 0.0})
            c["ms"] += v["ms"]
            c["flops"] += v["flops"]
e1.record()
loss, cnt = eng.read_loss()
ms = e0.elapsed_time(e1) / a.steps
h, I, V, hq, d = shp.hidden, shp.intermediate, shp.vocab, shp.q_heads, shp.head_dim
p_layer = h * qd + 2 * h * shp.kv_heads * d + qd * h + 3 * h * I
model_flops = a.seq * (6.0 * (p_layer + V * h) + 6.0 * a.seq * hq * d)
print(json.dumps({"shape": a.shape, "seq": a.seq, "sp": a.sp, "ms_per_step": round(ms, 2),
                  "tokens_per_s": round(a.seq / ms * 1e3, 1), "model_tflops": round(model_flops / ms / 1e9, 1),
                  "loss": loss, "peak_hbm_gib": round(eng.memory()["ledger"]["device"]["peak_bytes"] / 2**30, 2),
                  "class_ms": {k: round(v["ms"] / a.steps, 2) for k, v in cls.items()},
                  "class_tflops": {k: round(v["flops"] / v["ms"] / 1e9, 1) for k, v in cls.items() if v["flops"]}}))
eng.close()
grp.close()
