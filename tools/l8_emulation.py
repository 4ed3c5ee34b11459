"""L8 (BASELINE configs[2]: Llama-3-8B layer, Ulysses SP=8, 512K tokens) emulated on ONE B200: the engine runs
the 8 SP ranks as in-process loopback ranks (real K1/K2 reshard kernels, loopback all-to-all copies instead of
NVLink), so one step does the whole 8-GPU job's compute on one GPU.  Reported: step time, per-class device
time, and the per-rank projection = step / 8 (each rank's compute; NVLink all-to-all time, ~2.2 GiB per rank
per step, is NOT included — it cannot be measured on one GPU).  This is a projection, not an 8-GPU
measurement.

  python tools/l8_emulation.py [--seq 524288] [--sp 8] [--out file.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=524288)
ap.add_argument("--sp", type=int, default=8)
ap.add_argument("--out", default="")
a = ap.parse_args()
shp = S.LLAMA8B
grp = S.ProcessGroup.loopback_group(a.sp)
eng = S.UlyssesLayerStep(shp, a.seq, grp)
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
for k, s_ in {"g1": (shp.hidden,), "wqkv": (qkv, shp.hidden), "wo": (shp.hidden, shp.q_heads * shp.head_dim), "g2": (shp.hidden,),
              "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
              "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}.items():
    w = (1 + 0.05 * torch.randn(s_, device="cuda", generator=g)) if k[0] == "g" else 0.02 * torch.randn(
        s_, device="cuda", generator=g)
    eng.set_param(k, w.bfloat16(), on_host=False)
    del w
x = torch.randn(a.seq, shp.hidden, device="cuda", generator=g).bfloat16()
lab = torch.randint(0, shp.vocab, (a.seq,), device="cuda", generator=g)
lab[-1] = -100
eng.step_async(x, lab, None, on_host=False)  # warm-up
eng.read_loss()
eng.set_profiling(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.step_async(x, lab, None, on_host=False)
e1.record()
t = eng.timing()
loss, cnt = eng.read_loss()
ms = e0.elapsed_time(e1)
mem = eng.memory()
classes = {k: round(v["ms"], 1) for k, v in t["classes"].items() if k != "sites" and v["ms"] > 0}
res = {"config": f"L8 emulation: Llama-3-8B layer + lm_head, seq {a.seq}, SP={a.sp} loopback ranks on 1 GPU",
       "step_ms_all_ranks": round(ms, 1), "per_rank_projection_ms": round(ms / a.sp, 1),
       "projected_tokens_per_s_8gpu_compute_only": round(a.seq / (ms / a.sp) * 1e3, 1),
       "class_ms_all_ranks": classes, "loss": loss, "valid_tokens": cnt,
       "ledger_peak_gib_all_ranks": round(mem["ledger"]["device"]["peak_bytes"] / 2**30, 1),
       "comm_stats": mem["comm"], "note": "compute only; NVLink all-to-all not included (single GPU)"}
print(json.dumps(res))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
eng.close()
grp.close()
