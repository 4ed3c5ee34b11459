"""Maximum sequence length that fits one B200, measured (not extrapolated), plus the per-rank attention
cost of the 8-GPU configurations (L8: 512K tokens / SP=8 -> 4 q heads + 1 kv head over the full 512K
sequence per rank; Q8: 1M tokens / SP=8 -> 8 q + 1 kv heads over 1M).

For each N (SP=1, one GPU) the full layer step (Llama-3-8B shape + lm_head, TiledMLP, tiled loss) is created
and run twice (one warm-up, one timed with CUDA events); the ledger peak and the device's used bytes are
recorded.  The first N whose engine creation or step fails with an out-of-memory status ends the sweep.

  python tools/max_seq.py [--n 131072,262144,...] [--shape llama|qwen] [--attn] [--out file.json]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="65536,131072,262144,393216,524288")
ap.add_argument("--shape", default="llama")
ap.add_argument("--attn", action="store_true", help="also time per-rank attention of the L8 / Q8 configs")
ap.add_argument("--out", default="")
a = ap.parse_args()
shp = S.LLAMA8B if a.shape == "llama" else S.QWEN32B
dev = torch.device("cuda", 0)
total = torch.cuda.mem_get_info(dev)[1]
res = {"shape": a.shape, "device_total_bytes": total, "points": []}


def params(eng):
    g = torch.Generator(device=dev).manual_seed(1234)
    qkv = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
    ws = {"g1": (shp.hidden,), "wqkv": (qkv, shp.hidden), "wo": (shp.hidden, shp.q_heads * shp.head_dim),
          "g2": (shp.hidden,), "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
          "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}
    for k, s_ in ws.items():
        w = (1 + 0.05 * torch.randn(s_, device=dev, generator=g)) if k[0] == "g" else 0.02 * torch.randn(
            s_, device=dev, generator=g)
        eng.set_param(k, w.bfloat16(), on_host=False)
        del w


grp = S.ProcessGroup.loopback_group(1, 0)
for n in [int(v) for v in a.n.split(",")]:
    pt = {"n": n}
    eng = None
    try:
        eng = S.UlyssesLayerStep(shp, n, grp)
        params(eng)
        g = torch.Generator(device=dev).manual_seed(7)
        x = torch.randn(n, shp.hidden, device=dev, generator=g).bfloat16()
        lab = torch.randint(0, shp.vocab, (n,), device=dev, generator=g)
        lab[-1] = -100
        t0 = time.time()
        eng.step_async(x, lab, None, on_host=False)
        loss0, cnt0 = eng.read_loss()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step_async(x, lab, None, on_host=False)
        e1.record()
        loss, cnt = eng.read_loss()
        ms = e0.elapsed_time(e1)
        free, _ = torch.cuda.mem_get_info(dev)
        led = eng.memory()["ledger"]["device"]
        pt.update({"ok": True, "ms_per_step": round(ms, 1), "tokens_per_s": round(n / ms * 1e3, 1),
                   "loss": loss, "loss_finite": math.isfinite(loss), "ledger_peak_bytes": led["peak_bytes"],
                   "ledger_peak_gib": round(led["peak_bytes"] / 2**30, 2),
                   "device_used_bytes": total - free, "wall_s_two_steps": round(time.time() - t0, 1)})
        del x, lab
    except (S.SptError, torch.OutOfMemoryError) as e:  # engine or input allocation does not fit
        pt.update({"ok": False, "error": str(e)[:200]})
    finally:
        if eng is not None:
            eng.close()
        torch.cuda.empty_cache()
    res["points"].append(pt)
    print(json.dumps(pt), flush=True)
    if not pt["ok"]:
        break
ok = [p["n"] for p in res["points"] if p.get("ok")]
res["max_n_measured"] = max(ok) if ok else 0
grp.close()

if a.attn:
    L = S.lib()
    res["attention_per_rank"] = []
    for name, s, hq, hkv in (("L8 rank (512K, 4q/1kv)", 524288, 4, 1), ("Q8 rank (1M, 8q/1kv)", 1048576, 8, 1)):
        d = 128
        g = torch.Generator(device=dev).manual_seed(3)
        qkv = torch.randn(s, hq + 2 * hkv, d, device=dev, generator=g).bfloat16()
        o = torch.empty(s, hq, d, device=dev, dtype=torch.bfloat16)
        lse = torch.empty(hq, s, device=dev)
        do = torch.randn(s, hq, d, device=dev, generator=g).bfloat16()
        dqkv = torch.empty_like(qkv)
        ws = torch.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=torch.uint8, device=dev)
        sc = 1 / math.sqrt(d)
        fl = 4.0 * s * s * hq * d / 2
        S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
        ev[1].record()
        S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s, hq, hkv, d, None, sc,
                               dqkv.data_ptr(), ws.data_ptr(), None))
        ev[2].record()
        torch.cuda.synchronize()
        fw, bw = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        finite = bool(torch.isfinite(o.float()).all()) and bool(torch.isfinite(dqkv.float()).all())
        r = {"case": name, "s": s, "hq": hq, "hkv": hkv, "fwd_ms": round(fw, 1), "bwd_ms": round(bw, 1),
             "fwd_tflops": round(fl / fw / 1e9, 1), "bwd_tflops": round(2.5 * fl / bw / 1e9, 1), "finite": finite}
        res["attention_per_rank"].append(r)
        print(json.dumps(r), flush=True)
        del qkv, o, lse, do, dqkv, ws
        torch.cuda.empty_cache()
print(json.dumps({"max_n_measured": res["max_n_measured"]}))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
