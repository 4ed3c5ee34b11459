"""In-process A/B of an attention tuning switch: the tcgen05 backward (or forward, --fwd) is run under each value on the
same inputs (results compared bitwise against the first value) and timed with CUDA events, interleaved over
several rounds (best per value reported).

  python tools/attn_bwd_ab.py attn_dkdv_pair=0,1 [--shapes 32768x32x8,131072x4x1] [--rounds 5] [--seg]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("switch")
ap.add_argument("--shapes", default="32768x32x8,131072x4x1")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--seg", action="store_true", help="packed sequences (block-causal) instead of plain causal")
ap.add_argument("--fwd", action="store_true", help="time (and compare) the forward instead of the backward")
ap.add_argument("--set", action="append", default=[], help="extra fixed switch name=value (repeatable)")
a = ap.parse_args()
key, vals = a.switch.split("=")
vals = [int(v) for v in vals.split(",")]
L = S.lib()
for kv in a.set:
    k_, v_ = kv.split("=")
    S.check(L.spt_tuning_set(k_.encode(), int(v_)))
d = 128
out = []
for shp in a.shapes.split(","):
    s, hq, hkv = (int(x) for x in shp.split("x"))
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
    o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(hq, s, device="cuda")
    do = torch.randn(s, hq, d, device="cuda", generator=g).bfloat16()
    wsz = 0
    for v in vals:  # the workspace depends on the backward scheme (attn_bwd): size it for every value
        S.check(L.spt_tuning_set(key.encode(), v))
        wsz = max(wsz, L.spt_attn_bwd_workspace(s, hq, hkv, d))
    ws = torch.empty(max(wsz, 1), dtype=torch.uint8, device="cuda")
    seg = None
    if a.seg:  # segment starts: documents of ragged lengths
        starts = torch.zeros(s, dtype=torch.int32, device="cuda")
        cur, pos = 0, 0
        lens = torch.randint(s // 16, s // 3, (64,), generator=torch.Generator().manual_seed(1)).tolist()
        for ln in lens:
            if pos >= s:
                break
            starts[pos:pos + ln] = pos
            pos += ln
        seg = starts
    sp = None if seg is None else seg.data_ptr()
    sc = 1 / math.sqrt(d)
    S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, sp, sc, o.data_ptr(), lse.data_ptr(), None))
    res = {}
    best = {v: 1e9 for v in vals}
    for rnd in range(a.rounds):
        for v in vals:
            S.check(L.spt_tuning_set(key.encode(), v))
            dqkv = torch.zeros_like(qkv)
            o2 = torch.empty_like(o)
            if a.fwd:
                dqkv = o2
                bwd = lambda: S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, sp, sc, o2.data_ptr(),
                                                     lse.data_ptr(), None))
            else:
                bwd = lambda: S.check(L.spt_attn_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), s,
                                                     hq, hkv, d, sp, sc, dqkv.data_ptr(), ws.data_ptr(), None))
            bwd()
            torch.cuda.synchronize()
            if rnd == 0:
                res[v] = dqkv.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                bwd()
            e1.record()
            torch.cuda.synchronize()
            best[v] = min(best[v], e0.elapsed_time(e1) / 3)
    S.check(L.spt_tuning_set(key.encode(), vals[0]))
    ref = res[vals[0]]
    cmp = {}
    for v in vals[1:]:
        diff = (res[v].float() - ref.float()).abs()
        cmp[str(v)] = {"bitwise": bool(torch.equal(res[v], ref)), "max_abs": float(diff.max()),
                       "ref_absmax": float(ref.float().abs().max())}
    line = {"shape": shp, "seg": a.seg, "switch": key, "pass": "fwd" if a.fwd else "bwd",
            "ms_best": {str(v): round(t, 3) for v, t in best.items()},
            "vs_first": cmp}
    print(json.dumps(line), flush=True)
    out.append(line)
    del qkv, o, lse, do, ws, res
    torch.cuda.empty_cache()
