"""Interleaved A/B of attention-forward variants (spt_tuning_set("attn_fwd_bk128", v)) at given shapes, with the
output of every variant compared against the default (v=1): norm-wise O error and max |LSE| difference.
  python tools/attn_fwd_ab.py 1,12,13,14 32768:32:8 131072:4:1 [--rounds 3]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

vals = [int(v) for v in sys.argv[1].split(",")]
rounds = 3
args = [a for a in sys.argv[2:] if not a.startswith("--")]
if "--rounds" in sys.argv:
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1])
    args = [a for a in args if a != str(rounds)]
L = S.lib()
d = 128
for shp in args:
    s, hq, hkv = (int(x) for x in shp.split(":"))
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
    o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(hq, s, device="cuda")
    sc = 1 / math.sqrt(d)
    fl = 4.0 * s * s * hq * d / 2
    n = max(1, int(2e13 / fl))

    def run(v, reps):
        S.check(L.spt_tuning_set(b"attn_fwd_bk128", v))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    run(1, 1)
    o_ref, l_ref = o.float().clone(), lse.clone()
    best = {v: 1e30 for v in vals}
    for v in vals:
        run(v, 1)
        err = ((o.float() - o_ref).norm() / o_ref.norm()).item()
        lerr = (lse - l_ref).abs().max().item()
        print(f"s={s} hq={hq} hkv={hkv} v={v}: O rel {err:.2e}  LSE max abs {lerr:.2e}", flush=True)
    for _ in range(rounds):
        for v in vals:
            best[v] = min(best[v], run(v, n))
    print(f"s={s} hq={hq} hkv={hkv}: " + "  ".join(f"v={v} {best[v]:.3f} ms ({fl / best[v] / 1e9:.0f} TF/s)"
                                                    for v in vals), flush=True)
    S.check(L.spt_tuning_set(b"attn_fwd_bk128", 1))
    del qkv, o, lse
    torch.cuda.empty_cache()
