"""Interleaved A/B of attention-forward variants (spt_tuning_set(key, v), key attn_fwd_bk128 by default) at given
shapes, with the output of every variant compared against the first value's: norm-wise O error and max |LSE|
difference.
  python tools/attn_fwd_ab.py 1,11,12,13 32768:32:8 131072:4:1 [--rounds 3] [--key attn_kv_group --reset 0]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

vals = [int(v) for v in sys.argv[1].split(",")]
rounds = 3
key, reset = b"attn_fwd_bk128", 1
opts = {}
for o in ("--rounds", "--key", "--reset"):
    if o in sys.argv:
        opts[o] = sys.argv[sys.argv.index(o) + 1]
args = [a for a in sys.argv[2:] if not a.startswith("--") and a not in opts.values()]
rounds = int(opts.get("--rounds", rounds))
key = opts.get("--key", key.decode()).encode()
reset = int(opts.get("--reset", reset))
for a_ in sys.argv[1:]:
    if a_.startswith("--lib="):  # A/B against another build of the library (same switch values)
        S.LIB_PATH = os.path.abspath(a_.split("=", 1)[1])
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
        S.check(L.spt_tuning_set(key, v))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            S.check(L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, sc, o.data_ptr(), lse.data_ptr(), None))
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    run(vals[0], 1)
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
    S.check(L.spt_tuning_set(key, reset))
    del qkv, o, lse
    torch.cuda.empty_cache()
