"""Interleaved A/B of the attention forward between BUILDS of the library (compile-time variants): every library
file is loaded into the same process (separate ctypes handles), and the forward is timed alternately under each,
best of --rounds.  Outputs are compared bitwise against the first library.

  python tools/lib_ab_fwd.py path/a.so path/b.so ... [--shapes 32768:32:8,524288:4:1] [--rounds 5]
"""
import argparse
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--shapes", default="32768:32:8,524288:4:1,131072:4:1")
ap.add_argument("--rounds", type=int, default=5)
a = ap.parse_args()
P, I32, I64, F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
libs = []
for path in a.libs:
    L = C.CDLL(os.path.abspath(path), mode=C.RTLD_LOCAL)
    L.spt_attn_fwd.restype = I32
    L.spt_attn_fwd.argtypes = [P, I64, I32, I32, I32, P, F32, P, P, P]
    libs.append(L)
d = 128
for shp in a.shapes.split(","):
    s, hq, hkv = (int(x) for x in shp.split(":"))
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn(s, hq + 2 * hkv, d, device="cuda", generator=g).bfloat16()
    o = torch.empty(s, hq, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(hq, s, device="cuda")
    fl = 4.0 * s * s * hq * d / 2
    n = max(1, int(2e13 / fl))

    def run(L, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            assert L.spt_attn_fwd(qkv.data_ptr(), s, hq, hkv, d, None, 1 / math.sqrt(d), o.data_ptr(), lse.data_ptr(),
                                  None) == 0
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ref = None
    for i, L in enumerate(libs):
        run(L, 1)
        if ref is None:
            ref = o.clone()
        else:
            print(f"s={s} lib{i}: bitwise {'equal' if torch.equal(o, ref) else 'DIFFERENT'} to lib0")
    best = [1e30] * len(libs)
    for _ in range(a.rounds):
        for i, L in enumerate(libs):
            best[i] = min(best[i], run(L, n))
    print(f"s={s} hq={hq} hkv={hkv}: " + "  ".join(f"lib{i} {b:.3f} ms ({fl / b / 1e9:.0f} TF/s)" for i, b in enumerate(best)),
          flush=True)
