"""Time the tcgen05 GEMM on every GEMM site of the L1 layer step (exact shapes, operand majors and
epilogues, fp32 accumulate where the step accumulates) under the current SPT_GEMM_* environment.

  SPT_GEMM_PAIR_MN=1 SPT_GEMM_BN=128 python tools/gemm_sites.py [--check]

Prints one line per site (ms, TF/s) and a JSON summary line.  --check compares the first 256 rows with
a torch fp32 product.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

L = S.lib()
# name, M, N, K, a_mn, b_mn, f32, accumulate, calls per L1 step
SITES = [
    ("flce_dW", 128256, 4096, 8192, 1, 1, 1, 1, 4),
    ("flce_dx", 8192, 4096, 128256, 0, 1, 0, 0, 4),
    ("mlp_dWgu", 28672, 4096, 4096, 1, 1, 1, 1, 8),
    ("mlp_dx_gu", 4096, 4096, 28672, 0, 1, 0, 0, 8),
    ("mlp_dWd", 4096, 14336, 4096, 1, 1, 1, 1, 8),
    ("mlp_dact", 4096, 14336, 4096, 0, 1, 0, 0, 8),
    ("mlp_down", 4096, 4096, 14336, 0, 0, 0, 0, 8),
    ("qkv_dW", 6144, 4096, 32768, 1, 1, 1, 1, 1),
    ("qkv_dx", 32768, 4096, 6144, 0, 1, 0, 0, 1),
    ("qkv_fwd", 32768, 6144, 4096, 0, 0, 0, 0, 1),
    ("o_dW", 4096, 4096, 32768, 1, 1, 1, 1, 1),
    ("o_dx", 32768, 4096, 4096, 0, 1, 0, 0, 1),
    ("o_fwd", 32768, 4096, 4096, 0, 0, 0, 0, 1),
]
check = "--check" in sys.argv
# --ab key=v1,v2[,v3]: interleaved A/B of a tuning switch inside this process (best of --rounds per value)
ab = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--ab=")), None)
rounds = int(next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--rounds=")), "3"))
only = [a for a in sys.argv[1:] if not a.startswith("--")]
res = {}
tot_ms = 0.0
for name, M, N, K, amn, bmn, f32, acc, calls in SITES:
    if only and name not in only:
        continue
    g = torch.Generator(device="cuda").manual_seed(0)
    A = (torch.randn(K, M, device="cuda", generator=g) if amn else torch.randn(M, K, device="cuda", generator=g)).bfloat16()
    B = (torch.randn(K, N, device="cuda", generator=g) if bmn else torch.randn(N, K, device="cuda", generator=g)).bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)

    def run(a=acc):
        S.check(L.spt_gemm_bf16(A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn, C.data_ptr(), N, f32, a,
                                None, 0, M, N, K, 1.0, None))

    def timed(reps=10):
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    if ab:
        key, vals = ab.split("=")
        best = {}
        for _ in range(rounds):
            for v in vals.split(","):
                S.check(L.spt_tuning_set(key.encode(), int(v)))
                best[v] = min(best.get(v, 1e9), timed())
        S.check(L.spt_tuning_set(key.encode(), int(vals.split(",")[0])))
        print(f"{name:10s} " + "  ".join(f"{key}={v}: {2 * M * N * K / t / 1e9:7.1f} TF/s" for v, t in best.items()),
              flush=True)
        del A, B, C
        torch.cuda.empty_cache()
        continue
    ms = timed()
    tf = 2 * M * N * K / ms / 1e9
    line = f"{name:10s} M={M:6d} N={N:6d} K={K:6d} {'MN' if amn else 'K'}{'MN' if bmn else 'K'} " \
           f"{'f32' if f32 else 'bf16'}{'+acc' if acc else ''}: {ms:7.3f} ms {tf:7.1f} TF/s"
    if check:
        run(0)
        ref = (A.float().t() if amn else A.float())[:256] @ (B.float() if bmn else B.float().t())
        err = ((C[:256].float() - ref).norm() / ref.norm()).item()
        line += f"  err {err:.1e}"
        assert err < 1e-2, (name, err)
    print(line, flush=True)
    res[name] = round(tf, 1)
    tot_ms += ms * calls
    del A, B, C
    torch.cuda.empty_cache()
env = {k: v for k, v in os.environ.items() if k.startswith("SPT_")}
print(json.dumps({"env": env, "tflops": res, "step_gemm_ms_est": round(tot_ms, 3)}))
