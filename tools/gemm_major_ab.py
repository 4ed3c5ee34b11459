"""Operand-major A/B of the tcgen05 GEMM against cuBLAS on the L1 step's GEMM shapes.

For each (M, N, K) the same product runs with every operand-major combination (K-major = row-major [M, K] /
[N, K]; MN-major = [K, M] / [K, N]), bf16 output, on our kernel (spt_gemm_bf16) and on cuBLAS (torch.matmul
on the matching transposed views), interleaved, best of --rounds.  Separates what the operand layout costs
the kernel from what the step's power cap costs it.

  python tools/gemm_major_ab.py [--rounds=3] [--reps=20]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

L = S.lib()
SHAPES = [  # name, M, N, K
    ("mlp_dact_16384x14336x4096", 16384, 14336, 4096),
    ("mlp_dx_gu_16384x4096x28672", 16384, 4096, 28672),
    ("o_32768x4096x4096", 32768, 4096, 4096),
    ("flce_dx_8192x4096x128256", 8192, 4096, 128256),
]
rounds = int(next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--rounds=")), "3"))
reps = int(next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--reps=")), "20"))


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for name, M, N, K in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(0)
    Ak = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Bk = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    Am, Bm = Ak.t().contiguous(), Bk.t().contiguous()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ref = Ak[:256].float() @ Bk.float().t()
    fns = {}
    for amn, bmn in ((0, 0), (0, 1), (1, 1)):  # (MN, K) is not a step shape and has no kernel instance
        for mode in ("1sm", "pair"):
            A, B = (Am if amn else Ak), (Bm if bmn else Bk)
            tag = ("MN" if amn else "K") + ("MN" if bmn else "K")

            def ours(A=A, B=B, amn=amn, bmn=bmn, mode=mode):
                # 1sm: CTA pairs off; pair: CTA pairs for every operand major (gemm_pair_mn = 1)
                L.spt_tuning_set(b"gemm_1sm", 1 if mode == "1sm" else 0)
                L.spt_tuning_set(b"gemm_pair_mn", 1 if mode == "pair" else 0)
                S.check(L.spt_gemm_bf16(A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn, C.data_ptr(), N,
                                        0, 0, None, 0, M, N, K, 1.0, None))

            fns[f"ours_{mode}_" + tag] = ours

        def cublas(A=A, B=B, amn=amn, bmn=bmn):
            torch.matmul(A.t() if amn else A, B if bmn else B.t(), out=C)

        fns["cublas_" + tag] = cublas
    best = {k: float("inf") for k in fns}
    for _ in range(rounds):
        for k, fn in fns.items():
            best[k] = min(best[k], timed(fn))
    errs = {}
    for k, fn in fns.items():
        fn()
        torch.cuda.synchronize()
        errs[k] = ((C[:256].float() - ref).norm() / ref.norm()).item()
    fl = 2.0 * M * N * K
    out[name] = {k: {"ms": round(v, 4), "tflops": round(fl / v / 1e9, 1), "err": float(f"{errs[k]:.1e}")}
                 for k, v in best.items()}
    print(name, "  ".join(f"{k} {v:.3f} ms {fl / v / 1e9:.0f} TF/s" for k, v in best.items()), flush=True)
    del Ak, Bk, Am, Bm, C
    torch.cuda.empty_cache()
print(json.dumps(out))
