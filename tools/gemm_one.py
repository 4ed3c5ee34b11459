"""One GEMM shape on the tcgen05 kernel (bf16 out, or fp32 accumulate with --f32) for ncu captures / quick timing.

  python tools/gemm_one.py M N K a_mn b_mn [--f32 [--noacc]] [--pair|--1sm] [--reps 5] [--raster R] [--group G]  (gemm_raster mode, raster-0 group size)
e.g. the lm_head dgrad of one loss tile: python tools/gemm_one.py 8192 4096 128256 0 1"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

opt_vals = {sys.argv[i + 1] for i, a in enumerate(sys.argv[:-1]) if a in ("--reps", "--raster", "--group")}
pos = [int(a) for i, a in enumerate(sys.argv[1:], 1) if not a.startswith("--") and not (sys.argv[i - 1] in ("--reps", "--raster", "--group"))]
M, N, K, amn, bmn = pos[:5]
f32 = "--f32" in sys.argv
acc = f32 and "--noacc" not in sys.argv  # fp32 output accumulates (TMA reduce-add) unless --noacc
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
L = S.lib()
if "--pair" in sys.argv:
    L.spt_tuning_set(b"gemm_pair_mn", 1)
if "--1sm" in sys.argv:
    L.spt_tuning_set(b"gemm_1sm", 1)
if "--group" in sys.argv:
    L.spt_tuning_set(b"gemm_group_m", int(sys.argv[sys.argv.index("--group") + 1]))
if "--raster" in sys.argv:
    L.spt_tuning_set(b"gemm_raster", int(sys.argv[sys.argv.index("--raster") + 1]))
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randn(K, M, device="cuda", generator=g) if amn else torch.randn(M, K, device="cuda", generator=g)).bfloat16()
B = (torch.randn(K, N, device="cuda", generator=g) if bmn else torch.randn(N, K, device="cuda", generator=g)).bfloat16()
C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)


def run():
    S.check(L.spt_gemm_bf16(A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn, C.data_ptr(), N, int(f32),
                            int(acc), None, 0, M, N, K, 1.0, None))


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"M={M} N={N} K={K} a_mn={amn} b_mn={bmn} f32={int(f32)} acc={int(acc)}: {ms:.3f} ms {2.0 * M * N * K / ms / 1e9:.0f} TF/s")
