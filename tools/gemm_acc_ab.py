"""Wgrad-shaped GEMM (MN x MN) with bf16 output vs fp32 output vs fp32 accumulate (C += ...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

L = S.lib()
M, N, K = [int(x) for x in sys.argv[1:4]]
At = torch.randn(K, M, device="cuda").bfloat16()
Bt = torch.randn(K, N, device="cuda").bfloat16()
Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
Cf = torch.zeros(M, N, device="cuda", dtype=torch.float32)
for name, C, f32, acc in (("bf16", Cb, 0, 0), ("f32", Cf, 1, 0), ("f32+acc", Cf, 1, 1)):
    def run():
        S.check(L.spt_gemm_bf16(At.data_ptr(), M, 1, Bt.data_ptr(), N, 1, C.data_ptr(), N, f32, acc, None, 0, M, N, K,
                                1.0, None))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"MNMN {name:8s} M={M} N={N} K={K}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.1f} TF/s")
