"""A/B the same GEMM with B K-major vs MN-major (and A K/MN-major) to isolate the operand-major cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

L = S.lib()
M, N, K = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 28672))]
A = torch.randn(M, K, device="cuda").bfloat16()
At = A.t().contiguous()
B = torch.randn(N, K, device="cuda").bfloat16()
Bt = B.t().contiguous()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for name, a, amn, b, bmn in (("KK", A, 0, B, 0), ("KMN", A, 0, Bt, 1), ("MNK", At, 1, B, 0), ("MNMN", At, 1, Bt, 1)):
    def run():
        S.check(L.spt_gemm_bf16(a.data_ptr(), a.shape[1], amn, b.data_ptr(), b.shape[1], bmn, C.data_ptr(), N, 0, 0,
                                None, 0, M, N, K, 1.0, None))
    try:
        for _ in range(3):
            run()
    except Exception as e:  # unsupported combination
        print(name, "unsupported", e)
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name:5s} M={M} N={N} K={K}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.1f} TF/s")
