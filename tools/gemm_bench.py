"""Time the tcgen05 GEMM family on the layer's shapes (CUDA events), 1-SM vs CTA-pair via SPT_GEMM_1SM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

L = S.lib()
cases = [  # name, M, N, K, a_mn, b_mn, f32
    ("logits x.W^T  ", 4096, 128256, 4096, 0, 0, 1),
    ("dx dl.W       ", 4096, 4096, 128256, 0, 1, 0),
    ("dW dl^T.x     ", 128256, 4096, 4096, 1, 1, 1),
    ("mlp up        ", 4096, 28672, 4096, 0, 0, 0),
    ("qkv fwd       ", 32768, 6144, 4096, 0, 0, 0),
]
for name, M, N, K, amn, bmn, f32 in cases:
    A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)

    def run():
        S.check(L.spt_gemm_bf16(A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn, C.data_ptr(), N, f32, 0,
                                None, 0, M, N, K, 1.0, None))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    ref = (A.float().t() if amn else A.float())[:256] @ (B.float() if bmn else B.float().t())
    err = ((C[:256].float() - ref).norm() / ref.norm()).item()
    print(f"{name} M={M:6d} N={N:6d} K={K:6d}: {ms:7.3f} ms {2 * M * N * K / ms / 1e9:7.1f} TF/s  err {err:.1e}")
    del A, B, C
