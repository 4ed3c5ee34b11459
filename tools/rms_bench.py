"""RMSNorm fwd / bwd alone at the L1 shape (n = 32768, h = 4096) through the C-ABI: CUDA-event time and HBM GB/s
(fwd reads x, writes y: 4 h bytes per row; bwd reads x, dy, dres, writes dx: 8 h bytes per row).
  python tools/rms_bench.py [n] [h] [--lib=path/to/libsptrain_b200.so]   (--lib: A/B against another build)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

pos = [a for a in sys.argv[1:] if not a.startswith("--")]
for a in sys.argv[1:]:
    if a.startswith("--lib="):
        S.LIB_PATH = os.path.abspath(a.split("=", 1)[1])
n = int(pos[0]) if len(pos) > 0 else 32768
h = int(pos[1]) if len(pos) > 1 else 4096
L = S.lib()
x = torch.randn(n, h, device="cuda").bfloat16()
g = (1 + 0.05 * torch.randn(h, device="cuda")).bfloat16()
y = torch.empty_like(x)
dy = torch.randn_like(x)
dres = torch.randn_like(x)
dx = torch.empty_like(x)
rstd = torch.empty(n, device="cuda")
dg = torch.zeros(h, device="cuda")
ws = torch.empty(L.spt_rmsnorm_bwd_workspace(n, h), dtype=torch.uint8, device="cuda")


def fwd():
    S.check(L.spt_rmsnorm_fwd(x.data_ptr(), g.data_ptr(), y.data_ptr(), rstd.data_ptr(), n, h, 1e-5, None))


def bwd():
    S.check(L.spt_rmsnorm_bwd(x.data_ptr(), g.data_ptr(), rstd.data_ptr(), dy.data_ptr(), dres.data_ptr(),
                              dx.data_ptr(), dg.data_ptr(), ws.data_ptr(), n, h, None))


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tf = min(timed(fwd) for _ in range(3))
tb = min(timed(bwd) for _ in range(3))
print(f"rmsnorm n={n} h={h}: fwd {tf * 1e3:.1f} us ({4 * n * h / tf / 1e6:.0f} GB/s)  "
      f"bwd {tb * 1e3:.1f} us ({8 * n * h / tb / 1e6:.0f} GB/s, + dgamma column sum)")
