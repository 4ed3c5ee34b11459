"""Library yardstick for the attention kernels: torch SDPA (cuDNN / flash backends) at the L1 shape,
causal GQA 32q/8kv d=128, fwd and fwd+bwd timed with CUDA events (model flops, causal = half)."""
import sys
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

s = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
hq, hkv, d = 32, 8, 128
q = torch.randn(1, hq, s, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
k = torch.randn(1, hkv, s, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
v = torch.randn(1, hkv, s, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
fl = 4.0 * s * s * hq * d / 2
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            def f():
                return torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
            o = f()
            g = torch.randn_like(o)
            for _ in range(2):
                o = f(); o.backward(g)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            n = 5
            e[0].record()
            for _ in range(n):
                o = f()
            e[1].record()
            for _ in range(n):
                o = f(); o.backward(g)
            e[2].record()
            torch.cuda.synchronize()
            fw = e[0].elapsed_time(e[1]) / n
            fb = e[1].elapsed_time(e[2]) / n
            print(f"{name}: fwd {fw:.3f} ms ({fl / fw / 1e9:.0f} TF/s)  bwd {fb - fw:.3f} ms "
                  f"({2.5 * fl / (fb - fw) / 1e9:.0f} TF/s)", flush=True)
    except Exception as ex:  # backend unavailable for this shape
        print(f"{name}: unavailable ({str(ex).splitlines()[0][:120]})")
