"""Library yardstick #2: FlashAttention-4 (the CuTe-DSL sm100 kernels vendored in vllm, `vllm_flash_attn.cute`)
at the L1 attention shape and the L8 / Q8 per-rank shapes, fwd and bwd (non-deterministic and deterministic),
CUDA events, model flops (causal = half, bwd = 2.5x fwd).  Library code: a comparator, never on our path.
usage: python tools/attn_fa4_bench.py [s:hq:hkv ...]"""
import sys
import torch

from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd, _flash_attn_bwd

shapes = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(32768, 32, 8), (524288, 4, 1)]
d = 128
for s, hq, hkv in shapes:
    q = torch.randn(1, s, hq, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, s, hkv, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, s, hkv, d, device="cuda", dtype=torch.bfloat16)
    fl = 4.0 * s * s * hq * d / 2
    n = 5 if s <= 65536 else 2
    try:
        o, lse = _flash_attn_fwd(q, k, v, causal=True, return_lse=True)[:2]
        do = torch.randn_like(o)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(2):
            _flash_attn_fwd(q, k, v, causal=True, return_lse=True)
        torch.cuda.synchronize(); e[0].record()
        for _ in range(n):
            _flash_attn_fwd(q, k, v, causal=True, return_lse=True)
        e[1].record(); torch.cuda.synchronize()
        fw = e[0].elapsed_time(e[1]) / n
        res = [f"s={s} hq={hq} hkv={hkv}: fwd {fw:.3f} ms ({fl / fw / 1e9:.0f} TF/s)"]
        for det in (False, True):
            try:
                for _ in range(2):
                    _flash_attn_bwd(q, k, v, o, do, lse, causal=True, deterministic=det)
                torch.cuda.synchronize(); e[0].record()
                for _ in range(n):
                    _flash_attn_bwd(q, k, v, o, do, lse, causal=True, deterministic=det)
                e[1].record(); torch.cuda.synchronize()
                bw = e[0].elapsed_time(e[1]) / n
                res.append(f"bwd(det={int(det)}) {bw:.3f} ms ({2.5 * fl / bw / 1e9:.0f} TF/s)")
            except Exception as ex:
                res.append(f"bwd(det={int(det)}) unavailable ({str(ex).splitlines()[0][:160]})")
        print("  ".join(res), flush=True)
    except Exception as ex:
        print(f"s={s} hq={hq} hkv={hkv}: unavailable ({type(ex).__name__}: {str(ex).splitlines()[0][:200]})", flush=True)
    del q, k, v
    torch.cuda.empty_cache()
