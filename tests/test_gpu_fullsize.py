"""Parity at BASELINE config L1's full size (N=32768, Llama-3-8B layer shapes, V=128256) (pytest -m gpu).

The numpy oracle cannot run this size in test time, so the checker is tests/torch_ref.py — the same
step in plain PyTorch fp32 (TF32 off) with autograd, pinned to the oracle in test_torch_ref_cpu.py —
run on the same B200 from the same bf16 bits.  Tolerances are the north_star contract: loss
rel-err <= 1e-3, every weight grad and d x rel-err <= 2e-2 (norm-wise).  SURVEY.md §8(c) parity
protocol items 1-2: SP=1 and SP=2 (loopback virtual ranks through the real K1/K2 + all_to_all) at 32K.
"""
import pytest

from tests.gpu_util import torch

pytestmark = pytest.mark.gpu

import paper_2506_13996_b200 as S  # noqa: E402

LOSS_TOL = 1e-3
GRAD_TOL = 2e-2


def _synth(shape, N, packed, seed=11):
    T = torch()
    g = T.Generator(device="cuda").manual_seed(seed)
    h, I, V = shape.hidden, shape.intermediate, shape.vocab
    qkv = (shape.q_heads + 2 * shape.kv_heads) * shape.head_dim

    def w(*sh):
        return (T.randn(*sh, device="cuda", generator=g) * 0.02).bfloat16()

    def gam():
        return (1 + 0.05 * T.randn(h, device="cuda", generator=g)).bfloat16()

    params = dict(g1=gam(), wqkv=w(qkv, h), wo=w(h, shape.q_heads * shape.head_dim), g2=gam(), wg=w(I, h),
                  wu=w(I, h), wd=w(h, I), g3=gam(), wlm=w(V, h))
    x = T.randn(N, h, device="cuda", generator=g).bfloat16()
    lab = T.randint(0, V, (N,), device="cuda", generator=g)
    lab[T.rand(N, device="cuda", generator=g) < 0.05] = -100
    lab = T.cat([lab[1:], T.full((1,), -100, device="cuda", dtype=lab.dtype)])  # preshift
    if packed:  # runs of U[1K, 8K] tokens
        runs, tot = [], 0
        while tot < N:
            r = int(T.randint(1024, 8193, (1,), generator=T.Generator().manual_seed(seed + tot)).item())
            runs.append(min(r, N - tot))
            tot += runs[-1]
        pos = T.cat([T.arange(r, device="cuda") for r in runs])
    else:
        pos = T.arange(N, device="cuda")
    return params, x, lab, pos


def _rel(a, b):
    T = torch()
    a, b = a.double(), b.double()
    return float(T.linalg.vector_norm(a - b) / T.linalg.vector_norm(b).clamp_min(1e-300))


@pytest.fixture(scope="module")
def l1_case():
    T = torch()
    from tests import torch_ref as R

    shape = S.LLAMA8B
    out = {}
    for packed in (False, True):
        params, x, lab, pos = _synth(shape, 32768, packed)
        T.backends.cuda.matmul.allow_tf32 = False
        loss, cnt, grads, dx = R.layer_step({k: v.float() for k, v in params.items()}, x.float(), lab,
                                            pos if packed else None, shape.q_heads, shape.kv_heads, shape.head_dim)
        out[packed] = (params, x, lab, pos, (loss, cnt, grads, dx))
        T.cuda.empty_cache()
    return shape, out


@pytest.mark.parametrize("P,packed", [(1, False), (2, False), (1, True)])
def test_l1_fullsize_matches_fp32_reference(l1_case, P, packed):
    T = torch()
    shape, out = l1_case
    params, x, lab, pos, (rloss, rcnt, rgrads, rdx) = out[packed]
    N = x.shape[0]
    grp = S.ProcessGroup.loopback_group(P)
    eng = S.UlyssesLayerStep(shape, N, grp, packed=packed)
    try:
        for k in S.PARAM_NAMES:
            eng.set_param(k, params[k])
        loss, cnt = eng.step(x, lab, pos if packed else None)
        assert cnt == rcnt
        errs = {"loss": abs(loss - rloss) / abs(rloss)}
        print(f"\nL1 P={P} packed={packed} loss={loss:.6f} ref={rloss:.6f}", end=" ")
        assert abs(loss - rloss) / abs(rloss) <= LOSS_TOL, (loss, rloss)
        for k in S.PARAM_NAMES:
            gk = T.from_numpy(eng.grad(k)).cuda()
            e = _rel(gk, rgrads[k])
            errs[k] = e
            assert e <= GRAD_TOL, (k, e)
            del gk
        dx = T.from_numpy(eng.dx_bits(N).view("int16")).cuda().view(T.bfloat16).float()
        errs["dx"] = _rel(dx, rdx)
        print(" ".join(f"{k}={v:.2e}" for k, v in errs.items()))
        assert errs["dx"] <= GRAD_TOL
    finally:
        eng.close()
        grp.close()
