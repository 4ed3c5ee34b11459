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


# ---- BASELINE configs[4] shape (Q8: 64 q / 8 kv heads, d=128, hidden 5120 != Hq*d, I=25600, V=151936) at a
# reduced N on one GPU, with SP=8 through the loopback ranks (r=1) and a kv-replication variant (Hkv=2,
# SP=8 -> r=4), checked against the same fp32 reference.
Q8_KV2 = S.ModelShape(5120, 64, 2, 128, 25600, 151936)


@pytest.fixture(scope="module")
def q8_case():
    T = torch()
    from tests import torch_ref as R

    out = {}
    for name, shape in (("q8", S.QWEN32B), ("q8_kv2", Q8_KV2)):
        params, x, lab, pos = _synth(shape, 8192, False, seed=23)
        T.backends.cuda.matmul.allow_tf32 = False
        ref = R.layer_step({k: v.float() for k, v in params.items()}, x.float(), lab, None, shape.q_heads,
                           shape.kv_heads, shape.head_dim)
        out[name] = (shape, params, x, lab, ref)
        T.cuda.empty_cache()
    return out


@pytest.mark.parametrize("name,P", [("q8", 1), ("q8", 8), ("q8_kv2", 8)])
def test_q8_shape_matches_fp32_reference(q8_case, name, P):
    T = torch()
    shape, params, x, lab, (rloss, rcnt, rgrads, rdx) = q8_case[name]
    N = x.shape[0]
    plan = S.plan_head_shards(shape.q_heads, shape.kv_heads, P)
    grp = S.ProcessGroup.loopback_group(P)
    eng = S.UlyssesLayerStep(shape, N, grp)
    try:
        for k in S.PARAM_NAMES:
            eng.set_param(k, params[k])
        loss, cnt = eng.step(x, lab)
        assert cnt == rcnt
        errs = {"loss": abs(loss - rloss) / abs(rloss)}
        assert errs["loss"] <= LOSS_TOL, (loss, rloss)
        for k in S.PARAM_NAMES:
            gk = T.from_numpy(eng.grad(k)).cuda()
            errs[k] = _rel(gk, rgrads[k])
            assert errs[k] <= GRAD_TOL, (k, errs[k])
            del gk
        dx = T.from_numpy(eng.dx_bits(N).view("int16")).cuda().view(T.bfloat16).float()
        errs["dx"] = _rel(dx, rdx)
        print(f"\n{name} P={P} kv_replication={plan.kv_replication} " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()))
        assert errs["dx"] <= GRAD_TOL
    finally:
        eng.close()
        grp.close()
