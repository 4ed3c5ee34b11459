"""Self-oracle properties of the CPU oracle (SPEC.md §4 style): FD gradients, tiling invariance,
SP=P == SP=1, attention agnosticism, replication equivalence."""
import numpy as np
import pytest

from oracle import sptrain_oracle as O

MINI = O.LayerConfig(hidden=16, q_heads=4, kv_heads=2, head_dim=4, intermediate=32, vocab=50)


def _params(cfg, seed=0, wstd=0.3):
    return O.LayerParams(**O.synth_params(cfg, seed, wstd=wstd)).astype(np.float64)


def _loss(params, cfg, x, lab, pos, **kw):
    return O.layer_step(params, cfg, x, lab, pos, **kw).loss


@pytest.mark.parametrize("name", ["wqkv", "wo", "wg", "wd", "wlm", "g1", "g3"])
def test_layer_fd_gradients(name):
    """tape grads vs central differences, rel err < 1e-6 at f64."""
    cfg = MINI
    p = _params(cfg)
    x, lab, pos = O.synth_batch(cfg, 8, seed=1)
    x = x.astype(np.float64)
    res = O.layer_step(p, cfg, x, lab, pos, P=1, mlp_tiles=3, loss_tile=3)
    w = getattr(p, name)
    rng = np.random.default_rng(2)
    idx = [tuple(rng.integers(0, s) for s in w.shape) for _ in range(6)]
    for i in idx:
        old = w[i]
        w[i] = old + 1e-5
        fp = _loss(p, cfg, x, lab, pos, mlp_tiles=3, loss_tile=3)
        w[i] = old - 1e-5
        fm = _loss(p, cfg, x, lab, pos, mlp_tiles=3, loss_tile=3)
        w[i] = old
        fd = (fp - fm) / 2e-5
        g = res.grads[name][i]
        assert abs(fd - g) <= 1e-6 * max(1e-3, abs(fd)) + 1e-9, (name, i, fd, g)


def test_layer_fd_dx():
    cfg = MINI
    p = _params(cfg)
    x, lab, pos = O.synth_batch(cfg, 8, seed=3)
    x = x.astype(np.float64)
    res = O.layer_step(p, cfg, x, lab, pos)
    for i in [(0, 1), (5, 7), (7, 15)]:
        old = x[i]
        x[i] = old + 1e-5
        fp = _loss(p, cfg, x, lab, pos)
        x[i] = old - 1e-5
        fm = _loss(p, cfg, x, lab, pos)
        x[i] = old
        fd = (fp - fm) / 2e-5
        assert abs(fd - res.dx[i]) <= 1e-6 * max(1e-3, abs(fd)) + 1e-9


@pytest.mark.parametrize("tiles", [1, 2, 3, 7, 16])
def test_tiling_invariance(tiles):
    """values bit-exact per tile count; grads <= 1e-10."""
    cfg = MINI
    p = _params(cfg)
    x, lab, pos = O.synth_batch(cfg, 16, seed=4)
    base = O.layer_step(p, cfg, x, lab, pos, mlp_tiles=1, loss_tile=16)
    t = O.layer_step(p, cfg, x, lab, pos, mlp_tiles=tiles, loss_tile=max(1, 16 // tiles))
    assert t.count == base.count
    assert abs(t.loss_sum - base.loss_sum) <= 1e-10 * abs(base.loss_sum)
    for k in O.LayerParams.NAMES:
        assert np.max(np.abs(t.grads[k] - base.grads[k])) <= 1e-10


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("packed", [False, True])
def test_sp_equivalence(P, packed):
    """SP=P loss and grads equal SP=1 to <= 1e-10 (f64); block-diag callback (:341)."""
    cfg = MINI
    p = _params(cfg)
    x, lab, pos = O.synth_batch(cfg, 16, seed=5, packed=packed)
    base = O.layer_step(p, cfg, x, lab, pos, P=1)
    sp = O.layer_step(p, cfg, x, lab, pos, P=P)
    assert abs(sp.loss - base.loss) <= 1e-10
    assert np.max(np.abs(sp.dx - base.dx)) <= 1e-10
    for k in O.LayerParams.NAMES:
        assert np.max(np.abs(sp.grads[k] - base.grads[k])) <= 1e-10, k


def test_kv_replication_equivalence():
    """(Hq=4, Hkv=1, P=4) kv-projection grads equal the P=1 baseline."""
    cfg = O.LayerConfig(hidden=16, q_heads=4, kv_heads=1, head_dim=4, intermediate=32, vocab=50)
    p = _params(cfg)
    x, lab, pos = O.synth_batch(cfg, 16, seed=6)
    base = O.layer_step(p, cfg, x, lab, pos, P=1)
    sp = O.layer_step(p, cfg, x, lab, pos, P=4)
    assert np.max(np.abs(sp.grads["wqkv"] - base.grads["wqkv"])) <= 1e-10


def test_block_diag_equals_separate_samples():
    """block-diagonal attention on packed samples == per-sample attention."""
    rng = np.random.default_rng(7)
    runs = [5, 3, 8]
    pos = np.concatenate([np.arange(r) for r in runs])
    s = pos.size
    q, k, v = (rng.standard_normal((s, 4, 8)) for _ in range(3))
    k, v = k[:, :2], v[:, :2]
    o, _ = O.attention_fwd(q, k, v, O.block_causal_starts(pos))
    a = 0
    for r in runs:
        o2, _ = O.attention_fwd(q[a:a + r], k[a:a + r], v[a:a + r])
        assert np.max(np.abs(o[a:a + r] - o2)) <= 1e-12
        a += r


def test_all_ignored_loss():
    """all labels -100 -> (0,0) and zero d hidden."""
    cfg = MINI
    p = _params(cfg)
    x, lab, pos = O.synth_batch(cfg, 8, seed=8)
    s, c, dh, dw = O.tiled_logits_loss(x.astype(np.float64) @ np.eye(16), p.wlm, np.full(8, -100), 3, grad_scale=1.0)
    assert (s, c) == (0.0, 0) and not dh.any() and not dw.any()


# ---- L-layer stack (model_step): the SPEC's self-oracles extended to several layers
def test_model_step_sp_equals_sp1_and_fd():
    cfg = O.LayerConfig(hidden=16, q_heads=4, kv_heads=2, head_dim=4, intermediate=32, vocab=40)
    rng = np.random.default_rng(5)
    layers = [{k: v for k, v in O.synth_params(cfg, 11 + i, wstd=0.3).items() if k in O.LAYER_NAMES} for i in range(3)]
    head = O.synth_params(cfg, 3, wstd=0.3)
    N = 8
    x = rng.standard_normal((N, cfg.hidden))
    lab = rng.integers(0, cfg.vocab, N)
    lab[3] = -100
    r1 = O.model_step(layers, head["g3"], head["wlm"], cfg, x, lab, P=1)
    r2 = O.model_step(layers, head["g3"], head["wlm"], cfg, x, lab, P=2)
    assert abs(r1.loss - r2.loss) <= 1e-12
    for k in r1.grads:
        assert np.max(np.abs(r1.grads[k] - r2.grads[k])) <= 1e-10, k
    assert np.max(np.abs(r1.dx - r2.dx)) <= 1e-10
    # central differences on the middle layer's O projection and on the input
    def loss_with(wo):
        ls = [dict(l_) for l_ in layers]
        ls[1]["wo"] = wo
        return O.model_step(ls, head["g3"], head["wlm"], cfg, x, lab, P=1).loss
    fd = O.finite_diff_grad(loss_with, np.asarray(layers[1]["wo"], np.float64))
    assert np.linalg.norm(fd - r1.grads["layers.1.wo"]) / np.linalg.norm(fd) < 1e-6
    fdx = O.finite_diff_grad(lambda xx: O.model_step(layers, head["g3"], head["wlm"], cfg, xx, lab, P=1).loss, x)
    assert np.linalg.norm(fdx - r1.dx) / np.linalg.norm(fdx) < 1e-6


def test_layer_step_is_one_layer_model_step():
    cfg = O.LayerConfig(hidden=16, q_heads=4, kv_heads=2, head_dim=4, intermediate=32, vocab=40)
    p = O.synth_params(cfg, 2, wstd=0.3)
    x, lab, _ = O.synth_batch(cfg, 8, 2)
    a = O.layer_step(O.LayerParams(**p), cfg, x, lab)
    b = O.model_step([{k: p[k] for k in O.LAYER_NAMES}], p["g3"], p["wlm"], cfg, x, lab)
    assert a.loss == b.loss and np.array_equal(a.dx, b.dx)
    for k in O.LayerParams.NAMES:
        assert np.array_equal(a.grads[k], b.grads[k])


# ---- RoPE (row f4; the SPEC omits it, so these are self-oracles: rotation, FD gradient, SP invariance)
def test_rope_is_a_rotation_and_its_inverse():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((6, 3, 8))
    cos, sin = O.rope_angles(np.arange(6), 8, 10000.0)
    y = O.rope_apply(x, cos, sin)
    assert np.allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1))  # norm preserving
    assert np.allclose(O.rope_apply(y, cos, sin, inverse=True), x)
    assert np.allclose(y[0], x[0])  # position 0: identity


def test_model_step_with_rope_fd_and_sp():
    cfg = O.LayerConfig(hidden=16, q_heads=4, kv_heads=2, head_dim=4, intermediate=32, vocab=40)
    rng = np.random.default_rng(9)
    layers = [{k: v for k, v in O.synth_params(cfg, 21 + i, wstd=0.3).items() if k in O.LAYER_NAMES} for i in range(2)]
    head = O.synth_params(cfg, 4, wstd=0.3)
    N = 8
    x = rng.standard_normal((N, cfg.hidden))
    lab = rng.integers(0, cfg.vocab, N)
    r1 = O.model_step(layers, head["g3"], head["wlm"], cfg, x, lab, P=1, rope_theta=100.0)
    r2 = O.model_step(layers, head["g3"], head["wlm"], cfg, x, lab, P=2, rope_theta=100.0)
    r0 = O.model_step(layers, head["g3"], head["wlm"], cfg, x, lab, P=1)
    assert abs(r1.loss - r2.loss) <= 1e-12 and abs(r1.loss - r0.loss) > 1e-6  # rope changes the model
    for k in r1.grads:
        assert np.max(np.abs(r1.grads[k] - r2.grads[k])) <= 1e-10, k

    def loss_with(w):
        ls = [dict(l_) for l_ in layers]
        ls[0]["wqkv"] = w
        return O.model_step(ls, head["g3"], head["wlm"], cfg, x, lab, P=1, rope_theta=100.0).loss
    fd = O.finite_diff_grad(loss_with, np.asarray(layers[0]["wqkv"], np.float64))
    assert np.linalg.norm(fd - r1.grads["layers.0.wqkv"]) / np.linalg.norm(fd) < 1e-6


def test_embedding_oracle_properties():
    """embed_bwd is the adjoint of embed_fwd: <embed_fwd(ids, E), dx> == <E, embed_bwd(ids, dx)> (f64 check),
    and ids outside [0, V) are rejected."""
    rng = np.random.default_rng(5)
    V, h, n = 37, 6, 200
    ids = rng.integers(0, V, n)
    E = rng.standard_normal((V, h))
    dx = rng.standard_normal((n, h)).astype(np.float32)
    lhs = float(np.sum(O.embed_fwd(ids, E) * dx))
    rhs = float(np.sum(E * O.embed_bwd(ids, dx, V)))
    assert abs(lhs - rhs) < 1e-4 * max(1.0, abs(lhs))
    with pytest.raises(ValueError):
        O.embed_fwd([0, V], E)
    with pytest.raises(ValueError):
        O.embed_fwd([-1], E)


def test_attention_row_and_column_restrictions_match_full_attention():
    """attention_rows / attention_bwd_rows / attention_bwd_cols (the checkers of the L8 / Q8 rank-shape GPU
    tests) equal the full oracle attention on every sampled row / column, causal and packed."""
    rng = np.random.default_rng(5)
    s, Hq, Hkv, d = 300, 4, 2, 16
    q, k, v, do = (rng.standard_normal((s, h, d)) for h in (Hq, Hkv, Hkv, Hq))
    for starts in (None, O.block_causal_starts(np.concatenate([np.arange(120), np.arange(180)]))):
        o, lse = O.attention_fwd(q, k, v, starts)
        dq, dk, dv = O.attention_bwd(q, k, v, o, lse, do, starts)
        rows = np.array([0, 1, 57, 119, 120, 121, 299])
        orow, lrow = O.attention_rows(q, k, v, rows, starts, key_chunk=64)
        np.testing.assert_allclose(orow, o[rows], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(lrow, lse[:, rows], rtol=1e-12, atol=1e-12)
        dqr = O.attention_bwd_rows(q, k, v, do, rows, orow, lrow, starts, key_chunk=64)
        np.testing.assert_allclose(dqr, dq[rows], rtol=1e-9, atol=1e-11)
        cols = np.array([0, 5, 119, 120, 200, 299])
        D = np.sum(do * o, axis=2)
        dkc, dvc = O.attention_bwd_cols(q, k, v, do, lse, D, cols, starts, row_chunk=64)
        np.testing.assert_allclose(dkc, dk[cols], rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(dvc, dv[cols], rtol=1e-9, atol=1e-11)
