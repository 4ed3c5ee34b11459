"""memest through the C-ABI: the paper's numeric anchors, properties of the
max-seqlen solver, and (GPU) cross-validation of this engine's estimate against its own measured ledger."""
import pytest

import paper_2506_13996_b200 as S

GiB = 2.0 ** 30


def test_fixed_bytes_anchor():
    # PAPER §2.1 "144GiB": 16+64+32+32 GiB needs 8*2^30 params; with 8e9 params the same recipe gives 134.1 GiB
    # (SURVEY.md Appendix B #1 records the discrepancy in the paper's arithmetic).
    f = S.memest_fixed(8 * GiB)
    assert (f["weights_bytes"], f["optimizer_bytes"], f["master_weights_bytes"], f["grads_bytes"]) == (
        16 * GiB, 64 * GiB, 32 * GiB, 32 * GiB)
    assert f["total_bytes"] == 144 * GiB
    assert abs(S.memest_fixed(8e9)["total_bytes"] / GiB - 134.1) < 0.05
    assert S.memest_fixed(1)["total_bytes"] == 18
    # 70B, 8 GPUs, ZeRO-3 + optimizer offload fits an 80 GiB GPU (PAPER §5.3.2)
    assert S.memest_fixed(70e9, 8, zero3=True, offload_optimizer=True)["device_bytes_per_gpu"] < 80 * GiB


def test_paper_anchors():
    assert abs(S.memest_logits(16000, 128256, 4) / GiB - 7.65) < 0.01                       # PAPER §3.1
    assert abs(S.memest_activation_ckpt(125000, 4096, 32, 2, 1)[0] / GiB - 30.5) < 0.05      # §3.3
    assert abs(S.memest_activation_ckpt(3_000_000, 8192, 80, 2, 32, 8)[1] / GiB - 915) < 1   # §3.3 70B
    assert abs(S.memest_activation_ckpt(1_000_000, 5120, 64, 2, 32, 8)[1] / GiB - 152) < 1   # §5.3.3
    assert abs(S.memest_4d_mask(125000) / GiB - 29) < 0.2                                   # §3.4
    assert abs(S.memest_4d_mask(250000) / GiB - 116) < 0.5
    assert abs(S.memest_position_ids(125000) / 2**20 - 0.2) < 0.05
    assert S.memest_logits(1, 1, 4) == 4 and S.memest_4d_mask(1) == 2


def test_activation_ckpt_linear():
    a = S.memest_activation_ckpt(1000, 64, 4)[0]
    assert S.memest_activation_ckpt(2000, 64, 4)[0] == 2 * a
    assert S.memest_activation_ckpt(1000, 128, 4)[0] == 2 * a
    assert S.memest_activation_ckpt(1000, 64, 8)[0] == 2 * a


def test_max_seqlen_solver_properties():
    cfg = S.memest_engine(S.TINY, n_layers=2, act_bytes_per_token=40_000.0, act_bytes_per_seq_token=100.0)
    budget = 2 * GiB
    n = S.max_seqlen(cfg, budget, granularity=128)
    assert S.memest_engine_bytes(cfg, n) <= budget < S.memest_engine_bytes(cfg, n + 128)
    scan = max(s for s in range(128, n + 128 * 64, 128) if S.memest_engine_bytes(cfg, s) <= budget)  # brute force
    assert scan == n
    assert S.max_seqlen(cfg, 2 * budget) >= n  # monotone in the budget
    with pytest.raises(S.SptError):
        S.max_seqlen(cfg, 1.0)  # below the fixed share: infeasible


@pytest.mark.gpu
def test_engine_estimate_matches_measured_ledger():
    """Calibrate the two per-token coefficients from the ledgers of two engines, then the estimate must equal
    the ledger of a third configuration (the formulas are exact for this engine)."""
    shape = S.ModelShape(256, 4, 2, 128, 512, 2048)

    def ledger(N, P):
        g = S.ProcessGroup.loopback_group(P)
        e = S.UlyssesLayerStep(shape, N, g)
        led = e.memory()["ledger"]["device"]["peak_bytes"]
        e.close()
        g.close()
        return led

    base = S.memest_engine(shape)
    fixed = S.memest_engine_bytes(base, 0)  # weights + grads (+ tile-dependent workspace below)
    # two SP=1 points give the per-token coefficient (local == global tokens at SP=1)
    n1, n2 = 2048, 4096
    l1, l2 = ledger(n1, 1), ledger(n2, 1)
    ws1 = S.memest_engine_bytes(base, n1) - fixed
    ws2 = S.memest_engine_bytes(base, n2) - fixed
    per_tok = ((l2 - ws2) - (l1 - ws1)) / (n2 - n1)
    cfg = S.memest_engine(shape, act_bytes_per_token=per_tok)
    off = l1 - S.memest_engine_bytes(cfg, n1)  # constant term (scalars, tables, rounding to 256 B)
    for N in (8192, 16384):
        est = S.memest_engine_bytes(cfg, N) + off
        assert abs(est - ledger(N, 1)) / ledger(N, 1) < 1e-3, N


def test_engine_model_fixed_workspaces():
    """The engine model's sequence-independent terms: weights + grads at s = 0; above that the logits tile and
    TiledMLP tile workspaces (the engine's own tile rules: 4 GiB of logits, 2 GiB of MLP intermediates) and the
    per-token activations.  Once the local sequence exceeds one MLP tile the MLP workspace stops growing."""
    shp = S.LLAMA8B
    cfg = S.memest_engine(shp)  # no per-token activations: only the fixed and tile terms
    L = S.lib()
    base = S.memest_engine_bytes(cfg, 0)
    for n, mlp_tile, loss_tile in ((8192, 8192, 8192), (32768, 16384, 8192), (65536, 16384, 8192)):
        want = L.spt_flce_workspace(loss_tile, shp.vocab) + L.spt_mlp_workspace(mlp_tile, shp.intermediate)
        assert S.memest_engine_bytes(cfg, n) - base == want, n
