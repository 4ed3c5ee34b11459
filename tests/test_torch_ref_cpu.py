"""Pin the full-size torch fp32 checker (tests/torch_ref.py) to the numpy oracle before trusting it."""
import numpy as np
import pytest
import torch

from oracle import sptrain_oracle as O
from tests import torch_ref as R


@pytest.mark.parametrize("packed,chunks", [(False, (64, 100)), (True, (32, 77)), (False, (512, 512))])
def test_torch_ref_matches_oracle(packed, chunks):
    cfg = O.LayerConfig(hidden=64, q_heads=4, kv_heads=2, head_dim=16, intermediate=96, vocab=300)
    N = 256
    params = O.synth_params(cfg, 5)
    x, lab, pos = O.synth_batch(cfg, N, 5, packed=packed)
    ref = O.layer_step(O.LayerParams(**params), cfg, x, lab, pos if packed else None)
    tp = {k: torch.from_numpy(np.asarray(v, np.float64)) for k, v in params.items()}
    loss, cnt, grads, dx = R.layer_step(tp, torch.from_numpy(x.astype(np.float64)), torch.from_numpy(lab),
                                        torch.from_numpy(pos) if packed else None, cfg.q_heads, cfg.kv_heads,
                                        cfg.head_dim, attn_chunk=chunks[0], loss_chunk=chunks[1])
    assert cnt == ref.count
    assert abs(loss - ref.loss) <= 1e-12 * abs(ref.loss)
    for k in O.LayerParams.NAMES:
        np.testing.assert_allclose(grads[k].numpy(), ref.grads[k], rtol=1e-9, atol=1e-12, err_msg=k)
    np.testing.assert_allclose(dx.numpy(), ref.dx, rtol=1e-9, atol=1e-12)
