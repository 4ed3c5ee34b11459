"""The layer step across real GPUs, one process per GPU (pytest -m gpu; skipped below 2 GPUs).

world = min(device_count, 8) processes, rank r on cuda:r, over both transports:
  * peer: the fused K1 pack-and-store / K2 load-and-unpack all-to-alls and the fixed-order all-reduces over
    NVLink peer mappings (CUDA IPC across devices);
  * nccl: grouped ncclSend / ncclRecv all-to-alls between staging buffers and ncclAllReduce / ncclAllGather
     — the multi-rank NCCL path the one-GPU box cannot run ("Duplicate GPU detected").
Both are compared with the loopback group at the same P (P virtual ranks in one process, pinned to
the oracle by the layer tests): count and dx bitwise (the reshard is a bit-exact permutation and dx depends on the
loss only through the integer count), the loss bitwise on the peer transport (rank-ascending fp64 sum) and to
1e-6 relative on NCCL (its fp64 reduction order is the library's; the loss is returned in fp32), weight grads to 1e-6 (per-tile fp32 partial sums
associate differently across ranks).  The config exercises kv replication once P > Hkv (Hq = 8, Hkv = 2)."""
import numpy as np
import pytest
import torch

from oracle import sptrain_oracle as O
from tests import peer_worker as W
from tests.gpu_util import rel_err
from tests.test_gpu_peer import _loopback, _spawn

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(NGPU < 2, reason=f"needs >= 2 GPUs (found {NGPU})")]

CFG = dict(hidden=256, q_heads=8, kv_heads=2, head_dim=128, intermediate=512, vocab=2048)


@pytest.mark.parametrize("transport", ["peer", "nccl"])
@pytest.mark.parametrize("packed", [False, True])
def test_layer_step_across_gpus_matches_loopback(transport, packed, tmp_path):
    world = 1 << (min(NGPU, 8).bit_length() - 1)  # 2, 4 or 8 (Hq = 8 must split evenly)
    N = 256 * world
    ranks = _spawn(W.engine_case, world, tmp_path, CFG, N, 11, packed, 0.0, transport == "peer", transport, True)
    ref = _loopback(O.LayerConfig(**CFG), N, world, 11, packed, 0.0)
    n_loc = N // world
    for r, out in enumerate(ranks):
        assert int(out["count"]) == ref["count"], r
        if transport == "peer":
            assert float(out["loss"]) == ref["loss"], (r, float(out["loss"]), ref["loss"])
        else:
            assert abs(float(out["loss"]) - ref["loss"]) <= 1e-6 * abs(ref["loss"]), (r, float(out["loss"]))
        assert np.array_equal(out["dx"], ref["dx"][r * n_loc:(r + 1) * n_loc]), r
        for k in O.LayerParams.NAMES:
            g, gr = out["g_" + k], ref["grads"][k]
            assert np.array_equal(g, gr) or rel_err(g, gr) <= 1e-6, (r, k, rel_err(g, gr))
        if transport == "peer":
            assert float(out["graph_loss"]) == ref["loss"]
            assert np.array_equal(out["graph_dx"], out["dx"])
