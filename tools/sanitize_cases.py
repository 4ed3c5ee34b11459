"""Small layer steps for compute-sanitizer (memcheck / racecheck / synccheck): the smoke step (head_dim 128,
SP=2) plus packed SP=2 steps at head_dim 64 and 32, each checked against the oracle.
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import __graft_entry__ as G  # noqa: E402
import paper_2506_13996_b200 as S  # noqa: E402
from oracle import sptrain_oracle as O  # noqa: E402

G.smoke()
for d, hq, hkv in ((64, 4, 2), (32, 8, 2)):
    cfg = O.LayerConfig(hidden=256, q_heads=hq, kv_heads=hkv, head_dim=d, intermediate=512, vocab=2048)
    N = 512
    params = O.synth_params(cfg, 1)
    x, lab, pos = O.synth_batch(cfg, N, 1, packed=True)
    grp = S.ProcessGroup.loopback_group(2, 0)
    eng = S.UlyssesLayerStep(S.ModelShape(256, hq, hkv, d, 512, 2048), N, grp, packed=pos is not None)
    for k in O.LayerParams.NAMES:
        eng.set_param(k, O.f32_to_bf16_bits(params[k]))
    loss, cnt = eng.step(O.f32_to_bf16_bits(x), lab, pos)
    eng.close()
    grp.close()
    ref = O.layer_step(O.LayerParams(**params), cfg, x, lab, pos, P=1)
    assert cnt == ref.count and abs(loss - ref.loss) / abs(ref.loss) < 1e-3, (loss, ref.loss)
    print(f"d={d}: loss {loss:.6f} oracle {ref.loss:.6f}")
print("sanitize cases ok")
