"""Subprocess body for test_attention_bwd_fused_scheme (the backward scheme is chosen once per process from
SPT_ATTN_BWD): runs the tcgen05 backward on one case, checks it against the oracle and for bitwise
determinism, prints 'ok <dq err> <dk err> <dv err>'."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tests.test_gpu_kernels import _attn_case  # noqa: E402
from tests.gpu_util import bf16_dev, rel_err, to_np, torch  # noqa: E402
from oracle import sptrain_oracle as O  # noqa: E402
import paper_2506_13996_b200 as S  # noqa: E402

s, hq, hkv, packed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1"
d = 128
T = torch()
L = S.lib()
qkv, dout, starts = _attn_case(s, hq, hkv, d, packed, s + 7, 1)
q, k, v = qkv[:, :hq], qkv[:, hq:hq + hkv], qkv[:, hq + hkv:]
o_r, lse_r = O.attention_fwd(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), starts)
qkvd, doutd = bf16_dev(qkv), bf16_dev(dout)
o = T.empty(s, hq, d, dtype=T.bfloat16, device="cuda")
lse = T.empty(hq, s, device="cuda")
seg = T.from_numpy(starts.astype(np.int32)).cuda() if starts is not None else None
sc = 1.0 / math.sqrt(d)
S.check(L.spt_attn_fwd(qkvd.data_ptr(), s, hq, hkv, d, S.ptr(seg), sc, o.data_ptr(), lse.data_ptr(), None))
dq_r, dk_r, dv_r = O.attention_bwd(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64),
                                   to_np(o).astype(np.float64), lse_r, dout.astype(np.float64), starts)
ws = T.empty(L.spt_attn_bwd_workspace(s, hq, hkv, d), dtype=T.uint8, device="cuda")
outs = []
for _ in range(2):
    g = T.zeros(s, hq + 2 * hkv, d, dtype=T.bfloat16, device="cuda")
    S.check(L.spt_attn_bwd(qkvd.data_ptr(), o.data_ptr(), lse.data_ptr(), doutd.data_ptr(), s, hq, hkv, d, S.ptr(seg),
                           sc, g.data_ptr(), ws.data_ptr(), None))
    T.cuda.synchronize()
    outs.append(g)
g = to_np(outs[0])
e = (rel_err(g[:, :hq], dq_r), rel_err(g[:, hq:hq + hkv], dk_r), rel_err(g[:, hq + hkv:], dv_r))
assert max(e) < 2e-2, e
assert T.equal(outs[0].view(T.int16), outs[1].view(T.int16)), "fused backward not bitwise deterministic"
print("ok", *[f"{x:.2e}" for x in e])
