"""Helpers shared by the GPU parity tests (torch is plumbing only: device memory + streams)."""
import numpy as np

from oracle import sptrain_oracle as O


def torch():
    import torch as T

    return T


def bf16_dev(a_f32):
    """float32 numpy (already bf16-representable or not) -> cuda bf16 tensor with RNE rounding."""
    T = torch()
    bits = O.f32_to_bf16_bits(np.asarray(a_f32, dtype=np.float32))
    return T.from_numpy(bits.view(np.int16).copy()).view(T.bfloat16).cuda()


def to_np(t):
    T = torch()
    if t.dtype == T.bfloat16:
        return t.float().cpu().numpy()
    return t.cpu().numpy()


def rel_err(a, b):
    """Norm-wise relative error ||a-b|| / ||b|| (the tolerance contract, SURVEY.md §7 hard part 4)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def record(name, **vals):
    """Append measured parity numbers to $SPT_PARITY_LOG (JSON lines) when set: the margins behind a pass."""
    import json
    import os

    path = os.environ.get("SPT_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **{k: float(v) for k, v in vals.items()}}) + "\n")
