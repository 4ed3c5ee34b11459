"""Config F (BASELINE.json configs[3]): tiled fused logits + cross-entropy fwd+bwd sweep on one B200.

vocab 128256, hidden 4096, N in {64K .. 1M} tokens x token-tile sizes, through the C-ABI `spt_flce`
(SPEC.md:405-413 tiled_logits_loss).  Per point: device time (CUDA events on the launch stream, 1 warm-up +
2 timed calls), tokens/s, model TFLOP/s (6*N*h*V: logits + dx + dW GEMMs; the CE pass is HBM-bound),
workspace bytes (independent of N: [tile, V] fp32 logits + bf16 dlogits) and total device bytes.

Correctness at full size (size-independent properties):
  * device error flag stays 0 and the loss per token is finite;
  * tiling invariance: for a fixed N, dx is bit-identical for every tile size (each row's dlogits and its
    K=V reduction do not depend on the tiling) and the loss agrees to 1e-5 relative;
  * a 512-token slice is checked against a torch fp32 reference of the same op (loss rel <= 1e-4,
    dx / dW norm-wise rel <= 2e-2).

  python tools/flce_sweep.py [--n 65536,131072,...] [--tiles 1024,2048,4096,8192] [--out file.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_13996_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="65536,131072,262144,524288,1048576")
ap.add_argument("--tiles", default="1024,2048,4096,8192")
ap.add_argument("--hidden", type=int, default=4096)
ap.add_argument("--vocab", type=int, default=128256)
ap.add_argument("--out", default="")
a = ap.parse_args()
L = S.lib()
h, V = a.hidden, a.vocab
Ns = [int(x) for x in a.n.split(",")]
tiles = [int(x) for x in a.tiles.split(",")]
g = torch.Generator(device="cuda").manual_seed(2506_13996)
W = (0.02 * torch.randn(V, h, device="cuda", generator=g)).bfloat16()
dW = torch.empty(V, h, device="cuda")
scale = torch.empty(1, device="cuda")
loss = torch.zeros(1, dtype=torch.float64, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
ws_max = torch.empty(L.spt_flce_workspace(max(tiles), V), dtype=torch.uint8, device="cuda")


def run(x, lab, dx, n, tile):
    loss.zero_()
    S.check(L.spt_flce(x.data_ptr(), W.data_ptr(), lab.data_ptr(), n, h, V, tile, scale.data_ptr(), loss.data_ptr(),
                       dx.data_ptr(), dW.data_ptr(), 0, err.data_ptr(), ws_max.data_ptr(), None))


# ---- torch fp32 reference on a 512-token slice (same bf16 inputs)
n0 = 512
x0 = torch.randn(n0, h, device="cuda", generator=g).bfloat16()
lab0 = torch.randint(0, V, (n0,), device="cuda", generator=g)
lab0[::17] = -100
cnt0 = int((lab0 != -100).sum())
scale.fill_(1.0 / cnt0)
dx0 = torch.empty(n0, h, device="cuda", dtype=torch.bfloat16)
run(x0, lab0, dx0, n0, 256)
torch.cuda.synchronize()
xr = x0.float().requires_grad_(True)
Wr = W.float().requires_grad_(True)
lr = torch.nn.functional.cross_entropy(xr @ Wr.t(), lab0, ignore_index=-100, reduction="sum")
(lr / cnt0).backward()
ref = {
    "loss_rel": abs(float(loss) - float(lr)) / abs(float(lr)),
    "dx_rel": float((dx0.float() - xr.grad).norm() / xr.grad.norm()),
    "dW_rel": float((dW - Wr.grad).norm() / Wr.grad.norm()),
}
assert int(err) == 0 and ref["loss_rel"] <= 1e-4 and ref["dx_rel"] <= 2e-2 and ref["dW_rel"] <= 2e-2, ref
print(json.dumps({"check": "512-token slice vs torch fp32", **ref}), flush=True)
del xr, Wr, lr

points = []
for n in Ns:
    x = torch.randn(n, h, device="cuda", generator=g).bfloat16()
    lab = torch.randint(0, V, (n,), device="cuda", generator=g)
    lab[torch.rand(n, device="cuda", generator=g) < 0.05] = -100
    lab[-1] = -100
    cnt = int((lab != -100).sum())
    scale.fill_(1.0 / cnt)
    dx = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
    dx_ref_sum, loss_ref = None, None
    for tile in tiles:
        run(x, lab, dx, n, tile)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 2
        e0.record()
        for _ in range(reps):
            run(x, lab, dx, n, tile)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        lv = float(loss) / cnt
        assert int(err) == 0 and lv == lv, (n, tile, lv)
        dsum = int(dx.view(torch.int16).to(torch.int64).sum())  # bit-pattern checksum of dx
        if dx_ref_sum is None:
            dx_ref_sum, loss_ref = dsum, lv
        pt = {
            "n": n, "tile": tile, "ms": round(ms, 3), "tokens_per_s": round(n / ms * 1e3, 1),
            "model_tflops": round(6.0 * n * h * V / ms / 1e9, 1),
            "workspace_bytes": int(L.spt_flce_workspace(tile, V)),
            "device_bytes": int(L.spt_flce_workspace(tile, V)) + 2 * n * h * 2 + V * h * 6 + n * 8,
            "loss_per_token": round(lv, 6),
            "dx_bitexact_vs_first_tile": dsum == dx_ref_sum,
            "loss_rel_vs_first_tile": abs(lv - loss_ref) / abs(loss_ref),
        }
        assert pt["dx_bitexact_vs_first_tile"] and pt["loss_rel_vs_first_tile"] < 1e-5, pt
        points.append(pt)
        print(json.dumps(pt), flush=True)
    del x, lab, dx
    torch.cuda.empty_cache()
best = {}
for p in points:
    if p["n"] not in best or p["ms"] < best[p["n"]]["ms"]:
        best[p["n"]] = p
summary = {"config": f"F: tiled logits+CE fwd+bwd, h={h}, V={V}, 1xB200", "reference_check": ref,
           "best_tile_per_n": {str(k): {"tile": v["tile"], "tokens_per_s": v["tokens_per_s"],
                                        "model_tflops": v["model_tflops"]} for k, v in best.items()},
           "points": points}
print(json.dumps({k: v for k, v in summary.items() if k != "points"}), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
