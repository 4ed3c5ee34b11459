#!/usr/bin/env python
"""Benchmark: fwd+bwd tokens/s of one Llama-3-8B-shaped decoder layer + lm_head with Ulysses SP.

Default (N=1): BASELINE.json configs[1] — h 4096, 32 q / 8 kv heads (d 128), I 14336, V 128256,
seq 32768 on 1 B200.  N>1 (torchrun, one process per GPU, NCCL over NVLink): weak scaling, 32768
tokens per GPU, Ulysses SP=N over the whole sequence.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--seq-per-gpu S] [--impl ours|reference]

`--impl reference` times the CPU port of the reference algorithm (oracle/, float32 numpy/OpenBLAS on
all host cores) on a bounded token sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd tokens/s, Llama-8B-shape layer, 1/2/4/8-GPU Ulysses; peak HBM bytes"
SHAPE = dict(hidden=4096, q_heads=32, kv_heads=8, head_dim=128, intermediate=14336, vocab=128256)
CPU_SAMPLE_TOKENS = 256


def workload_name(seq, n, layers=1, offload=False):
    stack = "layer" if layers == 1 and not offload else (
        f"{layers}-layer stack (activation checkpoints {'offloaded to host' if offload else 'on device'})")
    return (f"llama3-8b-shape {stack} + lm_head (h4096, 32q/8kv d128, I14336, V128256), "
            f"seq {seq} over {n} GPU(s), Ulysses SP={n}, TiledMLP + tiled logits/CE")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------------------- CPU reference arm
_CPU_CACHE = {}


def cpu_layer_sample(n_tokens: int, seed: int = 0):
    """One oracle layer step (fwd+bwd) on an n_tokens sample of the workload; returns (seconds, loss)."""
    import numpy as np

    from oracle import sptrain_oracle as O

    cfg = O.LLAMA8B
    key = (n_tokens, seed)
    if key not in _CPU_CACHE:  # synthetic weights/batch are set-up, not part of the timed step
        p = O.LayerParams(**O.synth_params(cfg, seed)).astype(np.float32)
        _CPU_CACHE[key] = (p, O.synth_batch(cfg, n_tokens, seed))
    p, (x, lab, pos) = _CPU_CACHE[key]
    t0 = time.perf_counter()
    res = O.layer_step(p, cfg, x.astype(np.float32), lab, None, P=1, dtype=np.float32)
    return time.perf_counter() - t0, res.loss


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = CPU_SAMPLE_TOKENS
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_layer_sample(n)
    times = [cpu_layer_sample(n)[0] for _ in range(args.steps)]
    tot = sum(times)
    v = n * len(times) / tot
    seq = args.seq_per_gpu * world
    line = {
        "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * tot / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": workload_name(seq, world), "seq_len": seq, "sp_degree": world},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"{n}-token sample of the workload per step (oracle/sptrain_oracle.py "
                                   f"layer_step, float32 numpy/OpenBLAS, SP=1)"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for ln in (self.out or "").strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), float(f[2]), f[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        load = [r for r in rows if r[2] >= 50] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(load)}


# ------------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2506_13996_b200 as S

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist

        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(S.ProcessGroup.unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        grp = S.ProcessGroup.nccl_group(bytes(uid.cpu().numpy().tobytes()), world, rank, local_rank)
    else:
        grp = S.ProcessGroup.loopback_group(1, local_rank)
    seq = args.seq_per_gpu * world
    n_loc = args.seq_per_gpu
    shp = S.ModelShape(**SHAPE)
    eng = S.UlyssesLayerStep(shp, seq, grp, lr=args.lr, n_layers=args.layers, ckpt_offload=args.offload,
                             rope_theta=args.rope)
    # random-init weights of the architecture, identical on every rank (same seed)
    g = torch.Generator(device=dev).manual_seed(1234)
    qkv_out = (shp.q_heads + 2 * shp.kv_heads) * shp.head_dim
    wshapes = {"g1": (shp.hidden,), "wqkv": (qkv_out, shp.hidden), "wo": (shp.hidden, shp.q_heads * shp.head_dim),
               "g2": (shp.hidden,), "wg": (shp.intermediate, shp.hidden), "wu": (shp.intermediate, shp.hidden),
               "wd": (shp.hidden, shp.intermediate), "g3": (shp.hidden,), "wlm": (shp.vocab, shp.hidden)}
    names = [(k, s_) for k, s_ in wshapes.items() if k in ("g3", "wlm")]
    for i in range(args.layers):
        names += [(f"layers.{i}.{k}", s_) for k, s_ in wshapes.items() if k not in ("g3", "wlm")]
    for k, s_ in names:
        if k.split(".")[-1].startswith("g"):
            w = (1.0 + 0.05 * torch.randn(s_, device=dev, generator=g)).bfloat16()
        else:
            w = (0.02 * torch.randn(s_, device=dev, generator=g)).bfloat16()
        eng.set_param(k, w, on_host=False)
        del w
    # synthetic inputs for this rank's sequence shard (resident in HBM for the device-timed loop)
    gi = torch.Generator(device=dev).manual_seed(99 + rank)
    x = torch.randn(n_loc, shp.hidden, device=dev, generator=gi).bfloat16()
    lab = torch.randint(0, shp.vocab, (n_loc,), device=dev, generator=gi, dtype=torch.int64)
    lab[torch.rand(n_loc, device=dev, generator=gi) < 0.05] = -100
    if rank == world - 1:
        lab[-1] = -100  # pre-shifted labels end with -100
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            import torch.distributed as dist

            dist.barrier(device_ids=[local_rank])
            torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        eng.step_async(x, lab, None, on_host=False, stream=sp)
    loss0, cnt = eng.read_loss(stream=sp)
    eng.set_profiling(True)
    barrier()
    n0 = S.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof_acc = {}
    sites_acc = {}
    with Clocks(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            eng.step_async(x, lab, None, on_host=False, stream=sp)
            t = eng.timing()  # syncs on the step's end event only after it is recorded: accumulate per step
            for site, v in t["classes"].get("sites", {}).items():
                a = sites_acc.setdefault(site, {"ms": 0.0, "calls": 0})
                a["ms"] += v["ms"]
                a["calls"] += v["calls"]
                a["tflops"] = v["tflops"]
            for c, v in t["classes"].items():
                if c == "sites":
                    continue
                a = prof_acc.setdefault(c, {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0})
                for kk in a:
                    a[kk] += v[kk]
        ev1.record(stream)
        barrier()
    launches = S.kernel_launch_count() - n0
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_eager = ms
    loss, cnt = eng.read_loss(stream=sp)
    eng.set_profiling(False)
    # ---- the same step replayed as one CUDA graph (device-resident inputs at fixed addresses, 1 GPU): this is
    # the timed `value` when the capture succeeds; the profiled eager loop above supplies the breakdown
    graph_used = False
    if args.graph and world == 1:
        try:
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(stream)
            eng.graph_capture(x, lab, None, stream=gs.cuda_stream)
            for _ in range(2):
                eng.graph_launch(stream=gs.cuda_stream)
            gs.synchronize()
            barrier()
            n0 = S.kernel_launch_count()
            with Clocks(local_rank) as clk:
                ev0.record(gs)
                for _ in range(args.steps):
                    eng.graph_launch(stream=gs.cuda_stream)
                ev1.record(gs)
                gs.synchronize()
                barrier()
            launches = S.kernel_launch_count() - n0
            ms = ev0.elapsed_time(ev1) / args.steps
            loss, cnt = eng.read_loss(stream=gs.cuda_stream)
            graph_used = True
        except S.SptError as e:  # eager timing stands; the reason goes into the JSON line
            graph_used = f"capture failed: {e}"
    # max over ranks
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # ---- end-to-end through the public API with host buffers (H2D inputs, D2H loss every step)
    xh = x.cpu().pin_memory()
    labh = lab.cpu().pin_memory()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):  # H2D of every step's inputs + D2H of every step's loss, pipelined
        eng.step_async(xh, labh, None, on_host=True, stream=sp)
        eng.loss_async(i % 64, stream=sp)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    e2e_losses = [eng.loss_slot(i % 64)[0] for i in range(min(args.steps, 64))]
    assert all(math.isfinite(v) for v in e2e_losses), e2e_losses
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    mem = eng.memory()
    if rank != 0:
        eng.close()
        grp.close()
        return
    pk, pk_kind = peaks()
    led = mem["ledger"]
    peak_b = led["device"]["peak_bytes"]
    # roofline for the dominant kernel class (per launch averages over the timed region)
    cls = max(prof_acc.items(), key=lambda kv: kv[1]["ms"])
    name, c = cls
    if c["flops"] > 0:
        achieved = c["flops"] / (c["ms"] / 1e3) / 1e12
        peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        roof = {"kernel": name, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None, "peak_kind": f"{pk_kind} sustained bf16",
                "flops_per_launch": c["flops"] / max(1, c["launches"]), "avg_launch_ms": c["ms"] / max(1, c["launches"])}
    else:
        achieved = c["bytes"] / (c["ms"] / 1e3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None, "peak_kind": f"{pk_kind} hbm copy"}
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            tr = json.load(open(prof_path))
            roof["traffic"] = tr.get(name)
        except Exception:
            pass
    step_s = ms / 1e3
    tokens = seq  # whole-job tokens per step (all ranks)
    breakdown = {k: round(v["ms"] / args.steps, 3) for k, v in prof_acc.items() if v["ms"] > 0}
    tflops = {k: round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1) for k, v in prof_acc.items() if v["ms"] > 0 and v["flops"]}
    cpu_v = None
    if world == 1 and not args.no_cpu_baseline:
        n = CPU_SAMPLE_TOKENS
        cpu_layer_sample(n)
        ts = [cpu_layer_sample(n)[0] for _ in range(2)]
        cpu_v = {"value": n * len(ts) / sum(ts), "unit": "tokens/s", "cores": os.cpu_count() or 1, "kind": "port",
                 "sample": f"{n}-token sample of the workload (oracle layer_step, float32 numpy/OpenBLAS, SP=1), "
                           f"2 steps"}
    fixed = led["device"]["tags"]["weights"]["peak"] + led["device"]["tags"]["grads"]["peak"]
    per_tok = (peak_b - fixed) / n_loc
    free_total = mem["ledger"].get("cuda_mem_total_bytes", 0)
    est_max = int((0.95 * free_total - fixed) / per_tok) if free_total else None
    line = {
        "metric": METRIC, "value": tokens / step_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, N(0,1) hidden, uniform labels)",
        "config": {"workload": workload_name(seq, world, args.layers, args.offload), "seq_len": seq, "tokens_per_gpu": n_loc,
                   "sp_degree": world, "mlp_tile": mem["mlp_tile"], "loss_tile": mem["loss_tile"],
                   "l2": "inputs larger than L2 (x 256 MiB/GPU, weights 1.5 GiB, activations ~3 GiB per step)",
                   "optimizer": f"sgd lr={args.lr}" if args.lr > 0 else "none (fwd+bwd+SP grad all-reduce)",
                   "n_layers": args.layers, "rope_theta": args.rope,
                   "activation_checkpointing": ("offload to pinned host" if args.offload else
                                                ("device" if args.layers > 1 else "none (single layer)"))},
        "peak_hbm_bytes": peak_b, "peak_hbm_bytes_per_token": peak_b / n_loc,
        "est_max_seq_per_gpu": est_max,
        "loss": loss, "valid_tokens": cnt,
        "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(x.numel() * 2 + lab.numel() * 8), "d2h_bytes_per_step": 32},
        "gpu_launches": launches,
        "cuda_graph": graph_used, "ms_per_step_eager_profiled": ms_eager,
        "roofline": roof,
        "breakdown_ms_per_step": breakdown, "class_tflops": tflops,
        "gemm_sites": {k: {"ms_per_step": round(v["ms"] / args.steps, 3), "tflops": round(v["tflops"], 1)}
                       for k, v in sorted(sites_acc.items(), key=lambda kv: -kv[1]["ms"])},
        "clocks": clk.summary(),
        "cpu_baseline": cpu_v,
    }
    print(json.dumps(line), flush=True)
    eng.close()
    grp.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seq-per-gpu", type=int, default=32768)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lr", type=float, default=0.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layers", type=int, default=1,
                    help="decoder layers (> 1: per-layer activation checkpointing; not the BASELINE config)")
    ap.add_argument("--offload", action="store_true", help="activation checkpoints in pinned host memory")
    ap.add_argument("--rope", type=float, default=0.0, help="RoPE theta (> 0 turns it on; not the BASELINE config)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time `value` with eager launches instead of a CUDA-graph replay of the step")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
