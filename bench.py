#!/usr/bin/env python
"""Benchmark: fwd+bwd tokens/s of one Llama-3-8B-shaped decoder layer + lm_head with Ulysses SP.

Default (N=1): BASELINE.json configs[1] (L1) — h 4096, 32 q / 8 kv heads (d 128), I 14336, V 128256,
seq 32768 on 1 B200.  N>1: one process per GPU (torchrun; `--gpus N` without torchrun re-launches itself
under torch.distributed.run), Ulysses SP=N over the whole sequence: 32768 tokens per GPU at N=2/4 and
BASELINE configs[2] (L8: 524288 tokens, 65536 per GPU) at N=8.  The SP exchange runs on the peer-memory
transport (fused pack-store / load-unpack all-to-alls over NVLink, `--comm peer`, default) or NCCL
(`--comm nccl`, the library baseline).  `--workload tiny` runs BASELINE configs[0] (h 256, 8q/2kv d32,
V 32000, seq 8192) instead; `--workload qwen` BASELINE configs[4]'s layer shape (Qwen2.5-32B, 32K tokens per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--seq S] [--impl ours|reference] [--comm peer|nccl]

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
SHAPES = {
    "l1": dict(hidden=4096, q_heads=32, kv_heads=8, head_dim=128, intermediate=14336, vocab=128256),
    "tiny": dict(hidden=256, q_heads=8, kv_heads=2, head_dim=32, intermediate=1024, vocab=32000),
    # BASELINE configs[4]'s layer shape (Qwen2.5-32B: 64q/8kv, h=5120 != Hq*d, I=25600, V=151936); configs[4] itself
    # is SP=8 at 1M tokens on 8 GPUs, so one GPU runs it at 32K tokens (and at N>1 with 32K tokens per GPU)
    "qwen": dict(hidden=5120, q_heads=64, kv_heads=8, head_dim=128, intermediate=25600, vocab=151936),
}
SHAPE = SHAPES["l1"]
CPU_SAMPLE_TOKENS = 512
NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (spec)


def default_seq(workload, n):
    """L1 (N=1, 32768), weak scaling at 32768 tokens per GPU for N=2/4, the L8 config at N=8 (524288)."""
    if workload == "tiny":
        return 8192 * n
    if workload == "qwen":
        return 32768 * n
    return 524288 if n == 8 else 32768 * n


def workload_name(seq, n, layers=1, offload=False, workload="l1"):
    stack = "layer" if layers == 1 and not offload else (
        f"{layers}-layer stack (activation checkpoints {'offloaded to host' if offload else 'on device'})")
    if workload == "qwen":
        return (f"qwen2.5-32b-shape {stack} + lm_head (h5120, 64q/8kv d128, I25600, V151936; BASELINE configs[4]'s "
                f"layer), seq {seq} over {n} GPU(s), Ulysses SP={n}, TiledMLP + tiled logits/CE")
    if workload == "tiny":
        return (f"tiny llama-shape {stack} + lm_head (h256, 8q/2kv d32, I1024, V32000; BASELINE configs[0]), "
                f"seq {seq} over {n} GPU(s), Ulysses SP={n}, TiledMLP + tiled logits/CE")
    return (f"llama3-8b-shape {stack} + lm_head (h4096, 32q/8kv d128, I14336, V128256), "
            f"seq {seq} over {n} GPU(s), Ulysses SP={n}, TiledMLP + tiled logits/CE")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------------------- CPU reference arm
_CPU_CACHE = {}


def cpu_sample_tokens(args):
    """Tokens per CPU step: 512 of the L1 workload (each with its full causal attention context, below), the
    whole configs[0] sequence (8192) for --workload tiny."""
    return args.cpu_tokens or (8192 if args.workload == "tiny" else CPU_SAMPLE_TOKENS)


def cpu_layer_sample(n_tokens: int, seed: int = 0, workload: str = "l1", seq: int = 0, sp: int = 1):
    """One CPU step of the reference algorithm (oracle/sptrain_oracle.py, float32) on an n-token sample of the
    workload; returns (seconds, loss).

    The step is the oracle's layer_step (fwd+bwd: projections, attention, TiledMLP, tiled logits/CE, RMSNorms) on
    n tokens.  Every op but attention is token-local, so its per-token cost is the workload's.  Attention is not:
    in a seq-token sequence a token attends to its whole causal prefix.  When seq > n the step therefore also
    runs the attention of n query rows spread evenly over the seq-token sequence (mean context seq/2) against
    their full prefix: forward O / LSE (attention_rows) and dQ (attention_bwd_rows), float32, on synthetic Q/K/V/dO
    of the workload's shape (set up once, outside the timed region), one kv-head group per host thread."""
    import numpy as np

    from oracle import sptrain_oracle as O

    cfg = O.LayerConfig(**SHAPES[workload])
    # synthetic weights / batches are set-up, not part of the timed step
    if ("w", seed, workload) not in _CPU_CACHE:
        _CPU_CACHE[("w", seed, workload)] = O.LayerParams(**O.synth_params(cfg, seed)).astype(np.float32)
    if (n_tokens, seed, workload) not in _CPU_CACHE:
        _CPU_CACHE[(n_tokens, seed, workload)] = O.synth_batch(cfg, n_tokens, seed)
    p = _CPU_CACHE[("w", seed, workload)]
    x, lab, pos = _CPU_CACHE[(n_tokens, seed, workload)]
    attn = None
    if seq > n_tokens:
        akey = ("attn", seq, n_tokens, workload)
        if akey not in _CPU_CACHE:
            rng = np.random.default_rng(seed)
            hq, hkv, d = cfg.q_heads, cfg.kv_heads, cfg.head_dim
            qkv = [rng.standard_normal((seq, h, d), dtype=np.float32) for h in (hq, hkv, hkv, hq)]
            rows = ((np.arange(n_tokens) + 0.5) * (seq / n_tokens)).astype(np.int64)
            _CPU_CACHE[akey] = (qkv, rows)
        attn = _CPU_CACHE[akey]
    t0 = time.perf_counter()
    res = O.layer_step(p, cfg, x.astype(np.float32), lab, None, P=sp, dtype=np.float32)
    if attn is not None:
        (q, k, v, do), rows = attn
        g = cfg.q_heads // cfg.kv_heads

        def kv_group(j):  # one kv head and its q heads; numpy releases the GIL, so groups run on separate cores
            qs, ks = slice(j * g, (j + 1) * g), slice(j, j + 1)
            o, lse = O.attention_rows(q[:, qs], k[:, ks], v[:, ks], rows, dtype=np.float32)
            O.attention_bwd_rows(q[:, qs], k[:, ks], v[:, ks], do[:, qs], rows, o, lse, dtype=np.float32)

        from threadpoolctl import threadpool_limits

        with threadpool_limits(1):  # one BLAS thread per group: the groups already fill the cores
            list(_cpu_pool().map(kv_group, range(cfg.kv_heads)))
    return time.perf_counter() - t0, res.loss


def _cpu_pool():
    import concurrent.futures as cf

    if "pool" not in _CPU_CACHE:
        _CPU_CACHE["pool"] = cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1)
    return _CPU_CACHE["pool"]


def cpu_sample_desc(n, workload, seq):
    if workload != "tiny":
        ctx = (f" plus the attention forward + dQ of {n} query rows spread evenly over the {seq}-token sequence "
               f"against their full causal prefix (mean context {seq // 2}; the dK/dV share of the backward, 2 of "
               f"its 5 products, is not in the sample)") if seq > n else ""
        return (f"{n}-token sample of the workload per step: oracle/sptrain_oracle.py layer_step (float32 "
                f"numpy/OpenBLAS, SP=1){ctx}")
    return f"{n}-token step of configs[0] (oracle/sptrain_oracle.py layer_step, float32 numpy/OpenBLAS, SP=1)"


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = cpu_sample_tokens(args)
    cores = os.cpu_count() or 1
    seq = args.seq or default_seq(args.workload, world)
    for _ in range(args.warmup):
        cpu_layer_sample(n, workload=args.workload, seq=seq)
    times = [cpu_layer_sample(n, workload=args.workload, seq=seq)[0] for _ in range(args.steps)]
    tot = sum(times)
    v = n * len(times) / tot
    line = {
        "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * tot / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": workload_name(seq, world, workload=args.workload), "seq_len": seq,
                   "tokens_per_gpu": seq // world, "sp_degree": world, "cpu_model": cpu_model()},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": cpu_sample_desc(n, args.workload, seq)},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.workload == "tiny":
        # SURVEY.md §8(d) / BASELINE configs[0]: the same step as P in-process SP ranks (the oracle's SPMD form,
        # reshard, kv replication at P = 4 / 8, fixed-order all-reduces), one timed step each
        line["cpu_sp"] = []
        for P in (2, 4, 8):
            t, loss = cpu_layer_sample(n, workload="tiny", sp=P)
            line["cpu_sp"].append({"sp_degree": P, "value": n / t, "unit": "tokens/s", "ms_per_step": 1000.0 * t,
                                   "loss": loss})
    if args.workload == "l1" and args.cpu_reduced_n not in ("0", "", None):
        # the L shape at reduced N (2048 and 4096), measured whole (attention included), one timed
        # step each
        line["cpu_reduced_n"] = []
        for nr in (int(v) for v in str(args.cpu_reduced_n).split(",") if int(v) > 0):
            t, _ = cpu_layer_sample(nr, workload="l1")  # weights / batch set-up happens before the timer starts
            line["cpu_reduced_n"].append({"seq_len": nr, "value": nr / t, "unit": "tokens/s", "ms_per_step": 1000.0 * t,
                                          "note": "whole L-shape layer step at this N (1 timed step), not the L1 workload"})
    print(json.dumps(line), flush=True)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
def make_group(S, args, rank, world, local_rank):
    """Loopback (N=1), the peer-memory transport (default for N>1) or NCCL (--comm nccl)."""
    import torch

    if world == 1:
        return S.ProcessGroup.loopback_group(1, local_rank)
    if args.comm == "peer":
        return S.ProcessGroup.peer_group(world, rank, local_rank)  # IPC handles exchanged over torch.distributed
    import torch.distributed as dist

    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(S.ProcessGroup.unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    return S.ProcessGroup.nccl_group(bytes(uid.numpy().tobytes()), world, rank, local_rank)


def est_max_seq(S, shp, mem, n_loc, world):
    """max_seqlen_solver on this engine's memory model, calibrated from this run's ledger: the
    fixed bytes (weights, grads, logits tile and TiledMLP tile workspaces) are modelled exactly, the rest of the
    measured peak is charged per local token."""
    led = mem["ledger"]["device"]
    tags = led["tags"]
    # the TiledMLP workspace is sized by the MLP tile (fixed by its 2 GiB rule once N exceeds a tile), not by N
    mlp_ws = S.lib().spt_mlp_workspace(mem["mlp_tile"], shp.intermediate)
    fixed = tags["weights"]["peak"] + tags["grads"]["peak"] + tags["logits"]["peak"] + mlp_ws
    # + the caller's own device copy of the step inputs (x bf16 and int64 labels), which the ledger does not see
    per_tok = max(1.0, (led["peak_bytes"] - fixed) / n_loc) + 2 * shp.hidden + 8
    total = mem["ledger"].get("cuda_mem_total_bytes", 0)
    if not total:
        return None, per_tok
    cfg = S.memest_engine(shp, n_layers=1, sp=world, act_bytes_per_token=per_tok)
    budget = total - 3 * (1 << 30)  # CUDA context, allocator slack
    try:
        return S.max_seqlen(cfg, budget, granularity=128 * world), per_tok
    except S.SptError:
        return None, per_tok


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2506_13996_b200 as S

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    grp = make_group(S, args, rank, world, local_rank)
    seq = args.seq or default_seq(args.workload, world)
    assert seq % world == 0, "seq must be divisible by the GPU count"
    n_loc = seq // world
    shp = S.ModelShape(**SHAPES[args.workload])
    eng = S.UlyssesLayerStep(shp, seq, grp, lr=args.lr, n_layers=args.layers, ckpt_offload=args.offload,
                             rope_theta=args.rope, loss_tile=args.loss_tile)
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

            dist.barrier()
            torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist

        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        eng.step_async(x, lab, None, on_host=False, stream=sp)
    eng.read_loss(stream=sp)
    prof_acc, sites_acc = {}, {}

    gaps_last = {}

    def accumulate(t):  # per-kernel-class CUDA-event times of one step (spt_layer_timing_json)
        gaps_last.clear()
        gaps_last.update(t.get("gaps", {}))
        for site, v in t["classes"].get("sites", {}).items():
            a = sites_acc.setdefault(site, {"ms": 0.0, "calls": 0, "bytes": 0.0})
            a["ms"] += v["ms"]
            a["calls"] += v["calls"]
            a["bytes"] += v.get("bytes", 0.0)
            a["tflops"] = v["tflops"]
        for c, v in t["classes"].items():
            if c == "sites":
                continue
            a = prof_acc.setdefault(c, {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0})
            for kk in a:
                a[kk] += v[kk]

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # ---- the timed value: K replays of one CUDA graph of the whole step (device-resident inputs at fixed
    # addresses), the same method at every world size.  The graph is captured with per-kernel-class profiling on:
    # its CUDA events are event-record nodes of the graph, so the roofline and the breakdown are read from the
    # last timed replay itself.  Eager launches (and a separate profiled eager pass) only if the capture fails.
    graph_used = False
    gs = torch.cuda.Stream(dev)
    gs.wait_stream(stream)
    ms_eager = None
    eng.set_profiling(True)
    if args.graph:
        try:
            eng.graph_capture(x, lab, None, stream=gs.cuda_stream)
            for _ in range(2):
                eng.graph_launch(stream=gs.cuda_stream)
            graph_used = True
        except S.SptError as e:
            graph_used = f"capture failed: {e}"
    prof_steps = 1
    if graph_used is not True:  # fallback: profiled eager pass for the breakdown, unprofiled eager timed loop
        barrier()
        prof_steps = max(1, min(args.steps, 3))
        ev0.record(stream)
        for _ in range(prof_steps):
            eng.step_async(x, lab, None, on_host=False, stream=sp)
            accumulate(eng.timing())
        ev1.record(stream)
        barrier()
        ms_eager = max_over_ranks(ev0.elapsed_time(ev1) / prof_steps)
        eng.set_profiling(False)
    barrier()
    n0 = S.kernel_launch_count()
    with Clocks(local_rank) as clk:
        ev0.record(gs)
        for _ in range(args.steps):
            if graph_used is True:
                eng.graph_launch(stream=gs.cuda_stream)
            else:
                eng.step_async(x, lab, None, on_host=False, stream=gs.cuda_stream)
        ev1.record(gs)
        gs.synchronize()
        barrier()
    launches = S.kernel_launch_count() - n0
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    if graph_used is True:
        accumulate(eng.timing())  # the events of the last timed replay
    eng.set_profiling(False)
    loss, cnt = eng.read_loss(stream=gs.cuda_stream)
    # ---- end-to-end through the public API with host buffers (H2D inputs, D2H loss every step)
    xh = x.cpu().pin_memory()
    labh = lab.cpu().pin_memory()
    eng.step_async(xh, labh, None, on_host=True, stream=sp)  # untimed: creates the H2D staging buffers
    eng.read_loss(stream=sp)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):  # H2D of every step's inputs + D2H of every step's loss, pipelined
        eng.step_async(xh, labh, None, on_host=True, stream=sp)
        eng.loss_async(i % 64, stream=sp)
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    e2e_losses = [eng.loss_slot(i % 64)[0] for i in range(min(args.steps, 64))]
    assert all(math.isfinite(v) for v in e2e_losses), e2e_losses
    mem = eng.memory()
    if rank != 0:
        eng.close()
        grp.close()
        return
    pk, pk_kind = peaks()
    led = mem["ledger"]
    peak_b = led["device"]["peak_bytes"]
    # roofline for the dominant kernel class (per-launch averages over the profiled step(s))
    cls = max(((k, v) for k, v in prof_acc.items() if k != "a2a"), key=lambda kv: kv[1]["ms"])
    name, c = cls
    if c["flops"] > 0:
        achieved = c["flops"] / (c["ms"] / 1e3) / 1e12
        peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        roof = {"kernel": name, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None, "peak_kind": f"{pk_kind} sustained bf16",
                "peak_note": "MEASURED_PEAKS.json bf16_tflops_sustained: cuBLAS 8192^3 back to back for 4 s on the pod "
                             "that wrote the file; under the same ~1 kW cap an in-step GEMM class can reach or pass it "
                             f"on a cooler box (burst figure: {pk['bf16_tflops']})",
                "flops_per_launch": c["flops"] / max(1, c["launches"]), "avg_launch_ms": c["ms"] / max(1, c["launches"]),
                # operands read once + outputs written once (csrc/gemm.cu gemm_alg_bytes), the yardstick for traffic
                "algorithmic_bytes_per_launch": c["bytes"] / max(1, c["launches"]) if c["bytes"] else None}
    else:
        achieved = c["bytes"] / (c["ms"] / 1e3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None, "peak_kind": f"{pk_kind} hbm copy"}
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path) and args.workload == "l1":
        try:
            roof["traffic"] = json.load(open(prof_path)).get(name)
            if roof["traffic"] and roof.get("algorithmic_bytes_per_launch"):
                roof["traffic_over_algorithmic"] = roof["traffic"] / roof["algorithmic_bytes_per_launch"]
        except Exception:
            pass
    breakdown = {k: round(v["ms"] / prof_steps, 3) for k, v in prof_acc.items() if v["ms"] > 0}
    tflops = {k: round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1) for k, v in prof_acc.items() if v["ms"] > 0 and v["flops"]}
    # Ulysses all-to-alls (pack / unpack fused in on the peer transport): payload bytes per rank / time
    a2a = {k: {"ms_per_step": round(v["ms"] / prof_steps, 3), "bytes_per_step": v["bytes"] / prof_steps,
               "gbps": round(v["bytes"] / (v["ms"] * 1e6), 1) if v["ms"] > 0 else None,
               "frac_of_nvlink": round(v["bytes"] / (v["ms"] * 1e6) / NVLINK_GBS, 3) if v["ms"] > 0 else None}
           for k, v in sites_acc.items() if k.startswith("a2a_")}
    cpu_v = None
    if world == 1 and not args.no_cpu_baseline:
        n = cpu_sample_tokens(args)
        cpu_layer_sample(n, workload=args.workload, seq=seq)
        ts = [cpu_layer_sample(n, workload=args.workload, seq=seq)[0] for _ in range(2)]
        cpu_v = {"value": n * len(ts) / sum(ts), "unit": "tokens/s", "cores": os.cpu_count() or 1, "kind": "port",
                 "sample": cpu_sample_desc(n, args.workload, seq) + ", 2 steps", "cpu_model": cpu_model()}
    est, per_tok = est_max_seq(S, shp, mem, n_loc, world)
    tokens = seq  # whole-job tokens per step (all ranks)
    line = {
        "metric": METRIC, "value": tokens / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, N(0,1) hidden, uniform labels)",
        "config": {"workload": workload_name(seq, world, args.layers, args.offload, args.workload), "seq_len": seq,
                   "tokens_per_gpu": n_loc, "sp_degree": world,
                   "transport": grp.transport if world > 1 else "none (SP=1)",
                   "mlp_tile": mem["mlp_tile"], "loss_tile": mem["loss_tile"],
                   "l2": "inputs larger than L2 (x 256 MiB/GPU, weights 1.5 GiB, activations ~3 GiB per step)"
                         if args.workload == "l1" else ("inputs larger than L2 (x 320 MiB/GPU, weights 2.5 GiB)"
                                                        if args.workload == "qwen" else
                                                        "no flush (tiny config: weights and activations fit in L2)"),
                   "optimizer": f"sgd lr={args.lr}" if args.lr > 0 else "none (fwd+bwd+SP grad all-reduce)",
                   "n_layers": args.layers, "rope_theta": args.rope,
                   "activation_checkpointing": ("offload to pinned host" if args.offload else
                                                ("device" if args.layers > 1 else "none (single layer)"))},
        "peak_hbm_bytes": peak_b, "peak_hbm_bytes_per_token": peak_b / n_loc,
        "est_max_seq_per_gpu": est,
        "est_max_seq_method": (f"spt_max_seqlen_solver: weights + grads + logits / MLP tile workspaces exact, "
                               f"{per_tok:.0f} B per local token (this run's ledger + the caller's input copy), HBM total - 3 GiB"),
        "loss": loss, "valid_tokens": cnt,
        "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(x.numel() * 2 + lab.numel() * 8) * world, "d2h_bytes_per_step": 32 * world},
        "gpu_launches": launches,
        "timing": "cuda-graph replay" if graph_used is True else f"eager launches ({graph_used or 'graph off'})",
        "cuda_graph": graph_used, "ms_per_step_eager_profiled": ms_eager,
        "breakdown_source": ("per-kernel-class CUDA events recorded inside the timed graph replays (the last one)"
                             if graph_used is True else f"profiled eager pass of {prof_steps} step(s) before the timed loop"),
        "roofline": roof,
        "breakdown_ms_per_step": breakdown, "class_tflops": tflops,
        # time of the step outside the profiled kernel regions (unprofiled small kernels + launch gaps), last step
        "gaps_ms_per_step": ({"total": round(gaps_last["ms"], 3), "n": gaps_last["n"],
                              "largest": {k: round(v, 3) for k, v in gaps_last["top"].items()}} if gaps_last else None),
        "all_to_all": a2a or None,
        "gemm_sites": {k: {"ms_per_step": round(v["ms"] / prof_steps, 3), "tflops": round(v["tflops"], 1)}
                       for k, v in sorted(sites_acc.items(), key=lambda kv: -kv[1]["ms"]) if not k.startswith("a2a_")},
        "clocks": clk.summary(),
        "cpu_baseline": cpu_v,
    }
    print(json.dumps(line), flush=True)
    eng.close()
    grp.close()


def free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seq", type=int, default=0, help="global sequence length (0: the workload's default for N)")
    ap.add_argument("--workload", default="l1", choices=sorted(SHAPES))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"], help="SP transport for N > 1")
    ap.add_argument("--lr", type=float, default=0.0)
    ap.add_argument("--loss-tile", type=int, default=0, help="tokens per tiled-logits/CE tile (0: the engine's rule)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=0, help="CPU sample size (0: 512 for l1, 8192 for tiny)")
    ap.add_argument("--cpu-reduced-n", default="2048,4096",
                    help="--impl reference, l1: also time one whole L-shape step at each of these N (0: skip)")
    ap.add_argument("--layers", type=int, default=1,
                    help="decoder layers (> 1: per-layer activation checkpointing; not the BASELINE config)")
    ap.add_argument("--offload", action="store_true", help="activation checkpoints in pinned host memory")
    ap.add_argument("--rope", type=float, default=0.0, help="RoPE theta (> 0 turns it on; not the BASELINE config)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time `value` with eager launches instead of a CUDA-graph replay of the step")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (what the driver does for N > 1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("SPT_BENCH_SAME_GPU") == "1":
        # functional test of the multi-process path on a one-GPU box: every rank on cuda:0 (the peer transport
        # maps the other processes' buffers with CUDA IPC as across GPUs; timings are time-sliced, not scaling)
        local_rank = 0
    if world != args.gpus and rank == 0:
        print(f"[bench] note: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        # torch.distributed is only the control plane (IPC-handle / NCCL-id exchange, barriers, the max over
        # ranks of the timings): gloo on host tensors; the data plane is the engine's own transport
        dist.init_process_group("gloo")
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
