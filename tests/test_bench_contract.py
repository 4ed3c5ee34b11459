"""bench.py output contract: the one JSON line the driver parses (keys, types, units), for the reference arm
on CPU and for the B200 arm (pytest -m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _check_common(d):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["unit"] == "tokens/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1
    assert "workload" in d["config"]
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["unit"] == d["unit"]


def test_reference_arm_contract():
    # small sample (64 tokens, each with its full-context attention rows in the 32K sequence) + the reduced-N step
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-tokens", "64", "--cpu-reduced-n", "128"],
             timeout=900)
    _check_common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert "32768-token sequence" in cb["sample"]
    assert [r["seq_len"] for r in d["cpu_reduced_n"]] == [128] and d["cpu_reduced_n"][0]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_contract():
    d = _run(["--steps", "2", "--warmup", "3"], timeout=1200)
    _check_common(d)
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
    assert roof["bound"] in ("hbm", "tensor") and 0 < roof["frac"] < 1.2
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")


@pytest.mark.gpu
def test_b200_arm_two_ranks_peer_transport_same_gpu():
    """The N > 1 bench path end to end on the one-GPU box: `--gpus 2` re-launches itself under
    torch.distributed.run, both ranks run on cuda:0 (SPT_BENCH_SAME_GPU=1) on the peer transport (CUDA IPC),
    the step is graph-captured and replayed in both processes, rank 0 prints one line with n_gpus = 2 and the
    per-collective all-to-all payload rates.  (Timings are time-sliced between the processes: this checks the
    plumbing, not scaling.)"""
    env = dict(os.environ, SPT_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--seq", "4096"], capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["sp_degree"] == 2 and d["config"]["transport"] == "peer"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["timing"] == "cuda-graph replay"
    assert {"a2a_qkv", "a2a_o", "a2a_do", "a2a_dqkv"} <= set(d["all_to_all"])
    assert all(v["gbps"] and v["gbps"] > 0 for v in d["all_to_all"].values())
