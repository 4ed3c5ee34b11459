"""Summarise ncu reports (.ncu-rep) and launch lists (csv) into the numbers profiles/README.md quotes.

  python tools/ncu_summary.py report.ncu-rep [...]      # key metrics per profiled kernel
  python tools/ncu_summary.py --launches launches.csv   # per-kernel share of a launch list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_active_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu(mufu)_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefronts_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    hdr, units, rows = raw(rep)
    for r in rows:
        name = r[hdr.index("Kernel Name")][:90]
        print(f"== {name}")
        for k, lab in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {lab:20s} {r[i]:>14s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__average_warp_latency_issue_stalled_", "")[:-6]))
                except ValueError:
                    pass
        if stalls:
            top = ", ".join(f"{n}={v:.1f}" for v, n in sorted(stalls, reverse=True)[:6])
            print(f"   top stalls (cycles/issue): {top}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue  # launch lists that also carry dram counters: durations only
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:60]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
        print(f"{v:10.3f} ms {100 * v / T:5.1f}%  n={cnt[k]:4d}  {k}")
    print(f"{T:10.3f} ms total ({sum(cnt.values())} launches)")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        for rep in sys.argv[1:]:
            summarise(rep)
