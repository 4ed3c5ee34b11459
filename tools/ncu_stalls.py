"""Per-kernel stall breakdown from an ncu report: L2 / tensor / issue metrics, pc-sampling stall
reasons and the hottest SASS lines (with the instruction opcode mix of the stall samples)."""
import collections
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:60])
    for key in ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum.per_second",
                "l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
                "sm__cycles_elapsed.avg.per_second"):
        if key in hdr:
            print(f"   {key:70s} {r[hdr.index(key)]} {rows[1][hdr.index(key)]}")
    st = [(h, f(r[i])) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    for h, v in sorted(st, key=lambda x: -x[1])[:8]:
        print(f"   stall {h[33:]:30s} {100 * v / tot:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
seen, data = set(), []
for r in rows[2:]:
    if len(r) > si and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
tot = sum(f(r[si]) for r in data) or 1
ops = collections.Counter()
for r in data:
    t = r[1].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    ops[op.split(".")[0]] += f(r[si])
print("   opcode share of stall samples:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(10)))
addr = [r[0] for r in data]
for r in sorted(data, key=lambda r: -f(r[si]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    i = addr.index(r[0])
    ctx = " | ".join(x[1][:60] for x in data[max(0, i - 3):i])
    print(f"   {100 * f(r[si]) / tot:5.1f}%  {r[1][:70]:70s}  <- {ctx}")
