"""Summarise an ncu report: SOL numbers + SASS hot spots with source lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Registers Per Thread", "Achieved Occupancy", "Tensor", "Warp Cycles Per Issued")
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("ID") != "0":
        continue
    if any(w in d["Metric Name"] for w in want):
        print(f"  {d['Metric Name'][:50]:50s} {d['Metric Value']} {d['Metric Unit']}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
iSrc = h.index("Source"); iA = h.index("Address")
def f(x):
    try: return float(x)
    except Exception: return None
data, seen = [], set()
for r in src[2:]:
    if len(r) <= iE or f(r[iS]) is None:
        continue
    if r[iA] in seen:
        break
    seen.add(r[iA]); data.append(r)
ts = sum(f(r[iS]) for r in data); te = sum(f(r[iE]) or 0 for r in data)
print(f"  samples {ts:.0f}  instructions {te:.3e}")
for i, r in enumerate(data):
    r.append(i)
for r in sorted(sorted(data, key=lambda r: -f(r[iS]))[:top], key=lambda r: r[-1]):
    print(f"  {r[-1]:5d} {f(r[iS]) / ts * 100:5.1f}% {((f(r[iE]) or 0) / te * 100):5.2f}%  {r[iSrc][:90]}")
