"""Summarise an ncu report: headline metrics + stall samples per barrier-delimited segment."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(det)))
h = r[0]
keep = ['Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'No Eligible',
        'Grid Size', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'DRAM Throughput', 'Compute (SM) Throughput']
for row in r[1:]:
    if kfilter and kfilter not in row[h.index('Kernel Name')]:
        continue
    name = row[h.index('Metric Name')]
    if name in keep:
        print(f"{row[h.index('Kernel Name')][:28]:28s} {name[:38]:38s} {row[h.index('Metric Value')]} {row[h.index('Metric Unit')]}")
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kfilter:
    args[3:3] = ["-k", "regex:" + kfilter]
src = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = [i for i, x in enumerate(rows) if x and x[0] == "Address"]
if not hdr:
    sys.exit()
h = rows[hdr[0]]
end = hdr[1] if len(hdr) > 1 else len(rows)
data = [x for x in rows[hdr[0] + 1:end] if x and len(x) == len(h)]
isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(x[iss]) for x in data) or 1.0
seg, segs = 0, {}
for x in data:
    if 'BAR.SYNC' in x[isrc]:
        seg += 1
    segs.setdefault(seg, [0.0, 0.0])
    segs[seg][0] += f(x[iss])
    segs[seg][1] += f(x[iex])
print("segment  stall-samples%  warp-instr")
for k, v in segs.items():
    print(f"{k:7d}  {v[0] / tot * 100:13.1f}  {v[1]:.0f}")
top = sorted(data, key=lambda x: -f(x[iss]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]
print("top instructions by stall samples:")
for x in top:
    print(f"  {f(x[iss]) / tot * 100:5.1f}%  {x[isrc][:90]}")
