"""Top stalled SASS instructions of one kernel in an ncu report (source page):
samples, dominant stall reason, and the instruction, in address order for the
top N by samples.   python tools/ncu_hot.py report.ncu-rep kernel-regex [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = [i for i, x in enumerate(rows) if x and x[0] == "Address"][0]
h = rows[hdr]
data = [x for x in rows[hdr + 1:] if x and len(x) == len(h)]
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
isrc = h.index("Source")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[c]) for r in data for c in cols) or 1
scored = []
for idx, r in enumerate(data):
    s = {h[c][6:]: f(r[c]) for c in cols}
    scored.append((sum(s.values()), idx, s, r[isrc]))
top = sorted(scored, key=lambda x: -x[0])[:N]
for smp, idx, s, ins in sorted(top, key=lambda x: x[1]):
    main = sorted(s.items(), key=lambda x: -x[1])[:2]
    print(f"{idx:5d} {100*smp/tot:5.1f}%  {main[0][0]:>14s} {100*main[0][1]/max(smp,1):3.0f}%  {main[1][0]:>12s} {100*main[1][1]/max(smp,1):3.0f}%  {ins[:90]}")
