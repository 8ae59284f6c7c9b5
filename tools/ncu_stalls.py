"""Stall-reason totals of one kernel in an ncu report, overall and per
barrier-delimited segment (BAR/BSYNC/WARPSYNC splits)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
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


segs = [[]]
for r in data:
    segs[-1].append(r)
    if "BAR.SYNC" in r[isrc] or "BAR.RED" in r[isrc]:
        segs.append([])
tot = {h[c]: sum(f(r[c]) for r in data) for c in cols}
T = sum(tot.values()) or 1
print("overall:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v / T > 0.01))
for i, sg in enumerate(segs):
    t = {h[c]: sum(f(r[c]) for r in sg) for c in cols}
    S = sum(t.values())
    if S / T < 0.02:
        continue
    print(f"seg {i} ({100*S/T:.1f}% of samples, {len(sg)} instrs):",
          ", ".join(f"{k[6:]} {100*v/S:.0f}%" for k, v in sorted(t.items(), key=lambda x: -x[1]) if v / S > 0.04))
