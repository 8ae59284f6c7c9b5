"""Summary of tools/ab_r2.sh outputs."""
import json
import sys

for v in sys.argv[1:]:
    t = open(f"gpurun_out/ab/t_{v}.log").read().strip().splitlines()
    print(f"== {v}: tests: {t[-1] if t else '?'}")
    for w in ("b4", "b2"):
        try:
            d = json.loads(open(f"gpurun_out/ab/{w}_{v}.json").read())
        except Exception as e:  # noqa: BLE001
            print(f"   {w}: no result ({e})")
            continue
        ph = {k: round(x, 4) for k, x in d["phases_ms"].items()}
        print(f"   {d['config']['workload']}: {d['ms_per_step']:.4f} ms  frac {d['roofline']['frac']:.3f}  {ph}")
