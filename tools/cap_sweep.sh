#!/bin/bash
# Pass-threshold sweep (VPG_PASS_CAP) on one workload: phase times per cap.
W=${1:-cfg2}
for c in 0 16 32 64 128 256 1024 100000000; do
  VPG_PASS_CAP=$c python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']
print('$W cap', $c, round(d['ms_per_step'],4), {k: round(v,4) for k,v in p.items()})"
done
python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']
print('$W model', round(d['ms_per_step'],4), {k: round(v,4) for k,v in p.items()})"
