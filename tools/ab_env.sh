#!/bin/bash
# A/B of runtime switches: each argument is one variant, a space-separated
# list of VAR=VALUE settings ("-" = defaults).  Per variant: the symmetric
# near-field parity tests, then cfg4 (and $AB_WL, default cfg4) bench lines.
# usage: tools/ab_env.sh - "VPG_SYM_R4=1"
O=gpurun_out/abe; mkdir -p $O
WL=${AB_WL:-cfg4}
i=0
for v in "$@"; do
  i=$((i+1))
  envs=""; [ "$v" != "-" ] && envs="$v"
  if [ -z "$AB_NOTEST" ]; then
    env $envs VPG_SYM=1 timeout 400 python -m pytest tests/test_gpu_fmm.py -q -x -k "sym or cfg1 or cfg2 or shard" 2>&1 | tail -1
  fi
  for wl in $WL; do
    env $envs timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > $O/${wl}_$i.json 2>$O/${wl}_$i.err
    python -c "
import json
d=json.load(open('$O/${wl}_$i.json'))
print('$wl [$v]', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()}, 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || tail -2 $O/${wl}_$i.err
  done
done
