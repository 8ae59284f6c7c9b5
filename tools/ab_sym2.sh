#!/bin/bash
# A/B of symmetric-near-field builds with env switches: args are name[:ENV=VAL,...]
O=gpurun_out/abs; mkdir -p $O
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  tag=$(echo $spec | tr ':=,' '___')
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  E=$(echo $envs | tr ',' ' ')
  env $E VPG_SYM=1 timeout 300 python -m pytest tests/test_gpu_fmm.py -q -x -k "sym or cfg1 or cfg2 or shard" 2>&1 | tail -1
  for wl in cfg4 cfg3; do
    env $E python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu-baseline > $O/${wl}_$tag.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/${wl}_$tag.json')); print('$wl $tag', round(d['ms_per_step'],4), round(d['phases_ms']['p2p'],4))"
  done
done
