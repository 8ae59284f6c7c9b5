#!/bin/bash
# A/B of symmetric-near-field builds on cfg4 / cfg3 (reference mode), parity tests forced on.
O=gpurun_out/abs; mkdir -p $O
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  VPG_SYM=1 timeout 300 python -m pytest tests/test_gpu_fmm.py -q -x -k "sym or cfg1 or cfg2 or shard" 2>&1 | tail -1
  for wl in cfg4 cfg3; do
    python bench.py --workload $wl --steps 3 --warmup 2 --no-cpu-baseline > $O/${wl}_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/${wl}_$v.json')); print('$wl $v', round(d['ms_per_step'],4), round(d['phases_ms']['p2p'],4))"
  done
done
