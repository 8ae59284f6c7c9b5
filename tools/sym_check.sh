#!/bin/bash
# Symmetric near field: GPU tests (forced on), then cfg1/cfg2/cfg4 bench: auto / forced on / off.
O=gpurun_out/sym; mkdir -p $O
VPG_SYM=1 timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for wl in cfg2 cfg4 cfg1; do
  for v in auto on off; do
    case $v in auto) unset VPG_SYM;; on) export VPG_SYM=1;; off) export VPG_SYM=0;; esac
    timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > $O/b_${wl}_$v.json 2> $O/b_${wl}_$v.err || tail -3 $O/b_${wl}_$v.err
    python -c "import json; d=json.load(open('$O/b_${wl}_$v.json')); print('$wl $v', round(d['ms_per_step'],4), {k:round(x,4) for k,x in d['phases_ms'].items()})"
  done
done
unset VPG_SYM
