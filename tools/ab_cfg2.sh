#!/bin/bash
# A/B on cfg2 (and cfg4 phases) with FMM parity tests: main and the named variants.
O=gpurun_out/ab2; mkdir -p $O
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_golden.py -q -x 2>&1 | tail -1
  for wl in cfg2 cfg4; do
    python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > $O/${wl}_$v.json 2>$O/${wl}_$v.err
    python -c "import json; d=json.load(open('$O/${wl}_$v.json')); print('$wl $v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})"
  done
done
