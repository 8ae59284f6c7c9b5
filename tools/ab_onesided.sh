#!/bin/bash
# A/B of one-sided near-field builds: parity tests, then cfg2 / op_star / cfg3 native phases.
O=gpurun_out/ab1; mkdir -p $O
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_golden.py tests/test_gpu_native.py -q -x 2>&1 | tail -1
  for wl in cfg2 op_star "cfg3 --mode native"; do
    tag=$(echo $wl | tr ' -' '__')
    python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu-baseline > $O/${tag}_$v.json 2>$O/${tag}_$v.err
    python -c "import json; d=json.load(open('$O/${tag}_$v.json')); print('$tag $v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})"
  done
done
