#!/bin/bash
# A/B of Helmholtz (native Chebyshev FMM) builds on cfg5: parity tests, operator apply phases.
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_helm.py -q -x 2>&1 | tail -1
  python bench.py --workload cfg5 --mode native --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k:round(x,3) for k,x in d['phases_ms'].items()})"
done
