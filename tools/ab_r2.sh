#!/bin/bash
# Round-2 A/B: for main and every variants/<name>: FMM parity tests (the
# variant's .so via VPG_LIB_PATH), then cfg4 / cfg2 bench phases.
#   tools/ab_r2.sh [--quick] name...
O=gpurun_out/ab; mkdir -p $O
T="tests/test_gpu_fmm.py tests/test_gpu_golden.py tests/test_gpu_direct.py"
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  timeout 400 python -m pytest $T -q -x 2>&1 | grep -E "FAILED|Error|passed|failed|^E " | head -20 > $O/t_$v.log
  timeout 300 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $O/b4_$v.json 2> $O/b4_$v.err
  timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline > $O/b2_$v.json 2> $O/b2_$v.err
done
python tools/ab_show2.py main "$@"
