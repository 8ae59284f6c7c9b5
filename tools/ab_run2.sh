#!/bin/bash
# A/B with parity: for main and every variants/<name>: FMM parity tests (the
# variant's .so via VPG_LIB_PATH), then cfg2 / cfg4 bench phases.
O=gpurun_out/ab; mkdir -p $O
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_golden.py tests/test_gpu_native.py -q -x 2>&1 | tail -2 > $O/t_$v.log
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b2_$v.json 2> $O/b2_$v.err
  python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/b4_$v.json 2> $O/b4_$v.err
done
