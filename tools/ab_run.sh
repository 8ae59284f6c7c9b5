#!/bin/bash
# A/B loop: parity tests on the main build, then cfg2/cfg4 bench phases for
# the main build and every variants/<name>/libvolpot_b200.so given as args.
O=gpurun_out/ab; mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_native.py tests/test_gpu_direct.py -q -x 2>&1 | tail -2 > $O/t_main.log
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b2_$v.json 2> $O/b2_$v.err
  python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/b4_$v.json 2> $O/b4_$v.err
done
