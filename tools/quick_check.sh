#!/bin/bash
# Fast GPU iteration loop: FMM parity tests, then cfg2 / cfg4 bench phases.
timeout 400 python -m pytest tests/test_gpu_native.py tests/test_gpu_fmm.py tests/test_gpu_tree.py tests/test_gpu_golden.py -q -x 2>&1 | grep -E "Error|passed|failed" | tail -30 > gpurun_out/t.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2>> gpurun_out/b2.err
python bench.py --workload cfg3 --mode native --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2>> gpurun_out/b2.err
