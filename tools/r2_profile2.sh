#!/bin/bash
# Round-2 GPU check 2: the whole GPU suite, the default bench (cfg4) with the
# reference CPU arm, the operator and correction-build workloads.
T=${1:-v2}; O=gpurun_out/prof_$T; mkdir -p $O
timeout 1150 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err || tail -3 $O/bench_cfg4.err
timeout 900 python bench.py --workload op_star --steps 10 --warmup 3 > $O/bench_op_star.json 2> $O/bench_op_star.err || tail -3 $O/bench_op_star.err
timeout 900 python bench.py --workload corr --steps 3 --warmup 1 > $O/bench_corr.json 2> $O/bench_corr.err || tail -3 $O/bench_corr.err
timeout 600 python bench.py --workload cfg5 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5n.json 2> $O/bench_cfg5n.err
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
for f in bench_cfg4 bench_op_star bench_corr bench_cfg5n bench_cfg2 bench_ref_cfg4; do echo "== $f"; cat $O/$f.json; echo; done
