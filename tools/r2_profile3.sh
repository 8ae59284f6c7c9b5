#!/bin/bash
# Round-2 check 3: GPU suite, smoke, default bench, launch list + ncu of the cfg4 step kernels.
T=${1:-v3}; O=gpurun_out/prof_$T; mkdir -p $O
timeout 1150 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err || tail -3 $O/bench_cfg4.err
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 python tools/prof_apply.py --workload cfg4 --reps 1 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"p2p_sym_kernel|sym_finalize|l2p_kernel|m2l_kernel" -c 4 \
    -o $O/full_cfg4 python tools/prof_apply.py --workload cfg4 --reps 1 > $O/ncu_full4.log 2>&1
[ -f $O/full_cfg4.ncu-rep ] && python tools/ncu_raw.py $O/full_cfg4.ncu-rep > $O/full_cfg4_raw.txt 2>&1
for f in bench_cfg4 bench_cfg2; do echo "== $f"; cat $O/$f.json; echo; done
