#!/bin/bash
# Round-2 profile on one B200 (from the repo root, under gpurun):
#   GPU test suite, default bench line (cfg4 + CPU baseline), the reference arm,
#   the ncu launch list of the bench command, --set full captures of the cfg4
#   step kernels and of cfg2's M2L / near field, raw pipe counters summarised.
# usage: tools/r2_profile.sh <tag> [--no-tests]
T=${1:-v1}; O=gpurun_out/prof_$T; mkdir -p $O
if [ "$2" != "--no-tests" ]; then
  timeout 1150 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
  tail -3 $O/pytest_gpu.log
fi
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err || { echo bench failed; tail $O/bench_cfg4.err; }
timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 python tools/prof_apply.py --workload cfg4 --reps 1 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"p2p_sym_kernel|sym_finalize|m2l_kernel|p2m_kernel|l2p_kernel|shift_kernel" -c 8 \
    -o $O/full_cfg4 python tools/prof_apply.py --workload cfg4 --reps 1 > $O/ncu_full4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"m2l_kernel|l2p_p2p_kernel|p2m_kernel" -c 4 \
    -o $O/full_cfg2 python tools/prof_apply.py --workload cfg2 --reps 1 > $O/ncu_full2.log 2>&1
for r in full_cfg4 full_cfg2; do
  [ -f $O/$r.ncu-rep ] && python tools/ncu_raw.py $O/$r.ncu-rep > $O/${r}_raw.txt 2>&1
  [ -f $O/$r.ncu-rep ] && python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1
done
cat $O/bench_cfg4.json $O/bench_cfg2.json $O/bench_ref_cfg4.json
echo done
