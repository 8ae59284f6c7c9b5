#!/bin/bash
# Round profile on one B200 (run under gpurun from the repo root):
#   1. the default bench line (cfg2, with the CPU baseline), plain run first;
#   2. the ncu launch list of the same bench command (cold, serialised);
#   3. `ncu --set full` captures: cfg2 step kernels, cfg4's symmetric near field;
#   4. bench lines of the other workloads (no CPU baseline) and the layer potential.
# Output under gpurun_out/prof/; summaries are copied into profiles/ by hand.
O=gpurun_out/prof
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err || { echo "bench failed"; tail $O/bench_cfg2.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/prof_apply.py --workload cfg2 --reps 1 > $O/plain.log 2>&1 || { echo "prof_apply failed"; exit 1; }
ncu --set full --clock-control none --import-source on \
    -k regex:"m2l_kernel|l2p_p2p_kernel|p2m_kernel|l2p_kernel|gather_q|shift_kernel" -c 8 \
    -o $O/full_cfg2 python tools/prof_apply.py --workload cfg2 --reps 1 > $O/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"p2p_sym_kernel|sym_finalize|m2l_kernel" -c 3 \
    -o $O/full_cfg4 python tools/prof_apply.py --workload cfg4 --reps 1 > $O/ncu_full4.log 2>&1
for w in cfg1 cfg4 cfg5; do
    python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --workload cfg3 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3_native.json 2> $O/bench_cfg3_native.err
python bench.py --workload cfg4 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_native.json 2> $O/bench_cfg4_native.err
python bench.py --workload cfg5 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5_native.json 2> $O/bench_cfg5_native.err
python bench.py --workload layer --steps 10 --warmup 3 > $O/bench_layer.json 2> $O/bench_layer.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err
echo done
