#!/bin/bash
# Round-2 profile v7: GPU suite, smoke, every bench workload, the launch list of the bench
# command and ncu --set full captures of the step's kernels (cfg4) and of cfg2's M2L / near field.
T=${1:-v8}; O=gpurun_out/prof_$T; mkdir -p $O
timeout 1150 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err || tail -3 $O/bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
for e in 1e-6 1e-9; do timeout 600 python bench.py --eps $e --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_eps$e.json 2> $O/bench_cfg4_eps$e.err; done
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --workload cfg3 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3_native.json 2> $O/bench_cfg3_native.err
timeout 600 python bench.py --workload cfg4 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_native.json 2> $O/bench_cfg4_native.err
timeout 900 python bench.py --workload op_star --steps 10 --warmup 3 > $O/bench_op_star.json 2> $O/bench_op_star.err
timeout 900 python bench.py --workload corr --steps 3 --warmup 1 > $O/bench_corr.json 2> $O/bench_corr.err
timeout 600 python bench.py --workload cfg5 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5n.json 2> $O/bench_cfg5n.err
timeout 600 python bench.py --workload layer --steps 10 --warmup 3 > $O/bench_layer.json 2> $O/bench_layer.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/prof_apply.py --workload cfg4 --reps 1 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"lattice_near|p2p_sym_kernel|sym_finalize|m2l_kernel|p2m_kernel|shift_kernel|gather_q" -c 7 \
    -o $O/full_cfg4 python tools/prof_apply.py --workload cfg4 --reps 1 > $O/ncu_full4.log 2>&1
python tools/prof_apply.py --workload cfg2 --reps 1 > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"m2l_kernel|l2p_p2p_kernel|p2m_kernel|l2p_kernel" -c 4 \
    -o $O/full_cfg2 python tools/prof_apply.py --workload cfg2 --reps 1 > $O/ncu_full2.log 2>&1
for r in full_cfg4 full_cfg2; do [ -f $O/$r.ncu-rep ] && python tools/ncu_raw.py $O/$r.ncu-rep > $O/${r}_raw.txt 2>&1; done
for f in bench_cfg4 bench_ref_cfg4 bench_cfg2 bench_op_star bench_corr bench_cfg5n bench_layer; do echo "== $f"; head -c 400 $O/$f.json; echo; done
# the pairwise symmetric kernel on the same workload (VPG_LATTICE=0): bench line and ncu capture
VPG_LATTICE=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_pairwise.json 2> $O/bench_cfg4_pairwise.err
VPG_LATTICE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"p2p_sym_kernel|sym_finalize" -c 2 \
    -o $O/full_cfg4_pairwise python tools/prof_apply.py --workload cfg4 --reps 1 > $O/ncu_full4p.log 2>&1
[ -f $O/full_cfg4_pairwise.ncu-rep ] && python tools/ncu_raw.py $O/full_cfg4_pairwise.ncu-rep > $O/full_cfg4_pairwise_raw.txt 2>&1
