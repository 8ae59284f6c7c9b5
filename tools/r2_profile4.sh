#!/bin/bash
# Round-2 final check: GPU suite, smoke, every bench workload, launch list and
# ncu captures of the step kernels and the correction-build / operator kernels.
T=${1:-v4}; O=gpurun_out/prof_$T; mkdir -p $O
timeout 1150 python -m pytest tests -m gpu -q --durations=20 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err || tail -3 $O/bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --workload op_star --steps 10 --warmup 3 > $O/bench_op_star.json 2> $O/bench_op_star.err
timeout 900 python bench.py --workload corr --steps 3 --warmup 1 > $O/bench_corr.json 2> $O/bench_corr.err
timeout 600 python bench.py --workload cfg5 --mode native --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5n.json 2> $O/bench_cfg5n.err
timeout 600 python bench.py --workload layer --steps 10 --warmup 3 > $O/bench_layer.json 2> $O/bench_layer.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/op_probe.py --mesh star_h005 --reps 3 > $O/probe_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|charges_mma|corr_lattice|corr_desc16|classify_kernel" -c 8 \
    -o $O/op84k python tools/op_probe.py --mesh star_h005 --reps 3 > $O/ncu_op84k.log 2>&1
[ -f $O/op84k.ncu-rep ] && python tools/ncu_raw.py $O/op84k.ncu-rep > $O/op84k_raw.txt 2>&1
for f in bench_cfg4 bench_ref_cfg4 bench_cfg2 bench_op_star bench_corr bench_cfg5n bench_layer; do echo "== $f"; head -c 600 $O/$f.json; echo; done
