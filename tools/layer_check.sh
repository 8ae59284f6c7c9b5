#!/bin/bash
# Layer-potential evaluation on one B200: parity tests, bench line, launch list, one ncu --set full capture.
O=gpurun_out/layer; mkdir -p $O
timeout 500 python -m pytest tests/test_gpu_layer.py -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python bench.py --workload layer --steps 10 --warmup 3 > $O/bench_layer.json 2> $O/bench_layer.err || tail $O/bench_layer.err
python bench.py --workload layer --impl reference --steps 2 --warmup 1 > $O/bench_layer_ref.json 2> $O/bench_layer_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_layer.csv \
    python bench.py --workload layer --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"coarse_kernel|fine_kernel|records_kernel|ups_coef" -c 4 \
    -o $O/full_layer python bench.py --workload layer --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
