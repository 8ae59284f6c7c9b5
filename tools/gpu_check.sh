timeout 500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -3 gpurun_out/bench_cfg2.err
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -3 gpurun_out/bench_cfg4.err
python -c "
import json
for f in ['gpurun_out/bench_cfg2.json','gpurun_out/bench_cfg4.json']:
    d=json.loads(open(f).read()); print(f, round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['phases_ms'].items()}, 'm2l TF', round(d['kernels']['m2l']['tflops_executed'],2), 'p2p Gpair/s', round(d['kernels']['p2p']['pairs_per_s']/1e9,1))
"
