#!/bin/bash
# Round-2 GPU check: full GPU suite with durations, default bench (cfg4), a
# short reference-arm run.
mkdir -p gpurun_out
timeout 1150 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -3 gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err
cat gpurun_out/bench_default.json gpurun_out/bench_ref.json
