#!/bin/bash
# Symmetric near field, full and hybrid forms: parity tests, then bench auto vs off.
O=gpurun_out/sym2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
VPG_SYM=1 VPG_SYM_MIN=0 timeout 600 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
VPG_SYM=1 VPG_SYM_MIN=64 timeout 600 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
VPG_SYM=1 VPG_SYM_MIN=32 timeout 600 python -m pytest tests/test_gpu_fmm.py -x -q -k "sym or cfg1 or cfg2" 2>&1 | tail -1
for wl in cfg2 cfg4 cfg1 cfg3; do
  for v in auto off h32 h96; do
    case $v in auto) unset VPG_SYM VPG_SYM_MIN;; off) export VPG_SYM=0;; h32) export VPG_SYM=1 VPG_SYM_MIN=32;; h96) export VPG_SYM=1 VPG_SYM_MIN=96;; esac
    if [ $wl != cfg2 ] && [ $v = h32 -o $v = h96 ]; then continue; fi
    timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > $O/b_${wl}_$v.json 2> $O/b_${wl}_$v.err || tail -3 $O/b_${wl}_$v.err
    python -c "import json; d=json.load(open('$O/b_${wl}_$v.json')); print('$wl $v', round(d['ms_per_step'],4), round(d['phases_ms']['p2p'],4))"
    unset VPG_SYM VPG_SYM_MIN
  done
done
