#!/bin/bash
# A/B of layer-evaluation builds: parity tests on main, then ms per eval for main + variants.
O=gpurun_out/abl; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_layer.py -q -x 2>&1 | tail -1
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  python bench.py --workload layer --steps 10 --warmup 3 --no-cpu-baseline > $O/$v.json 2> $O/$v.err
  python -c "import json; d=json.load(open('$O/$v.json')); print('$v', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done
