#!/bin/bash
# M2L timing ablations (variants built with -DVPG_M2L_ABL=bits, tools/mkvariant.sh):
# cfg2 phase split per variant.  Results of ablated builds are wrong by design.
O=gpurun_out/abl; mkdir -p $O
for v in main "$@"; do
  if [ $v = main ]; then unset VPG_LIB_PATH; else export VPG_LIB_PATH=$PWD/variants/$v/libvolpot_b200.so; fi
  VPG_BENCH_ABLATION=1 timeout 300 python bench.py --workload ${AB_WL:-cfg2} --steps 10 --warmup 3 --no-cpu-baseline > $O/$v.json 2> $O/$v.err
  python -c "
import json
d=json.load(open('$O/$v.json'))
print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})" 2>/dev/null || tail -2 $O/$v.err
done
