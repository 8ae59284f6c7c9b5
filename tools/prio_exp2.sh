#!/bin/bash
run() { local name=$1; shift; env "$@" python bench.py --workload ${WL:-cfg2} --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/prio_$name.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/prio_$name.json')); print('${WL:-cfg2} $name', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"; }
for i in 1 2 3; do run base X=1; run prio VPG_PRIO=1; done
WL=cfg1; run base X=1; run prio VPG_PRIO=1
WL=cfg4; run base X=1; run prio VPG_PRIO=1
