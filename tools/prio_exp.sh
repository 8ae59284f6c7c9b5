#!/bin/bash
# Near field as retiring CTAs (VPG_P2P_QUOTA tasks per warp) on a low-priority side stream (VPG_PRIO=1).
run() { local name=$1; shift; env "$@" python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/prio_$name.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/prio_$name.json')); print('$name', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"; }
run base X=1
run prio VPG_PRIO=1
run q2 VPG_P2P_QUOTA=2
run prio_q1 VPG_PRIO=1 VPG_P2P_QUOTA=1
run prio_q2 VPG_PRIO=1 VPG_P2P_QUOTA=2
run prio_q4 VPG_PRIO=1 VPG_P2P_QUOTA=4
run prio_q8 VPG_PRIO=1 VPG_P2P_QUOTA=8
