#!/bin/bash
# Step time of the graph apply vs how the side-stream near field shares the SMs.
O=gpurun_out/fork; mkdir -p $O
run() {  # name, env..., workload
  local name=$1; shift; local wl=$1; shift
  env "$@" python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > $O/$name.json 2> $O/$name.err
  python -c "import json,sys; d=json.load(open('$O/$name.json')); print('$name', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"
}
for wl in cfg2 cfg1; do
run ${wl}_default $wl X=1
run ${wl}_nofork $wl VPG_NO_FORK=1
for p in 30 50 70 85; do run ${wl}_pct$p $wl VPG_P2P_SIDE_PCT=$p; done
done
run cfg4_default cfg4 X=1
run cfg4_nofork cfg4 VPG_NO_FORK=1
run cfg4_pct85 cfg4 VPG_P2P_SIDE_PCT=85
