#!/bin/bash
# usage: tools/ncu_kernel.sh <workload> <kernel-regex> <out-name> [count]
# Runs the plain command first (must exit 0), then one ncu --set full capture.
W=$1; K=$2; O=$3; C=${4:-1}
python tools/prof_apply.py --workload $W --reps 1 ${MODE:+--mode $MODE} > gpurun_out/$O.plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C -o gpurun_out/$O python tools/prof_apply.py --workload $W --reps 1 ${MODE:+--mode $MODE} > gpurun_out/$O.ncu.log 2>&1
tail -1 gpurun_out/$O.ncu.log
