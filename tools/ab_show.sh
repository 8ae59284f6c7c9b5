#!/bin/bash
# Summary of tools/ab_run.sh output (test tails, ms per step and phases).
cat gpurun_out/ab/t_*.log
for f in gpurun_out/ab/b*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d.get('phases_ms',{}).items()})"; done
