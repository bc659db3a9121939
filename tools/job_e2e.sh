#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in 6 8 12 16 24; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-chunks $c 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('chunks $c', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['indexless_decode']['value'])" >> gpurun_out/e2e_sweep.txt
done
