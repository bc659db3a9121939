#!/bin/bash
# Per-config bench lines (BASELINE configs 1-5) on one GPU -> gpurun_out/configs.jsonl
cd "$(dirname "$0")/.."
out=gpurun_out/configs.jsonl; : > $out
for w in cfg1 cfg2 cfg3; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e 2>>gpurun_out/configs.err | tail -1 >> $out
done
timeout 900 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-e2e 2>>gpurun_out/configs.err | tail -1 >> $out
timeout 1200 python tools/sweep_cfg5.py 2>>gpurun_out/configs.err > gpurun_out/cfg5_sweep.jsonl
