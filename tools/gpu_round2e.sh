#!/bin/bash
# Round-2 final measurement: GPU tests, smoke, default bench line,
# reference arm, other configs, launch list, ncu --set full of the encoder
# and decoder.  Outputs under gpurun_out/r2e_*.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/r2e_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2e_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2e_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2e_ref.json 2> gpurun_out/r2e_ref.err
for w in cfg1 cfg3 cfg4; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2e_configs.json 2>> gpurun_out/r2e_configs.err; done
timeout 600 python tools/time_encode.py > gpurun_out/r2e_time_encode.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2e_launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/r2e_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_v5|decode_v3" -s 6 -c 2 -o gpurun_out/r2e_full python bench.py --steps 2 --warmup 3 --profile > gpurun_out/r2e_ncu_full.log 2>&1
{ timeout 300 python tools/time_decode.py; timeout 300 python tools/time_ws_decode.py; } > gpurun_out/r2e_time_decode.txt 2>&1
