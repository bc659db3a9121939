#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 180 > gpurun_out/s4c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4c_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s4c_bench.json 2> gpurun_out/s4c_bench.err
for w in cfg1 cfg3; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/s4c_configs.json 2>> gpurun_out/s4c_configs.err; done
