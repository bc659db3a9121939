#!/bin/bash
# Session re-entry check: full GPU tests, smoke, bench, index-less timing.
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4a_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err
timeout 300 python tools/time_indexless.py > gpurun_out/s4a_il.txt 2>&1
timeout 300 python tools/time_whole_stream.py > gpurun_out/s4a_ws.txt 2>&1
