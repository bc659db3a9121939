#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/t5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t5_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/t5_bench.json 2> gpurun_out/t5_bench.err
