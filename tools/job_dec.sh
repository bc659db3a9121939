#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_decode.py > gpurun_out/d4_time.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_d3_errors.py tests/test_k5.py tests/test_range_decode.py -x -q -m gpu > gpurun_out/d4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d4_pytest.log
