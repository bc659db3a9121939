#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_k5.py tests/test_d3_errors.py tests/test_gpu_parity.py tests/test_range_decode.py -x -q -m gpu > gpurun_out/il2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/il2_pytest.log
timeout 300 python tools/time_indexless.py > gpurun_out/il2_time.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/il2_launches.csv python tools/ncu_indexless.py > gpurun_out/il2_ncu.log 2>&1
