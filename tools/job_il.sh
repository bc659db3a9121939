#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_k5.py tests/test_d3_errors.py tests/test_gpu_parity.py tests/test_range_decode.py tests/test_lossless_range.py -x -q -m gpu --timeout 300 > gpurun_out/il_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/il_pytest.log
timeout 300 python tools/time_decode.py > gpurun_out/il_time.txt 2>&1
timeout 600 python tools/fuzz_corrupt.py 400 > gpurun_out/il_fuzz.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/il_launches.csv python tools/ncu_indexless.py > gpurun_out/il_ncu.log 2>&1
