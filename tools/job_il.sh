#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_k5.py tests/test_d3_errors.py tests/test_gpu_parity.py tests/test_range_decode.py tests/test_fullsize_pins.py tests/test_distributed.py -x -q -m gpu --timeout 300 > gpurun_out/il_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/il_pytest.log
timeout 600 python tools/time_ws_decode.py > gpurun_out/ws_dec.txt 2>&1
timeout 600 python tools/fuzz_corrupt.py 300 9 > gpurun_out/il_fuzz.txt 2>&1
