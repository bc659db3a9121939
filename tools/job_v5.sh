#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/v5_check.py small > gpurun_out/v5_small.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_small.txt
grep -q "ALL OK" gpurun_out/v5_small.txt || exit 0
timeout 300 python tools/v5_check.py > gpurun_out/v5_full.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_full.txt
timeout 600 python -m pytest tests/test_encode_v5.py -m gpu -x -q --timeout 180 > gpurun_out/t5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t5_pytest.log
