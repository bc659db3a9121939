#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_encode_v5.py -m gpu -x -q --timeout 180 > gpurun_out/t5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t5_pytest.log
