cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_configs.py -x -q > gpurun_out/j7_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j7_pytest.log
timeout 600 python tools/time_encode.py whole LOSSLESS > gpurun_out/j7_time.txt 2>&1
