cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_configs.py -x -q -k "golden or whole or random or cfg1 or cast or short" > gpurun_out/j12_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j12_pytest.log
python tools/prof_ws.py fr > gpurun_out/j12_prof.txt 2>&1
python tools/prof_ws.py fq >> gpurun_out/j12_prof.txt 2>&1
python tools/time_encode.py whole > gpurun_out/j12_time.txt 2>&1
